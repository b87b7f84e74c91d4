for pm in 128 64 32; do
  for cfg in "1 32" "1 64" "1 128" "4 64" "8 128" "16 256"; do set -- $cfg
    python tools/stackbench.py --model 7b --layers 4 --deltas $1 --decode $2 --zipf 1.5 --pf-min $pm --steps 5 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('pf_min=$pm D=$1 B=$2', round(d['ms_per_step'],3), 'ms', d['t_pf'], d['n_pf_jobs'])"
  done
done
