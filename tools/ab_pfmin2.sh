for pm in 256 100000; do
  for cfg in "1 128" "1 256" "2 512"; do set -- $cfg
    python tools/stackbench.py --model 7b --layers 4 --deltas $1 --decode $2 --zipf 1.5 --pf-min $pm --steps 5 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('pf_min=$pm D=$1 B=$2', round(d['ms_per_step'],3), 'ms', d['t_pf'], d['n_pf_jobs'])"
  done
  python tools/stackbench.py --model 7b --layers 4 --deltas 8 --prefill 4x256 --decode 0 --pf-min $pm --steps 5 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('pf_min=$pm 4x256 prefill', round(d['ms_per_step'],3), 'ms', d['t_pf'], d['n_pf_jobs'])"
  python tools/stackbench.py --model 7b --layers 4 --deltas 8 --prefill 2x256 --decode 0 --pf-min $pm --steps 5 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('pf_min=$pm 2x256 prefill', round(d['ms_per_step'],3), 'ms', d['t_pf'], d['n_pf_jobs'])"
done
