#!/bin/bash
# Prefill job size / remainder rule A/B on the 13B stack (4 layers, 64 2-bit deltas, 128 decode tokens)
for v in default j256r16 j240r64 j240r16; do
  if [ "$v" != "default" ]; then export DZ_B200_LIB=$PWD/paper_2312_05215_b200/_dz_b200_$v.so; else unset DZ_B200_LIB; fi
  for pre in 8x256 8x300 8x512 4x1000; do
    echo -n "$v $pre "; python tools/stackbench.py --model 13b --layers 4 --deltas 64 --bits 2 --prefill $pre --decode 128 --steps 5 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(round(d['per_layer_ms'],3), 'ms/layer', d['t_pf'], d['n_pf_jobs'])"
  done
done
