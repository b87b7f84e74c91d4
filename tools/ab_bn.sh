#!/bin/bash
# A/B: base-GEMM jobs of 64 (default) vs 128 tokens (DZ_BASE_JOB_TOKENS=128) at T=64 and T=128
for v in default bn128; do
  if [ "$v" != "default" ]; then export DZ_B200_LIB=$PWD/paper_2312_05215_b200/_dz_b200_$v.so; else unset DZ_B200_LIB; fi
  for t in 64 128; do
    for s in "22016 4096" "4096 4096" "4096 11008" "12288 4096"; do set -- $s; echo -n "$v T=$t "; python tools/kbench.py --out $1 --in $2 --tokens $t --case full; done
  done
  echo -n "$v cfg3-decode "; python tools/stackbench.py --model 13b --layers 2 --deltas 64 --bits 2 --decode 128 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['per_layer_ms'], d['hbm_frac'])"
done
