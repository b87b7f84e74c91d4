#!/bin/bash
# A/B: tail-prefetch depth (stages of the next launch's first item): 6 (default) vs 3 vs 12
for i in 1 2; do for v in default tp3 tp12; do
  if [ "$v" = "default" ]; then unset DZ_B200_LIB; else export DZ_B200_LIB=$PWD/paper_2312_05215_b200/_dz_b200_$v.so; fi
  python bench.py --quick --no-e2e --steps 20 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', round(d['value'],1), round(d['ms_per_step'],3))"
done; done
