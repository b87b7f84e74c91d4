#!/bin/bash
# A/B on v17: non-volatile shared loads (nv) vs volatile (default)
DZ_B200_LIB=$PWD/paper_2312_05215_b200/_dz_b200_nv.so timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -1
for v in default nv; do
  if [ "$v" = "default" ]; then unset DZ_B200_LIB; else export DZ_B200_LIB=$PWD/paper_2312_05215_b200/_dz_b200_$v.so; fi
  for b in 4 2; do echo -n "$v bits$b "; python tools/kbench.py --out 13824 --in 5120 --tokens 128 --deltas 64 --bits $b --case full 2>/dev/null | tail -1; done
done
for i in 1 2 3; do for v in default nv; do
  if [ "$v" = "default" ]; then unset DZ_B200_LIB; else export DZ_B200_LIB=$PWD/paper_2312_05215_b200/_dz_b200_$v.so; fi
  python bench.py --quick --no-e2e --steps 20 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('bench $v', round(d['value'],1), round(d['ms_per_step'],3))"
done; done
