#!/bin/bash
# A/B on v17: mbarrier try_wait suspend-time hint 64 us (h64k) / 1 ms (h1m) vs hardware default
DZ_B200_LIB=$PWD/paper_2312_05215_b200/_dz_b200_h1m.so timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -1
for v in default h64k h1m; do
  if [ "$v" = "default" ]; then unset DZ_B200_LIB; else export DZ_B200_LIB=$PWD/paper_2312_05215_b200/_dz_b200_$v.so; fi
  echo -n "$v bits4 "; python tools/kbench.py --out 13824 --in 5120 --tokens 128 --deltas 64 --bits 4 --case full 2>/dev/null | tail -1
done
for i in 1 2 3; do for v in default h64k h1m; do
  if [ "$v" = "default" ]; then unset DZ_B200_LIB; else export DZ_B200_LIB=$PWD/paper_2312_05215_b200/_dz_b200_$v.so; fi
  python bench.py --quick --no-e2e --steps 20 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('bench $v', round(d['value'],1), round(d['ms_per_step'],3))"
done; done
