#!/bin/bash
# A/B: 16 consumer warps x 1 row group (nw16) vs 8 x 2 (default), current kernel
DZ_B200_LIB=$PWD/paper_2312_05215_b200/_dz_b200_nw16.so timeout 600 python -m pytest tests/test_gpu_decode.py -x -q 2>&1 | tail -1
for i in 1 2 3; do for v in default nw16; do
  if [ "$v" = "default" ]; then unset DZ_B200_LIB; else export DZ_B200_LIB=$PWD/paper_2312_05215_b200/_dz_b200_$v.so; fi
  python bench.py --quick --no-e2e --steps 20 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', round(d['value'],1), round(d['ms_per_step'],3))"
done; done
