#!/bin/bash
# A/B: L2 prefetch of an item's chunks ahead of the TMA ring (DZ_PF_AHEAD_BASE / _DELTA)
for v in default pfb4 pfb8 pfb4d2; do
  if [ "$v" = "default" ]; then unset DZ_B200_LIB; else export DZ_B200_LIB=$PWD/paper_2312_05215_b200/_dz_b200_$v.so; fi
  echo -n "$v base_only 4096x4096 T=16: "; python tools/kbench.py --out 4096 --in 4096 --tokens 16 --deltas 4 --case base_only 2>/dev/null | tail -1
  echo -n "$v cfg1: "; python tools/cfg1.py 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['device_us'],1), 'us')"
done
for i in 1 2; do for v in default pfb4 pfb4d2; do
  if [ "$v" = "default" ]; then unset DZ_B200_LIB; else export DZ_B200_LIB=$PWD/paper_2312_05215_b200/_dz_b200_$v.so; fi
  python bench.py --quick --no-e2e --steps 20 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('bench $v', round(d['value'],1), round(d['ms_per_step'],3), d['roofline']['per_launch_us'])"
done; done
