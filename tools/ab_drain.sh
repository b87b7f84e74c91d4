#!/bin/bash
# A/B on v16: base TMEM drain with two loads per wait (drain) vs one (default)
DZ_B200_LIB=$PWD/paper_2312_05215_b200/_dz_b200_drain.so timeout 600 python -m pytest tests/test_gpu_decode.py tests/test_gpu_parity.py -x -q 2>&1 | tail -1
for v in default drain; do
  if [ "$v" = "default" ]; then unset DZ_B200_LIB; else export DZ_B200_LIB=$PWD/paper_2312_05215_b200/_dz_b200_$v.so; fi
  echo -n "$v base_only 4096x11008 "; python tools/kbench.py --out 4096 --in 11008 --tokens 64 --deltas 4 --case base_only --debug 2 2>/dev/null | tail -1
  echo -n "$v base_only 12288x4096 "; python tools/kbench.py --out 12288 --in 4096 --tokens 64 --deltas 4 --case base_only --debug 2 2>/dev/null | tail -1
done
for i in 1 2 3; do for v in default drain; do
  if [ "$v" = "default" ]; then unset DZ_B200_LIB; else export DZ_B200_LIB=$PWD/paper_2312_05215_b200/_dz_b200_$v.so; fi
  python bench.py --quick --no-e2e --steps 20 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('bench $v', round(d['value'],1), round(d['ms_per_step'],3))"
done; done
