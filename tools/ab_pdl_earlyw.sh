#!/bin/bash
# A/B: PDL with the producer streaming delta weights before the wait (variant ew: DZ_PDL_EARLY_W=1,
# k_finalize 1 CTA/SM so k_sbmm can co-reside) under DZ_PDL=3, vs default (PDL off), vs f1 (1 CTA/SM
# finalize, PDL 3)
DZ_PDL=3 DZ_B200_LIB=$PWD/paper_2312_05215_b200/_dz_b200_ew.so timeout 600 python -m pytest tests/test_gpu_decode.py tests/test_gpu_stack.py tests/test_gpu_device_plan.py -x -q 2>&1 | tail -1
for i in 1 2 3; do for v in default ew f1; do
  if [ "$v" = "default" ]; then unset DZ_B200_LIB; unset DZ_PDL; else export DZ_B200_LIB=$PWD/paper_2312_05215_b200/_dz_b200_$v.so; export DZ_PDL=3; fi
  python bench.py --quick --no-e2e --steps 20 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', round(d['value'],1), round(d['ms_per_step'],3))"
done; done
