#!/bin/bash
# A/B: finalize inside k_sbmm after a grid barrier (default) vs a separate k_finalize launch
timeout 600 python -m pytest tests/test_gpu_decode.py tests/test_gpu_parity.py tests/test_gpu_prefill.py tests/test_gpu_device_plan.py -x -q 2>&1 | tail -1
for i in 1 2; do for f in 0 1; do
  if [ "$f" = "0" ]; then export DZ_FIN_INLINE=0; else unset DZ_FIN_INLINE; fi
  python bench.py --quick --no-e2e --steps 20 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('fin_inline=$f', round(d['value'],1), round(d['ms_per_step'],3), d['roofline']['per_launch_us'])"
done; done
