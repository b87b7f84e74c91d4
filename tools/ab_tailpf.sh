#!/bin/bash
# A/B: tail prefetch of the next launch's weights (default) vs none (DZ_TAIL_PREFETCH=0)
timeout 600 python -m pytest tests/test_gpu_stack.py tests/test_gpu_decode.py -x -q 2>&1 | tail -1
for i in 1 2 3; do for t in 0 1; do
  if [ "$t" = "0" ]; then export DZ_TAIL_PREFETCH=0; else unset DZ_TAIL_PREFETCH; fi
  python bench.py --quick --steps 20 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('tail_pf=$t', round(d['value'],1), round(d['ms_per_step'],3), 'e2e', round(d['e2e']['value'],1))"
done; done
