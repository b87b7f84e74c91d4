#!/bin/bash
# A/B: programmatic dependent launch on both the SBMM kernels and k_finalize (DZ_PDL=3) vs off
for i in 1 2 3; do for f in 0 3; do
  DZ_PDL=$f python bench.py --quick --no-e2e --steps 20 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('DZ_PDL=$f', round(d['value'],1), round(d['ms_per_step'],3))"
done; done
