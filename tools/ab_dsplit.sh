#!/bin/bash
# A/B: decode delta-job K-splits by shape (default) vs none (DZ_DELTA_SPLITS=1)
for ds in 1 0; do
  if [ "$ds" = "1" ]; then export DZ_DELTA_SPLITS=1; else unset DZ_DELTA_SPLITS; fi
  for s in "22016 4096" "4096 4096" "4096 11008" "12288 4096"; do set -- $s; echo -n "dsplit=$ds "; python tools/kbench.py --out $1 --in $2 --case full; done
done
for i in 1 2; do for ds in 1 0; do
  if [ "$ds" = "1" ]; then export DZ_DELTA_SPLITS=1; else unset DZ_DELTA_SPLITS; fi
  python bench.py --quick --no-e2e --steps 20 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('bench dsplit=$ds', round(d['value'],1), d['roofline']['per_launch_us'])"
done; done
