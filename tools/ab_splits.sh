#!/bin/bash
# A/B of the base K-split count per 7B decode shape (kbench, full case)
for sp in 1 2 3 4; do
  for s in "22016 4096" "4096 4096" "4096 11008" "12288 4096"; do set -- $s; echo -n "splits=$sp "; DZ_BASE_SPLITS=$sp python tools/kbench.py --out $1 --in $2 --case full; done
done
