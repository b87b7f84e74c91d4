#!/bin/bash
# A/B of library variants on the 7B decode shapes: bash tools/ab_generic.sh "" variant1 variant2 ...
for v in "$@"; do
  if [ -n "$v" ] && [ "$v" != "default" ]; then export DZ_B200_LIB=$PWD/paper_2312_05215_b200/_dz_b200_$v.so; else unset DZ_B200_LIB; fi
  for s in "22016 4096" "4096 4096" "4096 11008" "12288 4096"; do set -- $s; echo -n "$v "; python tools/kbench.py --out $1 --in $2 --case full; done
done
