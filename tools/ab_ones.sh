#!/bin/bash
# A/B: deferred code offset on the tensor core (ones-MMA, DZ_ONES_MMA=1) vs HSUB2 in registers
for v in "" ones; do
  if [ -n "$v" ]; then export DZ_B200_LIB=$PWD/paper_2312_05215_b200/_dz_b200_$v.so; else unset DZ_B200_LIB; fi
  for s in "22016 4096" "4096 4096" "4096 11008" "12288 4096"; do set -- $s; echo -n "$v "; python tools/kbench.py --out $1 --in $2 --case full; done
done
