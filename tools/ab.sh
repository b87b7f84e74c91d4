#!/bin/bash
# A/B kernel variants on the three 7B shapes: tools/ab.sh <variant>... ("" = default library)
for v in "$@"; do
  lib=paper_2312_05215_b200/_dz_b200${v:+_$v}.so
  echo "== ${v:-default}"
  for shp in "--out 4096" "--out 11008" "--out 4096 --in 11008" "--out 12288" "--out 22016"; do
    DZ_B200_LIB=$PWD/$lib python tools/kbench.py $shp --case full 2>&1 | tail -1
  done
done
