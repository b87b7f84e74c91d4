#!/bin/bash
# A/B: 16 consumer warps x 1 row group (DZ_NW=16) vs 8 x 2
DZ_B200_LIB=$PWD/paper_2312_05215_b200/_dz_b200_w16.so timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_decode.py -x -q -m "gpu and not slow" 2>&1 | tail -2
for v in "" w16; do
  if [ -n "$v" ]; then export DZ_B200_LIB=$PWD/paper_2312_05215_b200/_dz_b200_$v.so; else unset DZ_B200_LIB; fi
  for s in "22016 4096" "4096 4096" "4096 11008" "12288 4096"; do set -- $s; echo -n "$v "; python tools/kbench.py --out $1 --in $2 --case full; done
done
