for v in "" s2x5 s2x4 s4x3b1; do
  if [ -n "$v" ]; then export DZ_B200_LIB=$PWD/paper_2312_05215_b200/_dz_b200_$v.so; else unset DZ_B200_LIB; fi
  for s in "22016 4096" "4096 4096" "4096 11008" "12288 4096"; do set -- $s; echo -n "$v "; python tools/kbench.py --out $1 --in $2 --case full; done
done
