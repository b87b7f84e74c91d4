#!/bin/bash
# A/B of library variants on the default bench: tools/ab_libs.sh name1 name2 ... ("base" = _dz_b200.so)
mkdir -p gpurun_out
for rep in $(seq 1 ${REPS:-2}); do
for v in "$@"; do
  if [ "$v" = base ]; then unset DZ_B200_LIB; else export DZ_B200_LIB=$PWD/paper_2312_05215_b200/_dz_b200_$v.so; fi
  timeout 600 python bench.py --quick --no-e2e --steps 10 --warmup 3 ${BENCH_EXTRA} > gpurun_out/ab_$v.txt 2>&1
  tail -1 gpurun_out/ab_$v.txt | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['value'],1), {k: round(x,1) for k,x in d['roofline']['per_launch_us'].items()})" 2>/dev/null || (echo "$v FAILED"; tail -3 gpurun_out/ab_$v.txt)
done; done
