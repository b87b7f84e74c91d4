#!/bin/bash
# A/B of library variants on a cfg5 subset (7B, 4 layers, Zipf 1.5) and the headline bench:
#   tools/ab_cfg5.sh name1 name2 ...   ("base" = _dz_b200.so)
mkdir -p gpurun_out
PTS=${PTS:-"1:1,1:8,1:64,1:128,8:16,16:64,128:8,128:64,128:256"}
for rep in 1 2; do
for v in "$@"; do
  if [ "$v" = base ]; then unset DZ_B200_LIB; else export DZ_B200_LIB=$PWD/paper_2312_05215_b200/_dz_b200_$v.so; fi
  timeout 600 python tools/stackbench.py --model 7b --layers 4 --deltas 128 --sweep --zipf 1.5 --steps 5 --points $PTS ${EXTRA} > gpurun_out/ab5_$v.jsonl 2>&1
  python - "$v" <<'PY'
import json, sys
r = [json.loads(l) for l in open(f"gpurun_out/ab5_{sys.argv[1]}.jsonl") if l.startswith("{")]
print(sys.argv[1], " ".join(f"{d['sweep_D']}:{d['batch']}={d['hbm_frac']:.3f}" for d in r))
PY
done; done
