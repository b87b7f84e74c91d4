#!/bin/bash
# BASELINE configs 3-5 through the layer-stack bench (tools/stackbench.py); one JSON line each.
set -u
O=${1:-gpurun_out}
mkdir -p $O
timeout 900 python tools/stackbench.py --model 13b --layers 16 --deltas 64 --bits 2 --prefill 8x256 --decode 128 > $O/cfg3.json 2> $O/cfg3.err
timeout 900 python tools/stackbench.py --model 13b --layers 16 --deltas 64 --bits 2 --prefill 8x256 --decode 128 --pf-min 100000 > $O/cfg3_nopf.json 2> $O/cfg3_nopf.err
timeout 900 python tools/stackbench.py --model 70b --layers 8 --deltas 16 --decode 64 > $O/cfg4_tp1.json 2> $O/cfg4_tp1.err
for w in 2 4 8; do
  timeout 900 python tools/stackbench.py --model 70b --layers 8 --deltas 16 --decode 64 --world $w > $O/cfg4_tp$w.json 2> $O/cfg4_tp$w.err
done
timeout 1500 python tools/stackbench.py --model 7b --layers 4 --deltas 128 --sweep --zipf 1.5 --steps 5 > $O/cfg5_sweep.jsonl 2> $O/cfg5.err
