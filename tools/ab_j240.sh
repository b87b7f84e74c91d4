#!/bin/bash
# A/B: prefill jobs of 256 tokens (single-buffered accumulator next to the sparse metadata) vs 240
# (double-buffered): kernel bench at 240-token requests, and the cfg3 stack (256-token requests)
for v in default j240; do
  if [ "$v" != "default" ]; then export DZ_B200_LIB=$PWD/paper_2312_05215_b200/_dz_b200_$v.so; else unset DZ_B200_LIB; fi
  python tools/pfbench.py --ptok 240 --shapes 5120x5120,13824x5120,5120x13824,27648x5120 | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print('$v', d['shape'], round(d['us'],1), 'us', round(d['alg_tflops']), 'alg TF/s')"
  echo -n "$v cfg3 "; python tools/stackbench.py --model 13b --layers 4 --deltas 64 --bits 2 --prefill 8x256 --decode 128 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['per_layer_ms'])"
done
