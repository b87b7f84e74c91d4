#!/bin/bash
# cfg3 (13B, 16 layers, 64 deltas 2-bit, 8 x 256 prefill + 128 decode) per K3 SM share of the
# overlapped mixed launch (0 = K3 then K2 on one stream; "auto" = engine.split_sms)
for o in ${OVL:-0 auto 64 88 108}; do
  if [ "$o" = auto ]; then a=""; else a="--overlap-sms $o"; fi
  timeout 900 python tools/stackbench.py --model 13b --layers 16 --deltas 64 --bits 2 --prefill 8x256 --decode 128 $a > gpurun_out/cfg3_o$o.json 2> gpurun_out/cfg3_o$o.err
  python -c "import json; d=json.load(open('gpurun_out/cfg3_o$o.json')); print('overlap=$o', 't_pf', d['t_pf'], 'jobs', d['n_pf_jobs'], 'ms/layer %.3f' % d['per_layer_ms'], 'TF %.0f' % d['TFLOPs'], 'tensor_frac %.3f' % d['tensor_frac'])" 2>/dev/null || tail -3 gpurun_out/cfg3_o$o.err
done
