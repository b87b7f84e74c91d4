#!/bin/bash
# cfg3 per library variant: tools/ab_cfg3_libs.sh base variant ...  (EXTRA: extra stackbench args)
EXTRA=${EXTRA:-"--prefill 8x256 --decode 128"}
for rep in 1 2; do for v in "$@"; do
  if [ "$v" = base ]; then unset DZ_B200_LIB; else export DZ_B200_LIB=$PWD/paper_2312_05215_b200/_dz_b200_$v.so; fi
  timeout 900 python tools/stackbench.py --model 13b --layers 16 --deltas 64 --bits 2 $EXTRA > gpurun_out/cfg3_$v.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/cfg3_$v.json')); print('$v', 'jobs', d['n_pf_jobs'], 't_pf', d['t_pf'], 'ms/layer %.3f TF %.0f tensor %.3f' % (d['per_layer_ms'], d['TFLOPs'], d['tensor_frac']))"
done; done
