#!/bin/bash
# Standard GPU cycle: parity tests, then the default bench. Outputs under gpurun_out/.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gpu_tests.txt 2>&1
echo "TESTS: $(tail -1 gpurun_out/gpu_tests.txt)"
if [ "${SKIP_BENCH:-0}" != "1" ]; then
  timeout 900 python bench.py ${BENCH_ARGS} > gpurun_out/bench.txt 2>&1
  tail -1 gpurun_out/bench.txt | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('BENCH value=%.1f tok/s ms=%.2f GBps=%.0f frac=%.3f e2e=%.1f per_launch=%s clocks=%s' % (d['value'], d['ms_per_step'], d['roofline']['achieved'], d['roofline']['frac'], (d['e2e'] or {}).get('value', 0), d['roofline']['per_launch_us'], d['clocks']))" 2>/dev/null || tail -20 gpurun_out/bench.txt
fi
