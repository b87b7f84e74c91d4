#!/bin/bash
# compute-sanitizer (memcheck / racecheck / synccheck) over tools/sanitize.py and the 2-process
# fused-TP test, then the ncu launch list of the bench command and one --set full capture.
mkdir -p gpurun_out/san
python tools/sanitize.py > gpurun_out/san/plain.txt 2>&1; tail -1 gpurun_out/san/plain.txt
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize.py > gpurun_out/san/$tool.txt 2>&1
  echo "$tool rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/san/$tool.txt | tail -1)"
done
timeout 900 compute-sanitizer --tool memcheck --target-processes all python -m pytest tests/test_gpu_tp_fused.py -q -p no:cacheprovider > gpurun_out/san/memcheck_tp.txt 2>&1
echo "memcheck_tp rc=$? $(grep -E 'ERROR SUMMARY' gpurun_out/san/memcheck_tp.txt | tail -2 | tr '\n' ' ')"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_sbmm|k_finalize|k_plan" -c 300 --csv --log-file gpurun_out/r02_launches.csv python bench.py --steps 2 --warmup 1 --quick --no-e2e > gpurun_out/r02_launches.log 2>&1
echo "launch list rc=$?"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_sbmm|k_finalize" -s 16 -c 8 -o gpurun_out/r02_full python bench.py --layers 3 --steps 1 --warmup 1 --no-graph --quick --no-e2e > gpurun_out/r02_full.log 2>&1
echo "full capture rc=$?"
