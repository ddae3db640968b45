#!/bin/bash
# tracer tests + plane-cull exactness, sanitizer (memcheck/racecheck), bench lines, K6/K7 full ncu captures
mkdir -p gpurun_out/sanitizer
timeout 1500 python -m pytest tests -m gpu -q -rA -s -k "trace or plane_cull or full_frame" > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
rm -f gpurun_out/sanitizer/summary.txt
for tool in memcheck racecheck; do
  extra=""
  [ "$tool" = memcheck ] && extra="--leak-check full"
  timeout 1200 compute-sanitizer --tool $tool $extra --error-exitcode 9 \
      python tools/sanitize_run.py tiny small5k > gpurun_out/sanitizer/$tool.log 2>&1
  echo "$tool exit $?" >> gpurun_out/sanitizer/summary.txt
done
timeout 900 python bench.py --no-cpu > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 900 python bench.py --workload mip360_1m --trace --no-cpu > gpurun_out/bench_trace.json 2>&1
rm -f gpurun_out/prof_*.ncu-rep
for k in k6_forward k7_backward; do
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:$k -c 1 \
      -o gpurun_out/prof_$k python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_$k.log 2>&1
done
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k9_trace -c 1 \
      -o gpurun_out/prof_k9_trace python bench.py --workload mip360_1m --trace --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_k9.log 2>&1
