#!/bin/bash
mkdir -p gpurun_out/sanitizer
rm -f gpurun_out/sanitizer/summary.txt
PF_BENCH_SHARE_GPU=1 timeout 900 python bench.py --gpus 2 --steps 2 --warmup 1 --no-cpu --no-e2e > gpurun_out/bench_2rank.log 2>&1
echo "exit $?" >> gpurun_out/bench_2rank.log
PF_BENCH_SHARE_GPU=1 timeout 900 python bench.py --gpus 2 --steps 2 --warmup 1 --no-cpu --no-e2e --workload nerfsynth200k > gpurun_out/bench_2rank_nerf.log 2>&1
echo "exit $?" >> gpurun_out/bench_2rank_nerf.log
timeout 600 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1
echo "exit $?" >> gpurun_out/smoke.log
for tool in memcheck racecheck synccheck; do
  extra=""
  [ "$tool" = memcheck ] && extra="--leak-check full"
  [ "$tool" = racecheck ] && extra="--racecheck-report all"
  timeout 1200 compute-sanitizer --tool $tool $extra --error-exitcode 9 \
      python tools/sanitize_run.py tiny small5k > gpurun_out/sanitizer/$tool.log 2>&1
  echo "$tool exit $?" >> gpurun_out/sanitizer/summary.txt
done
