#!/bin/bash
mkdir -p gpurun_out
: > gpurun_out/ab.log
timeout 1500 python -m pytest tests -m gpu -q -x -k "trace or detail or fisheye" > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
PF_LIBRARY_PATH=$PWD/build/det_m2.so timeout 1200 python -m pytest tests -m gpu -q -x -k "detail" > gpurun_out/pytest_gpu_m2.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu_m2.log
VARIANTS="build/base.so default build/det_m2.so" BENCH_ARGS="--workload nerfsynth200k --detail 8" bash tools/ab.sh
cp gpurun_out/ab.log gpurun_out/ab_detail.log
timeout 900 python bench.py --workload mip360_1m --trace --no-cpu --no-e2e --steps 3 2>&1 | tail -1 > gpurun_out/bench_trace.json
