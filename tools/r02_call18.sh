#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x -k "full_image or plane_cull or large_sampled or fisheye or full_frame or static" > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
VARIANTS="build/cone.so default" bash tools/ab.sh
cp gpurun_out/ab.log gpurun_out/ab18.log
VARIANTS="build/cone.so default" BENCH_ARGS="--workload nerfsynth200k" bash tools/ab.sh
cat gpurun_out/ab.log >> gpurun_out/ab18.log
