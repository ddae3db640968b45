#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x -k "detail" > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
VARIANTS="default build/kp0.so" BENCH_ARGS="--workload nerfsynth200k --detail 8" bash tools/ab.sh; mv gpurun_out/ab.log gpurun_out/ab_nerf_detail.log
VARIANTS="default build/kp0.so" BENCH_ARGS="--detail 8" bash tools/ab.sh; mv gpurun_out/ab.log gpurun_out/ab_train_detail.log
