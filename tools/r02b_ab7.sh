#!/bin/bash
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_full.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu_full.log
VARIANTS="default build/g8.so build/g2.so build/k6d2.so" BENCH_ARGS="--workload nerfsynth200k --detail 8" bash tools/ab.sh; mv gpurun_out/ab.log gpurun_out/ab_nerf_detail.log
VARIANTS="default build/g8.so build/k6d2.so" BENCH_ARGS="--detail 8" bash tools/ab.sh; mv gpurun_out/ab.log gpurun_out/ab_train_detail.log
