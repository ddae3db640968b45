#!/bin/bash
mkdir -p gpurun_out
PF_LIBRARY_PATH=$PWD/build/ro1.so timeout 900 python -m pytest tests -m gpu -q -x -k "detail" > gpurun_out/pytest_gpu_ro.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu_ro.log
VARIANTS="build/ro0.so build/ro1.so" BENCH_ARGS="--detail 8" bash tools/ab.sh; mv gpurun_out/ab.log gpurun_out/ab_ro_train.log
VARIANTS="build/ro0.so build/ro1.so" BENCH_ARGS="--workload nerfsynth200k --detail 8" bash tools/ab.sh; mv gpurun_out/ab.log gpurun_out/ab_ro_nerf.log
