#!/bin/bash
# split detail backward on two streams (arena halves)
mkdir -p gpurun_out
PF_LIBRARY_PATH=$PWD/build/d2.so timeout 1500 python -m pytest tests -m gpu -q -x -k "detail or fisheye" > gpurun_out/pytest_gpu_d2.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu_d2.log
grep -q "pytest exit 0" gpurun_out/pytest_gpu_d2.log || exit 0
VARIANTS="build/d1.so build/d2.so" BENCH_ARGS="--detail 8" bash tools/ab.sh; mv gpurun_out/ab.log gpurun_out/ab_d2.log
