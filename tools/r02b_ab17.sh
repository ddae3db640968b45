#!/bin/bash
# K1 batched over the pinhole views of a sort batch
mkdir -p gpurun_out
PF_LIBRARY_PATH=$PWD/build/k1b.so timeout 900 python -m pytest tests -m gpu -q -x -k "binning or multiview or sweep or fisheye or static" > gpurun_out/pytest_gpu_k1.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu_k1.log
grep -q "pytest exit 0" gpurun_out/pytest_gpu_k1.log || exit 0
VARIANTS="build/k1a.so build/k1b.so" bash tools/ab.sh; mv gpurun_out/ab.log gpurun_out/ab_k1.log
VARIANTS="build/k1a.so build/k1b.so" BENCH_ARGS="--workload nerfsynth200k" bash tools/ab.sh; mv gpurun_out/ab.log gpurun_out/ab_k1_nerf.log
