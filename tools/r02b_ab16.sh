#!/bin/bash
# radix sort: ballot-built digit peers instead of __match_any_sync
mkdir -p gpurun_out
PF_LIBRARY_PATH=$PWD/build/sb1.so timeout 900 python -m pytest tests -m gpu -q -x -k "binning or cech or sweep or multiview" > gpurun_out/pytest_gpu_sb.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu_sb.log
grep -q "pytest exit 0" gpurun_out/pytest_gpu_sb.log || exit 0
VARIANTS="build/sb0.so build/sb1.so" bash tools/ab.sh; mv gpurun_out/ab.log gpurun_out/ab_sb.log
VARIANTS="build/sb0.so build/sb1.so" BENCH_ARGS="--workload nerfsynth200k" bash tools/ab.sh; mv gpurun_out/ab.log gpurun_out/ab_sb_nerf.log
