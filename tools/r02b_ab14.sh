#!/bin/bash
# onesweep radix sort: bit-exact binning / Cech tests with the variant, then timing
mkdir -p gpurun_out
PF_LIBRARY_PATH=$PWD/build/os1.so timeout 900 python -m pytest tests -m gpu -q -x -k "binning or cech or sweep or multiview" > gpurun_out/pytest_gpu_os.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu_os.log
grep -q "pytest exit 0" gpurun_out/pytest_gpu_os.log || exit 0
VARIANTS="build/os0.so build/os1.so" bash tools/ab.sh; mv gpurun_out/ab.log gpurun_out/ab_os.log
VARIANTS="build/os0.so build/os1.so" BENCH_ARGS="--workload nerfsynth200k" bash tools/ab.sh; mv gpurun_out/ab.log gpurun_out/ab_os_nerf.log
