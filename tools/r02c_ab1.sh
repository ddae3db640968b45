#!/bin/bash
# K6 kept-plane loop: position tracking (pt1), + unroll 4 (pt2) vs HEAD (pt0)
mkdir -p gpurun_out
for v in pt1 pt2; do
PF_LIBRARY_PATH=$PWD/build/$v.so timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_$v.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu_$v.log
done
VARIANTS="build/pt0.so build/pt1.so build/pt2.so" bash tools/ab.sh; mv gpurun_out/ab.log gpurun_out/ab_pt.log
VARIANTS="build/pt0.so build/pt1.so build/pt2.so" BENCH_ARGS="--workload mip360_1m" bash tools/ab.sh; mv gpurun_out/ab.log gpurun_out/ab_pt_mip.log
