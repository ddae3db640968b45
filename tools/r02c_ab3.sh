#!/bin/bash
# WarpStage float4 slots (ly1), + predicated tracked clip (ly2) vs pp0
mkdir -p gpurun_out
for v in ly1 ly2; do
PF_LIBRARY_PATH=$PWD/build/$v.so timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_$v.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu_$v.log
done
VARIANTS="build/pp0.so build/ly1.so build/ly2.so" bash tools/ab.sh; mv gpurun_out/ab.log gpurun_out/ab_ly.log
VARIANTS="build/pp0.so build/ly1.so build/ly2.so" BENCH_ARGS="--workload mip360_1m" bash tools/ab.sh; mv gpurun_out/ab.log gpurun_out/ab_ly_mip.log
VARIANTS="build/pp0.so build/ly1.so build/ly2.so" BENCH_ARGS="--detail 8 --workload nerfsynth200k" bash tools/ab.sh; mv gpurun_out/ab.log gpurun_out/ab_ly_det.log
