#!/bin/bash
# per-view K6 / K7 launches on two alternating streams
mkdir -p gpurun_out
PF_LIBRARY_PATH=$PWD/build/vs1.so timeout 2000 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_vs.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu_vs.log
grep -q "pytest exit 0" gpurun_out/pytest_gpu_vs.log || exit 0
VARIANTS="build/vs0.so build/vs1.so" bash tools/ab.sh; mv gpurun_out/ab.log gpurun_out/ab_vs.log
VARIANTS="build/vs0.so build/vs1.so" BENCH_ARGS="--dipoles" bash tools/ab.sh; mv gpurun_out/ab.log gpurun_out/ab_vs_dip.log
VARIANTS="build/vs0.so build/vs1.so" BENCH_ARGS="--detail 8" bash tools/ab.sh; mv gpurun_out/ab.log gpurun_out/ab_vs_det.log
