#!/bin/bash
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -x -k "not sweep" > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
VARIANTS="build/notab.so default" bash tools/ab.sh
cp gpurun_out/ab.log gpurun_out/ab20.log
VARIANTS="build/notab.so default" BENCH_ARGS="--dipoles" bash tools/ab.sh
cat gpurun_out/ab.log >> gpurun_out/ab20.log
