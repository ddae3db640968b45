#!/bin/bash
# K7 neighbour-RED aggregation A/B + GPU parity suite
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
VARIANTS="default build/agg0.so" bash tools/ab.sh; mv gpurun_out/ab.log gpurun_out/ab_plain.log
VARIANTS="default build/agg0.so" BENCH_ARGS="--dipoles" bash tools/ab.sh; mv gpurun_out/ab.log gpurun_out/ab_dip.log
