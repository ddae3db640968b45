#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x -k "record or overflow or multiview or dipole or cull" > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
VARIANTS="default build/base.so" bash tools/ab.sh; mv gpurun_out/ab.log gpurun_out/ab_plain.log
VARIANTS="default build/base.so" BENCH_ARGS="--dipoles" bash tools/ab.sh; mv gpurun_out/ab.log gpurun_out/ab_dip.log
