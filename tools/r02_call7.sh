#!/bin/bash
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
VARIANTS="build/base.so default" bash tools/ab.sh
timeout 600 python bench.py --workload sweep64_3m --no-cpu --no-e2e --steps 3 > gpurun_out/bench_sweep.json 2>&1
