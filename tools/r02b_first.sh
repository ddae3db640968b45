#!/bin/bash
# re-entry sanity: GPU parity suite + default bench on HEAD
mkdir -p gpurun_out
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_head.log 2>&1
echo "bench exit $?" >> gpurun_out/bench_head.log
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
