#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_multirank.py "tests/test_gpu_parity.py::test_binning_bit_exact" -q -x > gpurun_out/dbg1.log 2>&1
echo "exit $?" >> gpurun_out/dbg1.log
PF_REC_RATIO=6 timeout 600 python bench.py --no-cpu --no-e2e --steps 10 > gpurun_out/dbg_bench_rr6.json 2>&1
timeout 600 python bench.py --no-cpu --steps 10 > gpurun_out/dbg_bench.json 2>&1
