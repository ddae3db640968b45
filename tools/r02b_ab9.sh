#!/bin/bash
# small transfers off the copy engines (e2e) + 9-bit digits for the 64-bit-key sorts
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_full.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu_full.log
timeout 600 python bench.py --no-cpu > gpurun_out/bench_e2e.json 2>&1
timeout 600 python bench.py --no-cpu --workload nerfsynth200k > gpurun_out/bench_e2e_nerf.json 2>&1
PF_LIBRARY_PATH=$PWD/build/sort9.so timeout 1500 python -m pytest tests -m gpu -q -x -k "binning or cech or sweep" > gpurun_out/pytest_gpu_sort9.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu_sort9.log
VARIANTS="build/sort8.so build/sort9.so" bash tools/ab.sh; mv gpurun_out/ab.log gpurun_out/ab_sort.log
