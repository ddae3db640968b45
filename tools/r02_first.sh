#!/bin/bash
# round-2 first GPU call: GPU tests, default bench, the other workloads' bench lines, launch list
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 900 python bench.py --workload mip360_1m --no-cpu > gpurun_out/bench_mip360.json 2>&1
timeout 900 python bench.py --workload nerfsynth200k --no-cpu > gpurun_out/bench_nerfsynth.json 2>&1
timeout 1500 python bench.py --workload sweep64_3m --no-cpu --no-e2e --steps 3 > gpurun_out/bench_sweep.json 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu \
    > gpurun_out/ncu_launch.log 2>&1
lscpu > gpurun_out/lscpu.txt 2>&1
