#!/bin/bash
# Round-2 bench lines of every workload + the ncu launch list (no full captures)
# arm, the ncu launch list of the default bench and full captures of the hot kernels,
# each named prof_<kernel>@<workload> (the bench matches captures by workload)
mkdir -p gpurun_out/bench
rm -rf gpurun_out/prof_*.ncu-rep gpurun_out/launches.csv gpurun_out/export
B=gpurun_out/bench
timeout 900 python bench.py > $B/bench_train8_1m.json 2> $B/bench_train8_1m.err
timeout 900 python bench.py --dipoles --no-cpu > $B/bench_train8_1m_dipoles.json 2>&1
timeout 900 python bench.py --workload mip360_1m --no-cpu > $B/bench_mip360_1m.json 2>&1
timeout 900 python bench.py --workload nerfsynth200k --no-cpu > $B/bench_nerfsynth200k.json 2>&1
timeout 1500 python bench.py --workload sweep64_3m --no-cpu --no-e2e --steps 3 > $B/bench_sweep64_3m.json 2>&1
timeout 900 python bench.py --fisheye --no-cpu > $B/bench_train8_1m_fisheye.json 2>&1
timeout 900 python bench.py --workload nerfsynth200k --detail 8 --no-cpu > $B/bench_nerfsynth200k_detail8.json 2>&1
timeout 900 python bench.py --detail 8 --no-cpu --steps 5 > $B/bench_train8_1m_detail8.json 2>&1
timeout 900 python bench.py --lists knn --no-cpu > $B/bench_train8_1m_knn.json 2>&1
timeout 900 python bench.py --workload mip360_1m --trace --no-cpu --steps 5 > $B/bench_mip360_1m_trace.json 2>&1
timeout 900 python bench.py --workload mip360_1m --trace --fisheye --no-cpu --steps 5 > $B/bench_mip360_1m_trace_fisheye.json 2>&1
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $B/bench_reference.json 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu \
    > gpurun_out/ncu_launch.log 2>&1
mkdir -p gpurun_out/export
python tools/ncu_export.py r02 gpurun_out gpurun_out/export > gpurun_out/export/export.log 2>&1
