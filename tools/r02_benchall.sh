#!/bin/bash
# round-2 bench lines of every workload + ncu captures of the tracer and detail kernels
mkdir -p gpurun_out/r02
B=gpurun_out/r02
timeout 900 python bench.py > $B/bench_train8_1m.json 2> $B/bench_train8_1m.err
timeout 900 python bench.py --workload mip360_1m --no-cpu > $B/bench_mip360_1m.json 2>&1
timeout 900 python bench.py --workload nerfsynth200k --no-cpu > $B/bench_nerfsynth200k.json 2>&1
timeout 1500 python bench.py --workload sweep64_3m --no-cpu --no-e2e --steps 3 > $B/bench_sweep64_3m.json 2>&1
timeout 900 python bench.py --dipoles --no-cpu > $B/bench_train8_1m_dipoles.json 2>&1
timeout 900 python bench.py --fisheye --no-cpu > $B/bench_train8_1m_fisheye.json 2>&1
timeout 900 python bench.py --lists knn --no-cpu > $B/bench_train8_1m_knn.json 2>&1
timeout 900 python bench.py --workload nerfsynth200k --detail 8 --no-cpu > $B/bench_nerfsynth200k_detail8.json 2>&1
timeout 900 python bench.py --detail 8 --no-cpu --steps 5 > $B/bench_train8_1m_detail8.json 2>&1
timeout 900 python bench.py --workload mip360_1m --trace --no-cpu --steps 5 > $B/bench_mip360_1m_trace.json 2>&1
timeout 900 python bench.py --workload mip360_1m --trace --fisheye --no-cpu --steps 5 > $B/bench_mip360_1m_trace_fisheye.json 2>&1
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $B/bench_reference.json 2>&1
rm -f gpurun_out/prof_*.ncu-rep
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k9_trace -c 1 \
    -o gpurun_out/prof_k9_trace python bench.py --workload mip360_1m --trace --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_k9.log 2>&1
for k in k7_backward k6_forward; do
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:$k -c 1 \
      -o gpurun_out/prof_${k}_detail python bench.py --workload nerfsynth200k --detail 8 --steps 1 \
      --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_${k}_detail.log 2>&1
done
nvidia-smi -q -d CLOCK > gpurun_out/smi_clocks.txt 2>&1
lscpu > gpurun_out/lscpu.txt 2>&1
