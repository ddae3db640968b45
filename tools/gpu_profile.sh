#!/bin/bash
# Run on the B200 box (gpurun): bench lines (default + other workloads), the
# reference arm, the ncu launch list and full captures of the hot kernels.
mkdir -p gpurun_out
rm -f gpurun_out/prof_*.ncu-rep gpurun_out/launches.csv
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 900 python bench.py --dipoles --no-cpu > gpurun_out/bench_dipoles.json 2>&1
timeout 900 python bench.py --workload mip360_1m --no-cpu > gpurun_out/bench_mip360.json 2>&1
timeout 900 python bench.py --workload nerfsynth200k --no-cpu > gpurun_out/bench_nerfsynth.json 2>&1
timeout 1500 python bench.py --workload sweep64_3m --no-cpu --no-e2e --steps 3 > gpurun_out/bench_sweep.json 2>&1
timeout 900 python bench.py --fisheye --no-cpu > gpurun_out/bench_fisheye.json 2>&1
timeout 900 python bench.py --workload nerfsynth200k --detail 8 --no-cpu > gpurun_out/bench_nerfsynth_detail.json 2>&1
timeout 900 python bench.py --detail 8 --no-cpu --steps 5 > gpurun_out/bench_detail.json 2>&1
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu \
    > gpurun_out/ncu_launch.log 2>&1
for k in k7_backward k6_forward; do
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:$k -c 1 \
      -o gpurun_out/prof_${k}_detail python bench.py --workload nerfsynth200k --detail 8 --steps 1 \
      --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_${k}_detail.log 2>&1
done
for k in k7_backward k6_forward k4_scatter c4_query; do
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:$k -c 1 \
      -o gpurun_out/prof_$k python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_$k.log 2>&1
done
# the inference (non-recording) K6 and K7's L2 reduction counts
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base mangled \
    -k regex:k6_forwardILb0ELb0ELb0ELi0ELb0E -c 1 -o gpurun_out/prof_k6_forward_inference \
    python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_k6_inf.log 2>&1
timeout 600 ncu --metrics lts__t_sectors_op_red.sum,lts__t_sectors_op_atom.sum,lts__t_requests_op_red.sum,smsp__inst_executed_op_global_red.sum,gpu__time_duration.sum,smsp__inst_executed.sum,sm__inst_executed_pipe_fma.sum,sm__inst_executed_pipe_alu.sum,sm__inst_executed_pipe_xu.sum \
    --clock-control none -k regex:k7_backward -c 1 python bench.py --steps 1 --warmup 1 --no-e2e \
    --no-cpu > gpurun_out/ncu_k7_atomics.txt 2>&1
timeout 900 python bench.py --lists knn --no-cpu > gpurun_out/bench_knn.json 2>&1
nvidia-smi -q -d CLOCK > gpurun_out/smi_clocks.txt 2>&1
lscpu > gpurun_out/lscpu.txt 2>&1
