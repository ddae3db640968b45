#!/bin/bash
mkdir -p gpurun_out
M=gpu__time_duration.sum,smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,smsp__inst_executed_op_local_ld.sum,sm__warps_active.avg.pct_of_peak_sustained_active
for v in base default; do
  unset PF_LIBRARY_PATH
  [ $v = base ] && export PF_LIBRARY_PATH=$PWD/build/base.so
  timeout 900 ncu --metrics $M --clock-control none -k regex:k6_forward -s 8 -c 8 --csv \
    python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu16_$v.csv 2>&1
done
