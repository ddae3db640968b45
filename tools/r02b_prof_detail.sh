#!/bin/bash
# source-level ncu captures of the detail K6/K7 (nerfsynth200k --detail 8, fused launch = 8 views)
mkdir -p gpurun_out
for k in k7_backward k6_forward; do
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:$k -c 1 \
      -o gpurun_out/prof_${k}_detail@nerfsynth200k+detail8 python bench.py --workload nerfsynth200k --detail 8 --steps 1 \
      --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_${k}_detail.log 2>&1
done
