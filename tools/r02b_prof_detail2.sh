#!/bin/bash
# split detail backward: launch list + full captures of the replay K7 and K7D (nerfsynth200k+detail8)
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_detail.csv python bench.py --workload nerfsynth200k --detail 8 --steps 2 --warmup 1 --no-e2e --no-cpu \
    > gpurun_out/ncu_launch_detail.log 2>&1
for k in k7_backward k7d_detail_chain; do
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:$k -c 1 \
      -o gpurun_out/prof_${k}_detail@nerfsynth200k+detail8 python bench.py --workload nerfsynth200k --detail 8 --steps 1 \
      --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_${k}_detail.log 2>&1
done
