#!/bin/bash
# K6 -> K7 detail colour slots: parity (detail tests) + timing with / without slots
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x -k "detail or fisheye" > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
BENCH_ARGS="--workload nerfsynth200k --detail 8" bash tools/ab.sh; mv gpurun_out/ab.log gpurun_out/ab_nerf_detail.log
PF_COL_RATIO=0 BENCH_ARGS="--workload nerfsynth200k --detail 8" bash tools/ab.sh; mv gpurun_out/ab.log gpurun_out/ab_nerf_detail_nocol.log
BENCH_ARGS="--detail 8" bash tools/ab.sh; mv gpurun_out/ab.log gpurun_out/ab_train_detail.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_detail.csv python bench.py --workload nerfsynth200k --detail 8 --steps 2 --warmup 1 --no-e2e --no-cpu \
    > gpurun_out/ncu_launch_detail.log 2>&1
