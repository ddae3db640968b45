#!/bin/bash
# K7D contiguous-run loop A/B; K7 detail replay capture after the colour arena adapted
mkdir -p gpurun_out/export2
VARIANTS="build/rf0.so build/rf1.so" BENCH_ARGS="--workload nerfsynth200k --detail 8" bash tools/ab.sh; mv gpurun_out/ab.log gpurun_out/ab_nerf_detail.log
VARIANTS="build/rf0.so build/rf1.so" BENCH_ARGS="--detail 8" bash tools/ab.sh; mv gpurun_out/ab.log gpurun_out/ab_train_detail.log
NCU="timeout 900 ncu --set full --import-source on --clock-control none"
$NCU -k regex:k7_backward -s 8 -c 1 -o "gpurun_out/prof_k7_backward_detail@train8_1m+detail8" python bench.py --detail 8 --steps 2 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_k7d.log 2>&1
python tools/ncu_export.py r02 gpurun_out gpurun_out/export2 > gpurun_out/export2/export.log 2>&1
python tools/ncu_cuda_lines.py "gpurun_out/prof_k7_backward_detail@train8_1m+detail8.ncu-rep" 60 > gpurun_out/export2/k7_detail_lines.txt 2>&1
rm -f gpurun_out/prof_*.ncu-rep
