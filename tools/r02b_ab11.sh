#!/bin/bash
mkdir -p gpurun_out
VARIANTS="default build/k7m3.so" bash tools/ab.sh; mv gpurun_out/ab.log gpurun_out/ab_plain.log
VARIANTS="default build/k7m3.so" BENCH_ARGS="--workload nerfsynth200k" bash tools/ab.sh; mv gpurun_out/ab.log gpurun_out/ab_nerf.log
