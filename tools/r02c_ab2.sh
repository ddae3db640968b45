#!/bin/bash
# tracked plane clip: predicated moves (pp1) vs min/max (pp0, HEAD)
mkdir -p gpurun_out
PF_LIBRARY_PATH=$PWD/build/pp1.so timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_pp1.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu_pp1.log
VARIANTS="build/pp0.so build/pp1.so" bash tools/ab.sh; mv gpurun_out/ab.log gpurun_out/ab_pp.log
VARIANTS="build/pp0.so build/pp1.so" BENCH_ARGS="--dipoles" bash tools/ab.sh; mv gpurun_out/ab.log gpurun_out/ab_pp_dip.log
VARIANTS="build/pp0.so build/pp1.so" BENCH_ARGS="--workload nerfsynth200k" bash tools/ab.sh; mv gpurun_out/ab.log gpurun_out/ab_pp_ns.log
