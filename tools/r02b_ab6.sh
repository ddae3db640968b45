#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x -k "detail or fisheye or cull" > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
python tools/bitcmp.py dump q1 nerfsynth200k 8 2 > gpurun_out/bitcmp.log 2>&1
PF_LIBRARY_PATH=$PWD/build/q0.so python tools/bitcmp.py dump q0 nerfsynth200k 8 2 >> gpurun_out/bitcmp.log 2>&1
python tools/bitcmp.py cmp q1 q0 >> gpurun_out/bitcmp.log 2>&1
VARIANTS="default build/q0.so" BENCH_ARGS="--workload nerfsynth200k --detail 8" bash tools/ab.sh; mv gpurun_out/ab.log gpurun_out/ab_nerf_detail.log
VARIANTS="default build/q0.so" BENCH_ARGS="--detail 8" bash tools/ab.sh; mv gpurun_out/ab.log gpurun_out/ab_train_detail.log
