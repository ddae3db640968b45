#!/bin/bash
# K6 detail: warp-spread soft-Voronoi of the chart (bit-exactness + A/B)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x -k "detail or fisheye or cull" > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
: > gpurun_out/bitcmp.log
for pre in "nerfsynth200k 8 2" "small360 8 4" "small 3 2"; do
  set -- $pre
  PF_LIBRARY_PATH=$PWD/build/ws1.so python tools/bitcmp.py dump w1 $1 $2 $3 >> gpurun_out/bitcmp.log 2>&1
  PF_LIBRARY_PATH=$PWD/build/ws0.so python tools/bitcmp.py dump w0 $1 $2 $3 >> gpurun_out/bitcmp.log 2>&1
  echo "$pre: $(python tools/bitcmp.py cmp w1 w0)" >> gpurun_out/bitcmp.log 2>&1
done
rm -f gpurun_out/bitcmp_*.npy
VARIANTS="build/ws0.so build/ws1.so" BENCH_ARGS="--workload nerfsynth200k --detail 8" bash tools/ab.sh; mv gpurun_out/ab.log gpurun_out/ab_nerf_detail_ws.log
VARIANTS="build/ws0.so build/ws1.so" BENCH_ARGS="--detail 8" bash tools/ab.sh; mv gpurun_out/ab.log gpurun_out/ab_train_detail_ws.log
