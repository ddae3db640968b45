#!/bin/bash
mkdir -p gpurun_out
: > gpurun_out/exact.log
for v in build/tcull_base.so build/tcull_u4.so; do
  PF_LIBRARY_PATH=$PWD/$v timeout 900 python -m pytest tests -m gpu -q -x -k "plane_cull" >> gpurun_out/exact.log 2>&1
  echo "$v exit $?" >> gpurun_out/exact.log
done
VARIANTS="build/base.so build/tcull_base.so build/tcull_u4.so" bash tools/ab.sh
