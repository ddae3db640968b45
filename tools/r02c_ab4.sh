#!/bin/bash
# recording K6: plane-cull threshold (cells with fewer list planes clip by all) 6 / 3 / 0
mkdir -p gpurun_out
VARIANTS="build/cm6.so build/cm3.so build/cm0.so" bash tools/ab.sh; mv gpurun_out/ab.log gpurun_out/ab_cm.log
for v in cm3 cm0; do
PF_LIBRARY_PATH=$PWD/build/$v.so timeout 600 python -m pytest tests -m gpu -q -x -k "cull or image or grad or record" > gpurun_out/pytest_gpu_$v.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu_$v.log
done
