#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x -k "plane_cull or full_image or large_sampled or fisheye or detail or dipole or trace" > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
VARIANTS="build/base.so default" bash tools/ab.sh
