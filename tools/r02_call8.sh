#!/bin/bash
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -x -k "binning or full_image or large_sampled or fisheye or many_views or multiview or static or sweep or debug or counters" > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
VARIANTS="build/base.so default" bash tools/ab.sh
timeout 900 python bench.py --no-cpu > gpurun_out/bench.json 2> gpurun_out/bench.err
