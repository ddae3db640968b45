#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -k "per_view or detail_colour or queue" > gpurun_out/pytest_gpu_pv.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu_pv.log
