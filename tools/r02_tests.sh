#!/bin/bash
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -rA -s -k "${PYTEST_K:-}" > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
[ -n "$SANITIZE" ] && bash tools/sanitize.sh
true
