#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x -k "cech or trace or connect" > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
for v in build/base.so default; do
  if [ "$v" = default ]; then unset PF_LIBRARY_PATH; else export PF_LIBRARY_PATH=$PWD/$v; fi
  echo "== $v" >> gpurun_out/trace_ab.log
  timeout 900 python bench.py --workload mip360_1m --trace --no-cpu --no-e2e --steps 3 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],2), d['trace']['cells_per_ray'], d['trace']['locates_per_ray'], d['cech_graph'])" >> gpurun_out/trace_ab.log 2>&1
done
unset PF_LIBRARY_PATH
VARIANTS="default build/k7smem.so" bash tools/ab.sh
