#!/bin/bash
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
: > gpurun_out/ab13.log
for rep in 1 2; do
for v in base fused perview; do
  unset PF_LIBRARY_PATH PF_K6_PER_VIEW
  [ $v = base ] && export PF_LIBRARY_PATH=$PWD/build/base.so
  [ $v = perview ] && export PF_K6_PER_VIEW=1
  echo "== $v" >> gpurun_out/ab13.log
  timeout 600 python bench.py --warmup 3 --steps 10 --no-cpu --no-e2e 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['fwd_fps'],1), {k:round(v,3) for k,v in d['stage_ms_per_step'].items() if k in ('K4_sort','K6_forward','K7_backward')})" >> gpurun_out/ab13.log 2>&1
done; done
unset PF_LIBRARY_PATH PF_K6_PER_VIEW
for v in build/trace_thread.so default; do
  if [ "$v" = default ]; then unset PF_LIBRARY_PATH; else export PF_LIBRARY_PATH=$PWD/$v; fi
  echo "== trace $v" >> gpurun_out/ab13.log
  timeout 900 python bench.py --workload mip360_1m --trace --no-cpu --no-e2e --steps 3 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],2), d['trace']['cells_per_ray'], d['trace']['locates_per_ray'])" >> gpurun_out/ab13.log 2>&1
done
