#!/bin/bash
# A/B timing of library variants (PF_LIBRARY_PATH) on one box, interleaved twice.
# usage: VARIANTS="default build/x.so" BENCH_ARGS="..." bash tools/ab.sh
mkdir -p gpurun_out
: > gpurun_out/ab.log
for rep in 1 2; do
for v in ${VARIANTS:-default}; do
  if [ "$v" = default ]; then unset PF_LIBRARY_PATH; else export PF_LIBRARY_PATH=$PWD/$v; fi
  echo "== $v (rep $rep) $BENCH_ARGS" >> gpurun_out/ab.log
  timeout 600 python bench.py --warmup 3 --steps 10 --no-cpu --no-e2e $BENCH_ARGS 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['fwd_fps'],1), {k:round(v,3) for k,v in d['stage_ms_per_step'].items() if k in ('K1_preprocess','K4_sort','K6_forward','K7_backward')})" >> gpurun_out/ab.log 2>&1
done; done
unset PF_LIBRARY_PATH
