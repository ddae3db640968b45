#!/bin/bash
mkdir -p gpurun_out
for w in train8_1m mip360_1m nerfsynth200k; do
  timeout 600 python bench.py --workload $w --no-cpu --steps 10 > gpurun_out/e2e_$w.json 2>&1
done
