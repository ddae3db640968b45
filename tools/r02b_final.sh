#!/bin/bash
# final verification: full GPU suite, smoke, sanitizer tiers, default bench
mkdir -p gpurun_out/sanitizer
rm -f gpurun_out/sanitizer/summary.txt
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_full.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu_full.log
timeout 600 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1
echo "exit $?" >> gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench_default.json 2>&1
bash tools/sanitize.sh
