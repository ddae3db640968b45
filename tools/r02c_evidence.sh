#!/bin/bash
# Late round-2 evidence after the tracked-clip changes: GPU suite + smoke with the
# in-tree library, the bench lines whose K6 changed, the launch list and K6/K7 captures
mkdir -p gpurun_out/bench
rm -rf gpurun_out/prof_*.ncu-rep gpurun_out/launches.csv gpurun_out/export
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_final.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu_final.log
timeout 600 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1
echo "smoke exit $?" >> gpurun_out/smoke.log
B=gpurun_out/bench
timeout 900 python bench.py > $B/bench_train8_1m.json 2> $B/bench_train8_1m.err
timeout 900 python bench.py --dipoles --no-cpu > $B/bench_train8_1m_dipoles.json 2>&1
timeout 900 python bench.py --workload mip360_1m --no-cpu > $B/bench_mip360_1m.json 2>&1
timeout 900 python bench.py --workload nerfsynth200k --no-cpu > $B/bench_nerfsynth200k.json 2>&1
timeout 900 python bench.py --workload nerfsynth200k --detail 8 --no-cpu > $B/bench_nerfsynth200k_detail8.json 2>&1
timeout 900 python bench.py --fisheye --no-cpu > $B/bench_train8_1m_fisheye.json 2>&1
timeout 900 python bench.py --lists knn --no-cpu > $B/bench_train8_1m_knn.json 2>&1
timeout 900 python bench.py --detail 8 --no-cpu --steps 5 > $B/bench_train8_1m_detail8.json 2>&1
timeout 1500 python bench.py --workload sweep64_3m --no-cpu --no-e2e --steps 3 > $B/bench_sweep64_3m.json 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu \
    > gpurun_out/ncu_launch.log 2>&1
NCU="timeout 900 ncu --set full --import-source on --clock-control none"
$NCU -k regex:k6_forward -c 1 -o "gpurun_out/prof_k6_forward@train8_1m" python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_k6.log 2>&1
$NCU -k regex:k7_backward -c 1 -o "gpurun_out/prof_k7_backward@train8_1m" python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_k7.log 2>&1
nvidia-smi -q -d CLOCK > gpurun_out/smi_clocks.txt 2>&1
mkdir -p gpurun_out/export
python tools/ncu_export.py r02c gpurun_out gpurun_out/export > gpurun_out/export/export.log 2>&1
for r in gpurun_out/prof_*.ncu-rep; do
  b=$(basename "$r" .ncu-rep)
  python tools/ncu_cuda_lines.py "$r" 60 > "gpurun_out/export/${b}_lines.txt" 2>&1
done
rm -f gpurun_out/prof_*.ncu-rep
