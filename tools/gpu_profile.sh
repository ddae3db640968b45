#!/bin/bash
# Run on the B200 box (gpurun): bench line, reference arm, ncu launch list and
# full captures of the two blend kernels.  Outputs land in gpurun_out/.
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu \
    > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k7_backward -c 1 \
    -o gpurun_out/prof_k7 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_k7.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k6_forward -c 1 \
    -o gpurun_out/prof_k6 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_k6.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k4_scatter -c 1 \
    -o gpurun_out/prof_k4 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_k4.log 2>&1
nvidia-smi -q -d CLOCK > gpurun_out/smi_clocks.txt 2>&1
lscpu > gpurun_out/lscpu.txt 2>&1
