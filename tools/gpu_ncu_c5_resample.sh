#!/bin/bash
# ncu --set full of the resampling kernels (K4 scan, K6 gather/propose) at c5 (L = 2^20, N = 16).
tag=${1:-c5r}; mkdir -p gpurun_out
python -m paper_1506_02869_b200.build > gpurun_out/build_$tag.log 2>&1
timeout 300 python tools/prof_step.py 5 3 > gpurun_out/prof_plain_$tag.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$tag.csv python tools/prof_step.py 5 3 > gpurun_out/ncu_launch_$tag.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_scan|k_gather|k_anc" -c 3 -o gpurun_out/prof_$tag python tools/prof_step.py 5 3 > gpurun_out/ncu_$tag.log 2>&1
echo done
