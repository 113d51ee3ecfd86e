#!/bin/bash
# ncu --set full capture of one launch of kernels matching $2 (c2 workload, round >= 1).
tag=${1:-k}; rx=${2:-k_gather}; skip=${3:-2}; mkdir -p gpurun_out
python tools/prof_step.py 2 4 > gpurun_out/prof_plain_$tag.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$rx" -s $skip -c 1 -o gpurun_out/prof_$tag python tools/prof_step.py 2 4 > gpurun_out/ncu_$tag.log 2>&1
echo done
