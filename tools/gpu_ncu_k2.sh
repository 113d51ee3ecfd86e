#!/bin/bash
# ncu --set full capture of one K2 launch (c2, round 1: both MH candidates), source-attributed.
tag=${1:-k2}; mkdir -p gpurun_out
python -m paper_1506_02869_b200.build > gpurun_out/build_$tag.log 2>&1
python tools/prof_step.py 2 4 > gpurun_out/prof_plain_$tag.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_rollout -s 2 -c 1 -o gpurun_out/prof_k2_$tag python tools/prof_step.py 2 4 > gpurun_out/ncu_k2_$tag.log 2>&1
echo done
