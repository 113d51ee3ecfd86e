#!/bin/bash
# ncu --set full of one K2 launch (round 2, both candidates) for the given configs, no rebuild
# (uses the in-tree libsmcatm.so).  Usage: tools/gpu_ncu_k2only.sh TAG CFG...
tag=$1; shift; mkdir -p gpurun_out
for c in "$@"; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_rollout -s 2 -c 1 \
    -o gpurun_out/prof_k2c${c}_$tag python tools/prof_step.py $c 4 > gpurun_out/ncu_k2c${c}_$tag.log 2>&1
done
echo done
