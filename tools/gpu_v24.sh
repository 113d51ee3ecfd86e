#!/bin/bash
tag=${1:-v24}; mkdir -p gpurun_out
python tools/prof_overhead.py 2 5 > gpurun_out/overhead_$tag.log 2>&1
bash tools/gpu_ncu_k2.sh $tag
