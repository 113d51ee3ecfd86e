#!/bin/bash
# closed-loop audits (c3's solver) for the three traffic streams, plus the variants of N2
tag=${1:-l}; mkdir -p gpurun_out
for tr in c3 mixed congested; do
  timeout 900 python bench.py --loop 60 --traffic $tr > gpurun_out/loop_${tr}_$tag.log 2>&1
done
timeout 900 python bench.py --loop 60 --traffic mixed --mh 2 > gpurun_out/loop_mixed_mh2_$tag.log 2>&1
timeout 900 python bench.py --loop 60 --traffic mixed --warm 0.25 > gpurun_out/loop_mixed_warm_$tag.log 2>&1
grep -h '^{' gpurun_out/loop_*_$tag.log > gpurun_out/loops_$tag.jsonl
echo done
