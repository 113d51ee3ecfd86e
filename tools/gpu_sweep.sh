#!/bin/bash
# Bench sweep for profiles/: other configs, variants (N1-N4), closed-loop audits.
tag=${1:-sweep}; mkdir -p gpurun_out
python -m paper_1506_02869_b200.build > gpurun_out/build_$tag.log 2>&1
B="timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0"
{
for c in 3 4 5 6; do $B --config $c; done
$B --wind-grid 3,3,2; $B --wind-grid 4,4,4
$B --mh 2; $B --mh 0; $B --lfinal 4096
} > gpurun_out/bench_$tag.jsonl 2> gpurun_out/bench_${tag}_err.log
{
timeout 900 python bench.py --loop 100 --traffic mixed
timeout 900 python bench.py --loop 100 --traffic mixed --mh 2
timeout 900 python bench.py --loop 100 --traffic mixed --warm 0.05
timeout 900 python bench.py --loop 100 --traffic congested
} > gpurun_out/loop_$tag.jsonl 2> gpurun_out/loop_${tag}_err.log
echo done
