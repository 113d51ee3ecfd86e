#!/bin/bash
tag=${1:-perf}; mkdir -p gpurun_out
python -m paper_1506_02869_b200.build > gpurun_out/build_$tag.log 2>&1
for c in 3 4; do
  for lay in segment transposed; do
    SMC_K2_LAYOUT=$lay timeout 300 python bench.py --config $c --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_${tag}_c${c}_$lay.log 2>&1
  done
done
echo done
