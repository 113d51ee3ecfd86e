#!/bin/bash
# Perf sweep on the GPU box: both K2 layouts on c2-c4, c5 default; K2 ncu captures for c2.
tag=${1:-perf}; mkdir -p gpurun_out
python -m paper_1506_02869_b200.build > gpurun_out/build_$tag.log 2>&1
for c in 2 3 4; do
  for lay in segment transposed; do
    SMC_K2_LAYOUT=$lay timeout 300 python bench.py --config $c --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_${tag}_c${c}_$lay.log 2>&1
  done
done
timeout 400 python bench.py --config 5 --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_${tag}_c5.log 2>&1
if [ "$2" == "ncu" ]; then
  for lay in segment transposed; do
    SMC_K2_LAYOUT=$lay timeout 120 python tools/prof_step.py 2 4 > gpurun_out/prof_plain_${tag}_$lay.log 2>&1 && \
    SMC_K2_LAYOUT=$lay timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_rollout -s 2 -c 1 -o gpurun_out/prof_k2_${tag}_$lay python tools/prof_step.py 2 4 > gpurun_out/ncu_k2_${tag}_$lay.log 2>&1
  done
fi
echo done
