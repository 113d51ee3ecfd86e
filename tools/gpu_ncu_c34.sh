#!/bin/bash
# ncu --set full of one K2 launch (round 2: both MH candidates) at c4 and c3 (packed 12/24-lane segments).
tag=${1:-c34}; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$tag.log 2>&1 || { tail -30 gpurun_out/build_$tag.log; exit 1; }
for c in 4 3; do
  timeout 120 python tools/prof_step.py $c 4 > gpurun_out/prof_plain_c${c}_$tag.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_rollout -s 2 -c 1 -o gpurun_out/prof_k2c${c}_$tag python tools/prof_step.py $c 4 > gpurun_out/ncu_k2c${c}_$tag.log 2>&1
done
echo done
