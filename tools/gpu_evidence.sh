#!/bin/bash
# Round evidence on one GPU: build, pipe micro, bench (default c5) + reference arm, launch list,
# ncu --set full of K2 at c5 and c2 (round 2: both MH candidates).  Usage: tools/gpu_evidence.sh TAG [STEPS]
tag=${1:-e}; steps=${2:-3}; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$tag.log 2>&1 || { echo "build failed"; exit 1; }
timeout 1200 python bench.py --steps $steps --warmup 2 > gpurun_out/bench_$tag.log 2>&1; echo "bench rc $?" >> gpurun_out/bench_$tag.log
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_$tag.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches_$tag.csv \
  python bench.py --steps 1 --warmup 1 --phase-steps 1 --no-cpu-baseline --e2e-steps 0 > gpurun_out/ncu_launch_$tag.log 2>&1
timeout 120 python tools/prof_step.py 5 4 > gpurun_out/prof_plain_$tag.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_rollout -s 2 -c 1 -o gpurun_out/prof_k2c5_$tag python tools/prof_step.py 5 4 > gpurun_out/ncu_k2c5_$tag.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_rollout -s 2 -c 1 -o gpurun_out/prof_k2c2_$tag python tools/prof_step.py 2 4 > gpurun_out/ncu_k2c2_$tag.log 2>&1
echo done
