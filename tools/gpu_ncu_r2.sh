#!/bin/bash
# ncu evidence (in-tree library, no rebuild): K2 at c5/c2, resample kernels at c5, launch list of
# the default bench command limited to its first 700 launches (pipe micro + one c5 MPC step).
tag=${1:-r2}; mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_rollout -s 2 -c 1 -o gpurun_out/prof_k2c5_$tag python tools/prof_step.py 5 4 > gpurun_out/ncu_k2c5_$tag.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_rollout -s 2 -c 1 -o gpurun_out/prof_k2c2_$tag python tools/prof_step.py 2 4 > gpurun_out/ncu_k2c2_$tag.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:"k_scan|k_gather|k_mp|k_ancestors" -c 4 -o gpurun_out/prof_rsc5_$tag python tools/prof_step.py 5 3 > gpurun_out/ncu_rsc5_$tag.log 2>&1
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 700 --csv --log-file gpurun_out/launches_c5_$tag.csv \
  python bench.py --steps 1 --warmup 1 --phase-steps 1 --no-cpu-baseline --e2e-steps 0 > gpurun_out/ncu_launch_c5_$tag.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_c2_$tag.csv \
  python bench.py --config 2 --steps 1 --warmup 1 --phase-steps 1 --no-cpu-baseline --e2e-steps 0 > gpurun_out/ncu_launch_c2_$tag.log 2>&1
echo done
