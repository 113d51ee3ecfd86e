#!/bin/bash
# Full evidence pass: tests, bench, launch list, ncu of K2 / K6 / K4.
tag=${1:-r}; mkdir -p gpurun_out
python -m paper_1506_02869_b200.build > gpurun_out/build_$tag.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout=240 -o timeout_method=thread > gpurun_out/pytest_$tag.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_$tag.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke_$tag.log 2>&1; echo "smoke rc $?" >> gpurun_out/smoke_$tag.log
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi_$tag.txt 2>&1
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_$tag.log 2>&1; echo "bench rc $?" >> gpurun_out/bench_$tag.log
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_$tag.log 2>&1
python bench.py --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_small_$tag.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_$tag.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_launch_$tag.log 2>&1
timeout 120 python tools/prof_step.py 2 4 > gpurun_out/prof_plain_$tag.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_rollout|k_gather|k_scan" -s 2 -c 4 -o gpurun_out/prof_$tag python tools/prof_step.py 2 4 > gpurun_out/ncu_$tag.log 2>&1
echo done
