#!/bin/bash
# Resampling-side changes: GPU parity (all), then c2 / c5 bench lines.
tag=${1:-rs}; mkdir -p gpurun_out
python -m paper_1506_02869_b200.build > gpurun_out/build_$tag.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_$tag.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_$tag.log
timeout 300 python bench.py --config 2 --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_c2_$tag.log 2>&1
grep '^{' gpurun_out/bench_c2_$tag.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c2', d['ms_per_step'], d['phase_ms_per_step'], d['roofline_resample'])" >> gpurun_out/summary_$tag.txt
timeout 600 python bench.py --config 5 --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_c5_$tag.log 2>&1
grep '^{' gpurun_out/bench_c5_$tag.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c5', d['ms_per_step'], d['phase_ms_per_step'], d['roofline_resample'])" >> gpurun_out/summary_$tag.txt
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c5_$tag.csv python tools/prof_step.py 5 3 > gpurun_out/ncu_launch_$tag.log 2>&1
echo done
