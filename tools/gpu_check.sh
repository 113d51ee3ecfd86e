#!/bin/bash
# Run on the GPU box: parity tests, bench, K2 ncu capture.  Usage: tools/gpu_check.sh [tag] [ncu]
tag=${1:-run}; mkdir -p gpurun_out
python -m paper_1506_02869_b200.build > gpurun_out/build_$tag.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout=240 -o timeout_method=thread > gpurun_out/pytest_$tag.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_$tag.log
timeout 600 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_$tag.log 2>&1; echo "bench rc $?" >> gpurun_out/bench_$tag.log
if [ "$2" == "ncu" ]; then
  python tools/prof_step.py 2 4 > gpurun_out/prof_plain_$tag.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_rollout -s 2 -c 1 -o gpurun_out/prof_k2_$tag python tools/prof_step.py 2 4 > gpurun_out/ncu_k2_$tag.log 2>&1
fi
echo done
if [ "$3" == "launches" ]; then
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_small_$tag.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 5000 --csv --log-file gpurun_out/launches_$tag.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_launch_$tag.log 2>&1
fi
