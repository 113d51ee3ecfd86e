#!/bin/bash
# Round-end evidence pass without the long ncu --set full captures: tests, smoke, bench lines, launch list, K6 ncu.
tag=${1:-fin}; mkdir -p gpurun_out
python -m paper_1506_02869_b200.build > gpurun_out/build_$tag.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout=240 -o timeout_method=thread > gpurun_out/pytest_$tag.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_$tag.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke_$tag.log 2>&1; echo "smoke rc $?" >> gpurun_out/smoke_$tag.log
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_$tag.log 2>&1; echo "bench rc $?" >> gpurun_out/bench_$tag.log
for c in 3 4 5 6 7; do
  timeout 900 python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_${tag}_c$c.log 2>&1
done
python bench.py --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_small_$tag.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_$tag.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_launch_$tag.log 2>&1
timeout 120 python tools/prof_step.py 2 4 > gpurun_out/prof_plain_$tag.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_gather" -s 2 -c 1 -o gpurun_out/prof_k6_$tag python tools/prof_step.py 2 4 > gpurun_out/ncu_k6_$tag.log 2>&1
echo done
