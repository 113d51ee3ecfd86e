#!/bin/bash
mkdir -p gpurun_out
python -m paper_1506_02869_b200.build > gpurun_out/build_v19.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout=300 -o timeout_method=thread > gpurun_out/pytest_v19.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_v19.log
for g in 2,2,2 3,3,2 4,4,2 4,4,4; do
  timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 --wind-grid $g > gpurun_out/bench_wind_${g//,/x}_v19.log 2>&1
done
timeout 300 python bench.py --config 6 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_t1_v19.log 2>&1
echo done
