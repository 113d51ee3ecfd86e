#!/bin/bash
mkdir -p gpurun_out
python -m paper_1506_02869_b200.build > gpurun_out/build_v20.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout=300 -o timeout_method=thread -k "dense or fuel or warm or plant" > gpurun_out/pytest_v20.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_v20.log
for g in 3,3,2 4,4,4; do
  timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 --wind-grid $g > gpurun_out/bench_wind_${g//,/x}_v20.log 2>&1
done
echo done
