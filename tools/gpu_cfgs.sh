#!/bin/bash
# parity tests + bench lines for c2 (default) and c3/c4/c5
tag=${1:-cf}; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout=240 -o timeout_method=thread > gpurun_out/pytest_$tag.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_$tag.log
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_$tag.log 2>&1; echo "bench rc $?" >> gpurun_out/bench_$tag.log
for c in 3 4 5; do
  timeout 900 python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_${tag}_c$c.log 2>&1
done
echo done
