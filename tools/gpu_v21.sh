#!/bin/bash
# Re-entry validation: microbench FFMA vs FFMA2, parity tests, bench c2.
tag=${1:-v21}; mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ffma2 tools/micro/ffma2.cu && /tmp/ffma2 > gpurun_out/ffma2_$tag.log 2>&1
cuobjdump -sass /tmp/ffma2 | grep -c FFMA2 >> gpurun_out/ffma2_$tag.log
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout=240 -o timeout_method=thread > gpurun_out/pytest_$tag.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_$tag.log
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_$tag.log 2>&1; echo "bench rc $?" >> gpurun_out/bench_$tag.log
echo done
