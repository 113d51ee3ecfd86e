#!/bin/bash
# GPU parity tests + smoke only.  Usage: tools/gpu_tests.sh TAG [pytest -k expr]
tag=${1:-t}; mkdir -p gpurun_out
python -m paper_1506_02869_b200.build > gpurun_out/build_$tag.log 2>&1
if [ -n "$2" ]; then K=(-k "$2"); else K=(); fi
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout=300 -o timeout_method=thread "${K[@]}" > gpurun_out/pytest_$tag.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_$tag.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke_$tag.log 2>&1; echo "smoke rc $?" >> gpurun_out/smoke_$tag.log
tail -5 gpurun_out/pytest_$tag.log
