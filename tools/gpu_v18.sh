#!/bin/bash
# v18: parity suite, table-1 layout A/B, closed-loop audits (paper mixed traffic, cold vs warm start)
mkdir -p gpurun_out
python -m paper_1506_02869_b200.build > gpurun_out/build_v18.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout=240 -o timeout_method=thread > gpurun_out/pytest_v18.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_v18.log
SMC_K2_LAYOUT=segment timeout 300 python bench.py --config 6 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_t1seg_v18.log 2>&1
SMC_K2_LAYOUT=transposed timeout 300 python bench.py --config 6 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_t1tr_v18.log 2>&1
timeout 900 python bench.py --loop 100 --traffic mixed > gpurun_out/loop_mixed_cold_v18.log 2>&1
timeout 900 python bench.py --loop 100 --traffic mixed --warm 0.25 > gpurun_out/loop_mixed_warm_v18.log 2>&1
echo done
