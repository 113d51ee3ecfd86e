#!/bin/bash
# K5 merge-path ancestors: parity tests, then c2 / c5 bench lines with each ancestor mode.
tag=${1:-anc}; mkdir -p gpurun_out
python -m paper_1506_02869_b200.build > gpurun_out/build_$tag.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "resample or shrinking or full_size or virtual or replay" > gpurun_out/pytest_$tag.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_$tag.log
for m in mp bisect; do
  SMC_ANC=$m timeout 300 python bench.py --config 2 --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_c2_${m}_$tag.log 2>&1
  grep '^{' gpurun_out/bench_c2_${m}_$tag.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$m c2', d['ms_per_step'], d['phase_ms_per_step'], d['roofline_resample'])" >> gpurun_out/summary_$tag.txt
  SMC_ANC=$m timeout 600 python bench.py --config 5 --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_c5_${m}_$tag.log 2>&1
  grep '^{' gpurun_out/bench_c5_${m}_$tag.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$m c5', d['ms_per_step'], d['phase_ms_per_step'], d['roofline_resample'])" >> gpurun_out/summary_$tag.txt
done
echo done
