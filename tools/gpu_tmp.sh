python -m paper_1506_02869_b200.build > gpurun_out/build_ring.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_ring.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_ring.log
for c in 2 3 4; do
  timeout 900 python bench.py --config $c --steps 2 --warmup 2 --no-cpu-baseline --e2e-steps 0 2>&1 | grep '^{' >> gpurun_out/bench_ring.jsonl
done
echo done
