python -m paper_1506_02869_b200.build > gpurun_out/build_dn4.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "dense" > gpurun_out/pytest_dn4.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_dn4.log
for g in 3,3,2 4,4,4; do
  timeout 600 python bench.py --config 2 --steps 2 --warmup 2 --no-cpu-baseline --e2e-steps 0 --wind-grid $g 2>&1 | grep '^{' >> gpurun_out/bench_dn4.jsonl
done
echo done
