python -m paper_1506_02869_b200.build > gpurun_out/build_cs.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_cs.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_cs.log
for rep in 1 2 3; do
for cs in 1 0; do
  SMC_CDF_SAMPLE=$cs timeout 300 python bench.py --config 2 --steps 3 --warmup 2 --no-cpu-baseline --e2e-steps 0 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cs=$cs', d['ms_per_step'], d['phase_ms_per_step'])" >> gpurun_out/ab_cs.txt
done
done
echo done
