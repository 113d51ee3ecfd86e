python -m paper_1506_02869_b200.build > gpurun_out/build_cl2.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_cl2.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_cl2.log
for rep in 1 2 3; do
for sm in cluster lookback; do
  SMC_SCAN=$sm timeout 300 python bench.py --config 2 --steps 3 --warmup 2 --no-cpu-baseline --e2e-steps 0 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$sm', d['ms_per_step'], d['phase_ms_per_step'])" >> gpurun_out/ab_cl2.txt
done
done
SMC_SCAN=cluster timeout 300 python bench.py --config 4 --steps 2 --warmup 2 --no-cpu-baseline --e2e-steps 0 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c4 cluster', d['ms_per_step'], d['phase_ms_per_step'])" >> gpurun_out/ab_cl2.txt
SMC_SCAN=lookback timeout 300 python bench.py --config 4 --steps 2 --warmup 2 --no-cpu-baseline --e2e-steps 0 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c4 lookback', d['ms_per_step'], d['phase_ms_per_step'])" >> gpurun_out/ab_cl2.txt
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cl2.csv python tools/prof_step.py 2 4 > gpurun_out/ncu_cl2.log 2>&1
echo done
