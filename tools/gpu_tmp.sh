python -m paper_1506_02869_b200.build > gpurun_out/build_pdl.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_pdl.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_pdl.log
for rep in 1 2 3; do
for pd in 1 0; do
  SMC_PDL=$pd timeout 300 python bench.py --config 2 --steps 3 --warmup 2 --no-cpu-baseline --e2e-steps 0 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('pdl=$pd', d['ms_per_step'], d['phase_ms_per_step'])" >> gpurun_out/ab_pdl.txt
done
done
echo done
