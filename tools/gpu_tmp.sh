python -m paper_1506_02869_b200.build > gpurun_out/build_ch.log 2>&1
for rep in 1 2; do
for ch in 0 1; do
  SMC_K2_CHUNKS=$ch timeout 300 python bench.py --config 2 --steps 3 --warmup 2 --no-cpu-baseline --e2e-steps 0 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('chunks=$ch', d['ms_per_step'], d['phase_ms_per_step'])" >> gpurun_out/ab_ch.txt
  SMC_K2_CHUNKS=$ch timeout 300 python bench.py --config 4 --steps 2 --warmup 2 --no-cpu-baseline --e2e-steps 0 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c4 chunks=$ch', d['ms_per_step'], d['phase_ms_per_step'])" >> gpurun_out/ab_ch.txt
done
done
echo done
