#!/bin/bash
# Round-2 evidence: build, tests + smoke, default bench (c5) + reference arm, other configs,
# closed loops, launch list, ncu --set full of K2 (c5, c2) and K4/K6 (c5).  Usage: tools/gpu_round2.sh TAG
tag=${1:-r2}; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$tag.log 2>&1 || { tail -30 gpurun_out/build_$tag.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout=600 -o timeout_method=thread > gpurun_out/pytest_$tag.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_$tag.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke_$tag.log 2>&1; echo "smoke rc $?" >> gpurun_out/smoke_$tag.log
timeout 1500 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_c5_$tag.log 2>&1; echo "rc $?" >> gpurun_out/bench_c5_$tag.log
timeout 300 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref_$tag.log 2>&1
for c in 2 3 4 6 7; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c${c}_$tag.log 2>&1
done
for tr in c3 mixed congested; do
  timeout 900 python bench.py --loop 60 --traffic $tr > gpurun_out/loop_${tr}_$tag.log 2>&1
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2500 --csv --log-file gpurun_out/launches_c5_$tag.csv \
  python bench.py --steps 1 --warmup 1 --phase-steps 1 --no-cpu-baseline --e2e-steps 0 > gpurun_out/ncu_launch_c5_$tag.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_rollout -s 2 -c 1 -o gpurun_out/prof_k2c5_$tag python tools/prof_step.py 5 4 > gpurun_out/ncu_k2c5_$tag.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_rollout -s 2 -c 1 -o gpurun_out/prof_k2c2_$tag python tools/prof_step.py 2 4 > gpurun_out/ncu_k2c2_$tag.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:"k_scan|k_gather|k_mp|k_ancestors" -c 4 -o gpurun_out/prof_rsc5_$tag python tools/prof_step.py 5 3 > gpurun_out/ncu_rsc5_$tag.log 2>&1
# keep the merged output under gpurun's 64 MiB: metrics of every capture as JSON, only the c5 K2 report kept
for r in prof_k2c2_$tag prof_rsc5_$tag prof_k2c5_$tag; do
  [ -f gpurun_out/$r.ncu-rep ] && python tools/ncu_full_json.py gpurun_out/$r.ncu-rep > gpurun_out/$r.json
done
rm -f gpurun_out/prof_k2c2_$tag.ncu-rep gpurun_out/prof_rsc5_$tag.ncu-rep
echo done
