#!/bin/bash
# Quick iteration: build, selected GPU tests, short bench lines (c2 full K, c5 with 21 rounds).
# Usage: tools/gpu_quick.sh TAG "pytest -k expr" [extra bench configs...]
tag=${1:-q}; kexpr=${2:-}; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$tag.log 2>&1 || { tail -30 gpurun_out/build_$tag.log; exit 1; }
if [ -n "$kexpr" ]; then
  timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout=600 -o timeout_method=thread -k "$kexpr" > gpurun_out/pytest_$tag.log 2>&1
  echo "pytest rc $?" >> gpurun_out/pytest_$tag.log; tail -4 gpurun_out/pytest_$tag.log
fi
timeout 300 python bench.py --config 2 --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 --phase-steps 2 > gpurun_out/bench_c2_$tag.log 2>&1
timeout 600 python bench.py --config 5 --rounds 21 --steps 3 --warmup 1 --no-cpu-baseline --e2e-steps 0 --phase-steps 1 > gpurun_out/bench_c5k21_$tag.log 2>&1
for c in "${@:3}"; do
  timeout 600 python bench.py --config $c --steps 3 --warmup 2 --no-cpu-baseline --e2e-steps 0 --phase-steps 1 > gpurun_out/bench_c${c}_$tag.log 2>&1
done
python - "$tag" <<'PY'
import json, sys, glob
tag = sys.argv[1]
for f in sorted(glob.glob(f"gpurun_out/bench_*_{tag}.log")):
    for line in open(f):
        if line.startswith("{"):
            d = json.loads(line)
            r = d["roofline"]
            print(f, f"{d['ms_per_step']:.2f} ms/step", f"K2 {r['k2_ms_per_step']:.2f} ms", f"frac {r['frac']:.3f} ({r['pipe']})")
PY
