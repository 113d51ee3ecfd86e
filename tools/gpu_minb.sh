#!/bin/bash
# Register budget per K2 instance: single-candidate (MINB1), two-candidate (MINB), 32-lane (MINB32)
tag=${1:-minb}; mkdir -p gpurun_out
for v in "4 4 4" "5 4 4" "6 4 4" "4 5 4" "4 4 5" "4 4 3"; do
  set -- $v
  SMC_NVCC_FLAGS="-DSMC_K2_MINB1=$1 -DSMC_K2_MINB=$2 -DSMC_K2_MINB32=$3" python -m paper_1506_02869_b200.build --force > gpurun_out/build_${tag}.log 2>&1
  for c in 6 2 4 3; do
    timeout 600 python bench.py --config $c --steps 2 --warmup 2 --no-cpu-baseline --e2e-steps 0 2>&1 | grep '^{' | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'minb1': $1, 'minb': $2, 'minb32': $3, 'config': d['config']['workload'][:24], 'ms_per_step': round(d['ms_per_step'],3), 'k2_ms': round(d['phase_ms_per_step']['rollout'],3)}))" >> gpurun_out/minb_$tag.jsonl
  done
done
python -m paper_1506_02869_b200.build --force > /dev/null 2>&1
echo done
