#!/bin/bash
# Launch-geometry sweep of K2 (N3; cf. the paper's Table 1): threads per block x
# resident blocks per SM, on the Table-1 workload (--config 6) and c2.  Rebuilds per variant.
tag=${1:-geo}; mkdir -p gpurun_out
for v in "64 8" "128 4" "256 2" "512 1" "128 3" "128 5" "64 10" "256 1"; do
  set -- $v
  SMC_NVCC_FLAGS="-DSMC_K2_BLOCK=$1 -DSMC_K2_MINB=$2" python -m paper_1506_02869_b200.build --force > gpurun_out/build_${tag}_$1_$2.log 2>&1
  for c in 6 2; do
    timeout 600 python bench.py --config $c --steps 3 --warmup 2 --no-cpu-baseline --e2e-steps 0 2>&1 | grep '^{' | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'block': $1, 'min_blocks_per_sm': $2, 'config': d['config']['workload'][:60], 'ms_per_step': d['ms_per_step'], 'k2_ms_per_step': d['phase_ms_per_step']['rollout'], 'roofline_frac': d['roofline']['frac']}))" >> gpurun_out/geometry_$tag.jsonl
  done
done
python -m paper_1506_02869_b200.build --force > /dev/null 2>&1
echo done
