#!/bin/bash
# A/B of build variants on c2: tools/gpu_ab.sh tag "flagsA" "flagsB" ...
tag=$1; shift; mkdir -p gpurun_out; i=0
for fl in "$@"; do
  SMC_NVCC_FLAGS="$fl" python -m paper_1506_02869_b200.build --force > gpurun_out/build_${tag}_$i.log 2>&1
  echo "flags: $fl" > gpurun_out/bench_${tag}_$i.log
  timeout 300 python bench.py --config 2 --steps 3 --warmup 2 --no-cpu-baseline --e2e-steps 0 >> gpurun_out/bench_${tag}_$i.log 2>&1
  i=$((i+1))
done
python -m paper_1506_02869_b200.build --force > /dev/null 2>&1
echo done
