#!/bin/bash
# A/B of build variants on c2 (3 repeats each, interleaved): tools/gpu_ab2.sh tag "flagsA" "flagsB" ...
tag=$1; shift; mkdir -p gpurun_out; i=0
for fl in "$@"; do
  mkdir -p /tmp/v$i
  SMC_NVCC_FLAGS="$fl" python -m paper_1506_02869_b200.build --force > gpurun_out/build_${tag}_$i.log 2>&1
  cp paper_1506_02869_b200/libsmcatm.so /tmp/v$i/
  i=$((i+1))
done
for rep in 1 2 3; do
  j=0
  for fl in "$@"; do
    cp /tmp/v$j/libsmcatm.so paper_1506_02869_b200/libsmcatm.so
    echo "flags: $fl rep $rep" >> gpurun_out/ab_${tag}.txt
    timeout 300 python bench.py --config 2 --steps 3 --warmup 2 --no-cpu-baseline --e2e-steps 0 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['phase_ms_per_step'])" >> gpurun_out/ab_${tag}.txt
    j=$((j+1))
  done
done
echo done
