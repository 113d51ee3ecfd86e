#!/bin/bash
# A/B of build variants on one config (1 repeat each): tools/gpu_ab_cfg.sh tag config "flagsA" "flagsB" ...
tag=$1; cfg=$2; shift 2; mkdir -p gpurun_out; i=0
for fl in "$@"; do
  mkdir -p /tmp/w$i
  SMC_NVCC_FLAGS="$fl" python -m paper_1506_02869_b200.build --force > gpurun_out/build_${tag}_$i.log 2>&1
  cp paper_1506_02869_b200/libsmcatm.so /tmp/w$i/
  i=$((i+1))
done
j=0
for fl in "$@"; do
  cp /tmp/w$j/libsmcatm.so paper_1506_02869_b200/libsmcatm.so
  echo "flags: $fl config $cfg" >> gpurun_out/ab_${tag}.txt
  timeout 600 python bench.py --config $cfg --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['phase_ms_per_step'])" >> gpurun_out/ab_${tag}.txt
  j=$((j+1))
done
echo done
