#!/bin/bash
# A/B of prebuilt library variants (build/variants/<name>/libsmcatm.so, built here with
# SMC_NVCC_FLAGS / SMC_LIB_OUT): production-round parity of each variant, then interleaved
# repeats of c2 (K = 101), c5 (21 rounds) and c4 (K = 101).
# Usage: tools/gpu_variants.sh TAG REPS name1 name2 ...   (CFGS="c k steps warmup;..." overrides the configs)
tag=$1; reps=$2; shift 2; mkdir -p gpurun_out; out=gpurun_out/variants_$tag.txt
for v in "$@"; do
  SMC_LIB=$PWD/build/variants/$v/libsmcatm.so timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider \
    -k "production_rounds or evaluate_parity" > gpurun_out/pytest_${tag}_$v.log 2>&1
  echo "$v parity: $(tail -1 gpurun_out/pytest_${tag}_$v.log)" >> $out
done
for rep in $(seq 1 $reps); do
  for v in "$@"; do
    IFS=';' read -ra cfgs <<< "${CFGS:-2 0 3 2;5 21 2 1;4 0 3 2}"
    for cfg in "${cfgs[@]}"; do
      read c k st wu <<< "$cfg"
      line=$(SMC_LIB=$PWD/build/variants/$v/libsmcatm.so timeout 600 python bench.py --config $c --rounds $k --steps $st --warmup $wu \
             --no-cpu-baseline --e2e-steps 0 --phase-steps 1 2>&1 | grep '^{')
      echo "$line" | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$v', 'c$c', 'rep $rep', round(d['ms_per_step'],3), 'K2', round(r['k2_ms_per_step'],3), 'frac', round(r['frac'],4))" >> $out 2>&1
    done
  done
done
cat $out
