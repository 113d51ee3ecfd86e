#!/bin/bash
# A/B of prebuilt library variants (build/variants/<name>/libsmcatm.so, built here with
# SMC_NVCC_FLAGS / SMC_LIB_OUT): interleaved repeats of c2 (K = 101) and c5 (21 rounds).
# Usage: tools/gpu_variants.sh TAG REPS name1 name2 ...
tag=$1; reps=$2; shift 2; mkdir -p gpurun_out; out=gpurun_out/variants_$tag.txt
for rep in $(seq 1 $reps); do
  for v in "$@"; do
    for cfg in "2 0 3 2" "5 21 2 1"; do
      read c k st wu <<< "$cfg"
      line=$(SMC_LIB=$PWD/build/variants/$v/libsmcatm.so timeout 600 python bench.py --config $c --rounds $k --steps $st --warmup $wu \
             --no-cpu-baseline --e2e-steps 0 --phase-steps 1 2>&1 | grep '^{')
      echo "$line" | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$v', 'c$c', 'rep $rep', round(d['ms_per_step'],3), 'K2', round(r['k2_ms_per_step'],3), 'frac', round(r['frac'],4))" >> $out 2>&1
    done

  done
done
cat $out
