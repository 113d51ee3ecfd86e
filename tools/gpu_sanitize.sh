#!/bin/bash
# compute-sanitizer racecheck / synccheck / memcheck of small c1 and c2 MPC updates.
tag=${1:-s}; mkdir -p gpurun_out
python -m paper_1506_02869_b200.build > gpurun_out/build_$tag.log 2>&1
for tool in racecheck synccheck memcheck; do
  for cfg in "1 256 4" "2 1024 3"; do
    set -- $cfg
    timeout 1200 compute-sanitizer --tool $tool --error-exitcode 9 python tools/sanitize_step.py $1 $2 $3 \
      > gpurun_out/sanitize_${tool}_c$1_$tag.log 2>&1
    echo "$tool c$1 L=$2 K=$3 rc $?" >> gpurun_out/sanitize_summary_$tag.txt
  done
done
cat gpurun_out/sanitize_summary_$tag.txt
