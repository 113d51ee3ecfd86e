#!/bin/bash
# Pipe microbenchmarks (tools/micro/pipes.cu) + their SASS instruction counts.
tag=${1:-m}; mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gpurun_out/pipes tools/micro/pipes.cu > gpurun_out/micro_build_$tag.log 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv > gpurun_out/micro_smi_$tag.txt
./gpurun_out/pipes > gpurun_out/micro_$tag.jsonl 2>&1; echo "rc $?" >> gpurun_out/micro_$tag.jsonl
./gpurun_out/pipes > gpurun_out/micro2_$tag.jsonl 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv >> gpurun_out/micro_smi_$tag.txt
rm -f gpurun_out/pipes
