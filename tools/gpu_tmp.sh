python -m paper_1506_02869_b200.build > gpurun_out/build_loop.log 2>&1
for tr in c3 mixed congested; do
  timeout 900 python bench.py --loop 60 --traffic $tr 2>&1 | grep '^{' >> gpurun_out/loop_f2.jsonl
done
timeout 900 python bench.py --loop 60 --traffic mixed --warm 0.25 2>&1 | grep '^{' >> gpurun_out/loop_f2.jsonl
timeout 900 python bench.py --loop 60 --traffic mixed --mh 2 2>&1 | grep '^{' >> gpurun_out/loop_f2.jsonl
echo done
