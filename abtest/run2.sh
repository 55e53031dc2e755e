#!/bin/bash
for v in a b a b; do
  cp abtest/lib_$v.so paper_2311_09275_b200/lib/libising.so; touch paper_2311_09275_b200/lib/libising.so
  for w in c2 c3; do
    timeout 600 python bench.py --workload $w --steps 3 --warmup 2 --no-cpu --no-e2e > gpurun_out/ab_$v.log 2>&1
    tail -1 gpurun_out/ab_$v.log | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v $w', d['value'], d['ms_per_step'])"
  done
done
