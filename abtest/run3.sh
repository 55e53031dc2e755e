#!/bin/bash
for spec in "a 1024" "b 768" "c 512" "a 1024" "b 768" "c 512"; do
  set -- $spec
  cp abtest/lib_$1.so paper_2311_09275_b200/lib/libising.so; touch paper_2311_09275_b200/lib/libising.so
  timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu --no-e2e --threads $2 > gpurun_out/ab_$1.log 2>&1
  echo "$1 rc=$?"; tail -1 gpurun_out/ab_$1.log | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', d['value'], d['ms_per_step'])"
done
