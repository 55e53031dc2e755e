#!/bin/bash
# own-queue stage 2 vs base on the bit-packed workloads (incl. the band-split 8-GPU share)
for rep in 1 2; do for v in head nobar; do
  cp abtest/lib_$v.so paper_2311_09275_b200/lib/libising.so; touch paper_2311_09275_b200/lib/libising.so
  for w in c2 c3; do
    timeout 600 python bench.py --workload $w --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/own.log 2>&1
    tail -1 gpurun_out/own.log | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v $w', '%.4g'%d['value'])"
  done
  timeout 600 python bench.py --workload c4b --copies 16 --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/own.log 2>&1
  tail -1 gpurun_out/own.log | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v share16', '%.4g'%d['value'])"
done; done
cp abtest/lib_nobar.so paper_2311_09275_b200/lib/libising.so; touch paper_2311_09275_b200/lib/libising.so
