#!/bin/bash
# stage-2 queue limit per warp (words per 8 passes; w0 = one 32-lane round per 8 passes, the default)
for rep in 1 2; do for v in w0 w26 w29 w36; do
  cp abtest/lib_$v.so paper_2311_09275_b200/lib/libising.so; touch paper_2311_09275_b200/lib/libising.so
  for w in c2 c4b; do
    timeout 600 python bench.py --workload $w --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/wl.log 2>&1
    tail -1 gpurun_out/wl.log | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v $w', '%.4g'%d['value'])"
  done
done; done
cp abtest/lib_w0.so paper_2311_09275_b200/lib/libising.so; touch paper_2311_09275_b200/lib/libising.so
