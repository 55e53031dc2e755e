#!/bin/bash
# A/B of packed-row C5 variants (abtest/lib_<name>.so), alternating
mkdir -p gpurun_out
for r in 1 2; do for v in "$@"; do
  cp abtest/lib_$v.so paper_2311_09275_b200/lib/libising.so
  timeout 300 python bench.py --workload c5 --steps 3 --warmup 2 --no-cpu --no-e2e > gpurun_out/abpk_$v.log 2>&1
  tail -1 gpurun_out/abpk_$v.log | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['value'], d['clocks']['sm_mhz'], d['clocks']['reasons'])" 2>&1 | tail -1
done; done
