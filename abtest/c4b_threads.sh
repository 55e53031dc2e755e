#!/bin/bash
mkdir -p gpurun_out
for r in 1 2; do for t in 512 480 448 416; do
  timeout 300 python bench.py --workload c4b --threads $t --sweeps 5000 --steps 3 --warmup 2 --no-cpu --no-e2e --no-c5 --no-projection > gpurun_out/abt_$t.log 2>&1
  tail -1 gpurun_out/abt_$t.log | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('$t', d['value'], d['roofline']['kernel'], d['clocks']['sm_mhz'])" 2>&1 | tail -1
done; done
