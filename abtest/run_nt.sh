#!/bin/bash
for nt in 768 800 832 704 768 800; do
  timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu --no-e2e --threads $nt > gpurun_out/ab_nt.log 2>&1
  tail -1 gpurun_out/ab_nt.log | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('nt $nt', d['value'], d['ms_per_step'])"
done
