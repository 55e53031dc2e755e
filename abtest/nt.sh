#!/bin/bash
# CTA-size sweep of one workload: NTS="640 768" W=c2 bash abtest/nt.sh
for nt in ${NTS:-768 800}; do
  timeout 600 python bench.py --workload ${W:-c2} --steps 3 --warmup 3 --no-cpu --no-e2e --threads $nt > gpurun_out/nt.log 2>&1
  tail -1 gpurun_out/nt.log | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('${W:-c2} nt $nt', '%.4g'%d['value'], '%.2f'%d['ms_per_step'])" 2>&1 | tail -1
done
