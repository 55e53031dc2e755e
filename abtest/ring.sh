#!/bin/bash
# int8-row C5 kernel variants: ring parity tests on the first, then alternating A/B (ISING_I8_PACKED=0)
mkdir -p gpurun_out
v=$1
cp abtest/lib_$v.so paper_2311_09275_b200/lib/libising.so
ISING_I8_PACKED=0 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "float or c5" > gpurun_out/rt_$v.log 2>&1; echo "rc=$?" >> gpurun_out/rt_$v.log
tail -2 gpurun_out/rt_$v.log
for r in 1 2; do for v in "$@"; do
  cp abtest/lib_$v.so paper_2311_09275_b200/lib/libising.so
  ISING_I8_PACKED=0 timeout 300 python bench.py --workload c5 --steps 3 --warmup 2 --no-cpu --no-e2e > gpurun_out/abr_$v.log 2>&1
  tail -1 gpurun_out/abr_$v.log | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['value'], d['roofline']['frac'], d['clocks']['sm_mhz'], d['clocks']['reasons'])" 2>&1 | tail -1
done; done
