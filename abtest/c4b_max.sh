#!/bin/bash
mkdir -p gpurun_out
cp abtest/lib_m640.so paper_2311_09275_b200/lib/libising.so
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bench_parity.py -m gpu -q -x -k "sched or grid or torus or fused" > gpurun_out/m640_pytest.log 2>&1; echo "m640 tests rc=$?"; tail -1 gpurun_out/m640_pytest.log
for r in 1 2; do for v in m512 m576 m640; do
  cp abtest/lib_$v.so paper_2311_09275_b200/lib/libising.so
  timeout 300 python bench.py --workload c4b --sweeps 5000 --steps 3 --warmup 2 --no-cpu --no-e2e --no-c5 --no-projection > gpurun_out/abm_$v.log 2>&1
  tail -1 gpurun_out/abm_$v.log | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['value'], d['roofline']['kernel'], d['clocks']['sm_mhz'])" 2>&1 | tail -1
done; done
