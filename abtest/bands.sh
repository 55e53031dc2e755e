#!/bin/bash
# band-split kernel: parity tests (every torus test with 2 bands, the C4b 8-GPU share), then A/B of the 8-GPU share
mkdir -p gpurun_out
cp abtest/lib_ba.so paper_2311_09275_b200/lib/libising.so
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bench_parity.py -m gpu -q -x -k "band or grid or c4b_eight or torus or fused or icm or anneal or checkpoint" > gpurun_out/bands_pytest.log 2>&1; echo "rc=$?"; tail -1 gpurun_out/bands_pytest.log
for r in 1 2; do for v in ba bb; do
  cp abtest/lib_$v.so paper_2311_09275_b200/lib/libising.so
  timeout 300 python bench.py --workload c4b --copies 16 --steps 3 --warmup 2 --no-cpu --no-e2e --no-c5 > gpurun_out/abb_$v.log 2>&1
  tail -1 gpurun_out/abb_$v.log | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['value'], d['roofline']['kernel'], d['clocks']['sm_mhz'])" 2>&1 | tail -1
done; done
