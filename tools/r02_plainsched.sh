#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_bench_parity.py tests/test_gpu_parity.py -m gpu -q -x -k "sched or north_star or fused or grid" > gpurun_out/ps_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/ps_pytest.log
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --no-c5 > gpurun_out/ps_bench.log 2>&1; echo "rc=$?" >> gpurun_out/ps_bench.log
echo done
