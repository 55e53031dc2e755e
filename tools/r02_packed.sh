#!/bin/bash
# Packed-row C5 path: parity tests, then C5 with the packed rows (default) and with the int8 ring kernel.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "packed or float or c5" > gpurun_out/pk_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/pk_pytest.log
timeout 600 python bench.py --workload c5 --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/pk_bench_c5.log 2>&1; echo "rc=$?" >> gpurun_out/pk_bench_c5.log
ISING_I8_PACKED=0 timeout 600 python bench.py --workload c5 --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/pk_bench_c5_ring.log 2>&1; echo "rc=$?" >> gpurun_out/pk_bench_c5_ring.log
echo done
