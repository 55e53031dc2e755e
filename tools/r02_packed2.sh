#!/bin/bash
# Packed-row C5 path (ring version): parity tests, C5 bench (packed default), ncu capture of one class phase.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "packed or float or c5" > gpurun_out/pk2_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/pk2_pytest.log
timeout 600 python bench.py --workload c5 --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/pk2_bench_c5.log 2>&1; echo "rc=$?" >> gpurun_out/pk2_bench_c5.log
bash tools/prof.sh c5 k_csr_packed 5 c5pk_v2
echo done
