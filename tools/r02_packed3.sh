#!/bin/bash
# Packed-row C5 (final build): parity tests, default bench line (C4b + nested C5 on packed rows + int8-row
# record), per-sweep pipe counts of the packed kernel, ncu capture of one class phase, C5 launch list.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bench_parity.py -m gpu -q -x -k "packed or float or c5" > gpurun_out/pk3_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/pk3_pytest.log
timeout 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/pk3_bench_default.log 2>&1; echo "rc=$?" >> gpurun_out/pk3_bench_default.log
python tools/pipes_profile.py c5:packed > gpurun_out/pk3_pipes.log 2>&1
bash tools/prof.sh c5 k_csr_packed 5 c5pk_v3
python bench.py --workload c5 --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/pk3_plain_launch_c5.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/pk3_launches_c5.csv \
  python bench.py --workload c5 --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/pk3_ncu_launch_c5.log 2>&1
echo done
