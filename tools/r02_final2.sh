#!/bin/bash
# Round-2 evidence refresh after the C1 register path: C1 line, the default line (C4b + nested C5),
# the full GPU test suite, smoke, and an ncu capture of the C1 kernel.
mkdir -p gpurun_out
timeout 600 python bench.py --workload c1 --steps 5 --warmup 3 --no-c5 > gpurun_out/fin2_bench_c1.log 2>&1
timeout 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/fin2_bench_default.log 2>&1; echo "rc=$?" >> gpurun_out/fin2_bench_default.log
bash tools/prof.sh c1 k_i8_cluster 1 fin2_c1 --no-c5
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/fin2_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/fin2_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin2_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/fin2_smoke.log
echo done
