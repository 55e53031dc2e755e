#!/bin/bash
# Round-2 evidence on the final build (packed-row C5): full GPU suite, smoke, the default line as the
# driver runs it, the reference arm, the C5 workload line.
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/f6_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/f6_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f6_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/f6_smoke.log
timeout 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/f6_bench_default.log 2>&1; echo "rc=$?" >> gpurun_out/f6_bench_default.log
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/f6_bench_ref.log 2>&1
timeout 600 python bench.py --workload c5 --steps 5 --warmup 3 > gpurun_out/f6_bench_c5.log 2>&1; echo "rc=$?" >> gpurun_out/f6_bench_c5.log
echo done
