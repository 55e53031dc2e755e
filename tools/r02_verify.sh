#!/bin/bash
# Re-verify the current HEAD on a B200: GPU tests, smoke, default bench line.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/v_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/v_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/v_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/v_smoke.log
timeout 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/v_bench_default.log 2>&1; echo "rc=$?" >> gpurun_out/v_bench_default.log
echo done
