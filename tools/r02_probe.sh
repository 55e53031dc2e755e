mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/r13_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r13_tests.log
timeout 600 python bench.py --sweeps 10000 --steps 3 --warmup 2 --no-cpu --no-e2e --no-c5 --no-projection > gpurun_out/r13_c4b.log 2>&1
timeout 600 python bench.py --workload c4b --copies 16 --sweeps 10000 --steps 3 --warmup 2 --no-cpu --no-e2e --no-c5 > gpurun_out/r13_share16.log 2>&1
timeout 600 python bench.py --workload c2 --steps 5 --warmup 3 --no-cpu --no-e2e --no-c5 > gpurun_out/r13_c2.log 2>&1
echo done
