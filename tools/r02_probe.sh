mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/r8_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r8_tests.log
ISING_GRID_SCHED=1 timeout 600 python bench.py --sweeps 5000 --steps 2 --warmup 1 --no-cpu --no-e2e --no-c5 --no-projection > gpurun_out/r8_c4b_sched1.log 2>&1
echo done
