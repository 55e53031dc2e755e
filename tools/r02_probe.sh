mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_bench_parity.py tests/test_gpu_create.py tests/test_gpu_parity.py -x -q -k "sched or c4 or create or jp or ring or c5 or checks or int8 or readback or exp_bracket" > gpurun_out/r7_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r7_tests.log
for s in 1 0; do
  ISING_GRID_SCHED=$s timeout 600 python bench.py --sweeps 5000 --steps 2 --warmup 1 --no-cpu --no-e2e --no-c5 --no-projection > gpurun_out/r7_c4b_sched$s.log 2>&1
done
timeout 600 python bench.py --workload c2 --steps 3 --warmup 2 --no-cpu --no-e2e --no-c5 > gpurun_out/r7_c2.log 2>&1
timeout 900 python bench.py --workload c5 --steps 3 --warmup 2 --no-cpu > gpurun_out/r7_c5.log 2>&1
python tools/pipes_profile.py c4b c2 > gpurun_out/r7_pipes.log 2>&1
echo done
