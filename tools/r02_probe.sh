mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bench_parity.py -x -q -k "csr or c3 or torus_equal or grid_kernel_equals or icm or anneal or checkpoint" > gpurun_out/r16_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r16_tests.log
timeout 600 python bench.py --workload c3 --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/r16_c3.log 2>&1
python tools/pipes_profile.py c3 > gpurun_out/r16_pipes.log 2>&1
echo done
