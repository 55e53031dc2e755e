mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_bench_parity.py -x -q -k "sched or merge" > gpurun_out/r2_sched_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2_sched_tests.log
for s in 1 0; do
  ISING_GRID_SCHED=$s timeout 600 python bench.py --sweeps 5000 --steps 2 --warmup 1 --no-cpu --no-e2e --no-c5 --no-projection > gpurun_out/r2_c4b_sched$s.log 2>&1
done
M=smsp__inst_executed.sum,sm__inst_executed_pipe_alu.sum,sm__inst_executed_pipe_fma.sum,sm__inst_executed_pipe_fmaheavy.sum,sm__inst_executed_pipe_fmalite.sum,sm__inst_executed_pipe_uniform.sum,sm__inst_executed_pipe_lsu.sum,sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active,sm__cycles_elapsed.avg,sm__cycles_active.avg,smsp__issue_active.avg.pct_of_peak_sustained_active
tools/alu_peak 1 1024 2 2000 > /dev/null && ncu --metrics $M --clock-control none -c 1 --csv tools/alu_peak 1 1024 2 2000 > gpurun_out/r2_alu_pipes.csv 2>&1
tools/alu_peak 0 1024 2 2000 > /dev/null && ncu --metrics $M --clock-control none -c 1 --csv tools/alu_peak 0 1024 2 2000 > gpurun_out/r2_alu0_pipes.csv 2>&1
python bench.py --workload c2 --sweeps 100 --steps 1 --warmup 3 --no-cpu --no-e2e --no-c5 > gpurun_out/r2_c2_plain.log 2>&1 && ncu --metrics $M --clock-control none -k regex:k_grid_bits -s 3 -c 1 --csv python bench.py --workload c2 --sweeps 100 --steps 1 --warmup 3 --no-cpu --no-e2e --no-c5 > gpurun_out/r2_c2_pipes.csv 2>&1
echo done
