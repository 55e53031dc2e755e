mkdir -p gpurun_out
python tools/alu_peak.py --ncu --out gpurun_out/alu_peak.json > gpurun_out/r4_alu_peak.log 2>&1
python tools/pipes_profile.py c4b c4b:clusters c2 c4a c3 c4b:share16 c1 > gpurun_out/r4_pipes.log 2>&1
ISING_GRID_SCHED=1 python bench.py --sweeps 100 --steps 1 --warmup 1 --no-cpu --no-e2e --no-c5 --no-projection > gpurun_out/r4_plain_sched.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_grid_sched -s 1 -c 1 -o gpurun_out/r4_c4b_sched python bench.py --sweeps 100 --steps 1 --warmup 1 --no-cpu --no-e2e --no-c5 --no-projection > gpurun_out/r4_ncu_sched.log 2>&1
ISING_GRID_SCHED=0 python bench.py --sweeps 100 --steps 1 --warmup 1 --no-cpu --no-e2e --no-c5 --no-projection > gpurun_out/r4_plain_clu.log 2>&1 && \
ISING_GRID_SCHED=0 ncu --set full --clock-control none --import-source on -k regex:k_grid_bits -s 1 -c 1 -o gpurun_out/r4_c4b_clusters python bench.py --sweeps 100 --steps 1 --warmup 1 --no-cpu --no-e2e --no-c5 --no-projection > gpurun_out/r4_ncu_clu.log 2>&1
echo done
