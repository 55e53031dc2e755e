# Round-2 evidence (run under gpurun): the default bench line as the driver runs it, the reference
# arm, launch lists, per-launch pipe counts of the bench's own launches, full ncu captures.
mkdir -p gpurun_out
python tools/alu_peak.py --ncu --out gpurun_out/alu_peak.json > gpurun_out/ev_alu_peak.log 2>&1
timeout 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/ev_bench_default.log 2>&1; echo "rc=$?" >> gpurun_out/ev_bench_default.log
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/ev_bench_ref.log 2>&1
for w in c2 c3 c4a c1; do
  timeout 900 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu --no-c5 > gpurun_out/ev_bench_$w.log 2>&1
done
timeout 900 python bench.py --workload c4b --copies 16 --steps 5 --warmup 3 --no-cpu --no-c5 > gpurun_out/ev_bench_c4b_share16.log 2>&1
python tools/pipes_profile.py c4b:full c4a:full c4b c4a > gpurun_out/ev_pipes.log 2>&1
python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-c5 --no-projection > gpurun_out/ev_plain_launch.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/ev_launches_c4b.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-c5 --no-projection > gpurun_out/ev_ncu_launch.log 2>&1
python bench.py --workload c5 --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/ev_plain_launch_c5.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/ev_launches_c5.csv \
  python bench.py --workload c5 --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/ev_ncu_launch_c5.log 2>&1
bash tools/prof.sh c4b k_grid_sched 1 c4b_sched --sweeps 100 --no-c5 --no-projection
bash tools/prof.sh c5 k_csr_i8_ring 5 c5ring --no-c5
echo done
