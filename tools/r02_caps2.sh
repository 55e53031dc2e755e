#!/bin/bash
# Final-build evidence for the headline kernel: a second default line, per-attempt pipe counts of the
# bench's own C4b launch, an ncu --set full capture of a 100-sweep k_grid_sched launch
mkdir -p gpurun_out
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/c2_bench_default.log 2>&1; echo "rc=$?" >> gpurun_out/c2_bench_default.log
python tools/pipes_profile.py c4b:full > gpurun_out/c2_pipes.log 2>&1
bash tools/prof.sh c4b k_grid_sched 1 c4b_sched_final --sweeps 100 --no-c5 --no-projection
echo done
