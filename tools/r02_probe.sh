mkdir -p gpurun_out
bash tools/prof.sh c4b k_grid_sched 1 c4b_sched_v2 --sweeps 100 --no-c5 --no-projection
python tools/pipes_profile.py c4b:full c2 c4a:full > gpurun_out/r14_pipes.log 2>&1
echo done
