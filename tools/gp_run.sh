mkdir -p gpurun_out
for cfg in "ring 4 3" "ring 4 4" "ring 6 2" "ring 6 3" "ring 8 2" "ldg 4 4" "ldg 4 8" "ldg 8 4" "ldg 2 8"; do
  set -- $cfg
  timeout 120 tools/gather_peak $1 $2 $3 10 >> gpurun_out/gp.jsonl 2>&1
done
nvidia-smi --query-gpu=clocks.sm,clocks.mem,power.draw,clocks_throttle_reasons.active --format=csv >> gpurun_out/gp.jsonl
timeout 300 python bench.py --workload c5 --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/gp_c5.log 2>&1
