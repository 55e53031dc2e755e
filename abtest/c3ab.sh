mkdir -p gpurun_out
for rep in 1 2; do
for cfg in "c768 768" "c1024 768" "c1024 832" "c1024 896" "c1024 960" "c1024 1024"; do
  set -- $cfg
  cp abtest/lib_$1.so paper_2311_09275_b200/lib/libising.so; touch paper_2311_09275_b200/lib/libising.so
  timeout 600 python bench.py --workload c3 --steps 3 --warmup 3 --no-cpu --no-e2e --no-c5 --threads $2 > gpurun_out/c3ab.log 2>&1
  tail -1 gpurun_out/c3ab.log | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1 $2', '%.4g'%d['value'])" 2>&1 | tail -1
done; done
