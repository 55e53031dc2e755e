mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/r19_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r19_tests.log
timeout 600 python bench.py --workload c4b --copies 16 --steps 5 --warmup 3 --no-cpu --no-e2e --no-c5 > gpurun_out/r19_share16.log 2>&1
python tools/pipes_profile.py c4b:share16 > gpurun_out/r19_pipes.log 2>&1
echo done
