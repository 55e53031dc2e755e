#!/bin/bash
# Round-end evidence (run under gpurun): GPU tests, bench lines of every workload, the
# reference arm, the ncu launch list of the default bench command and a full ncu capture
# of the C5 ring kernel.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench_c2.json.log 2>&1
for w in c1 c3 c4a c4b c5; do
  timeout 900 python bench.py --workload $w --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_$w.json.log 2>&1
done
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json.log 2>&1
python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/plain_launch.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_launch.log 2>&1
bash tools/prof.sh c5 k_csr_i8_ring 5 c5ring
echo done
