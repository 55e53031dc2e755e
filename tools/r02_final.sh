#!/bin/bash
# Final round-2 evidence (run under gpurun): the measured memory roof of the C5 pattern, the default
# bench line as the driver runs it, the reference arm, the other workloads, launch lists, ncu
# captures of the two dominant kernels, the GPU test suite.
mkdir -p gpurun_out
python tools/gather_peak.py --out gpurun_out/gather_peak.json > gpurun_out/fin_gather_peak.log 2>&1
cp gpurun_out/gather_peak.json profiles/gather_peak.json 2>/dev/null
timeout 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/fin_bench_default.log 2>&1; echo "rc=$?" >> gpurun_out/fin_bench_default.log
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/fin_bench_ref.log 2>&1
for w in c2 c3 c4a c1; do
  timeout 900 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu --no-c5 > gpurun_out/fin_bench_$w.log 2>&1
done
timeout 900 python bench.py --workload c4b --copies 16 --steps 5 --warmup 3 --no-cpu --no-c5 > gpurun_out/fin_bench_c4b_share16.log 2>&1
timeout 900 python bench.py --workload c5 --steps 5 --warmup 3 > gpurun_out/fin_bench_c5.log 2>&1
python bench.py --workload c5 --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/fin_plain_launch_c5.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/fin_launches_c5.csv \
  python bench.py --workload c5 --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/fin_ncu_launch_c5.log 2>&1
bash tools/prof.sh c5 k_csr_i8_ring 5 fin_c5ring --no-c5
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/fin_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/fin_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/fin_smoke.log
echo done
