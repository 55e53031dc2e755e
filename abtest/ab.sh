#!/bin/bash
# A/B: alternate builds of libising.so (abtest/lib_<v>.so) over workloads; prints attempts/s.
# usage: VARIANTS="a b" WORKLOADS="c2 c3" REPS=2 bash abtest/ab.sh [extra bench args]
for rep in $(seq ${REPS:-2}); do
  for v in ${VARIANTS:-a b}; do
    cp abtest/lib_$v.so paper_2311_09275_b200/lib/libising.so; touch paper_2311_09275_b200/lib/libising.so
    for w in ${WORKLOADS:-c2}; do
      timeout 600 python bench.py --workload $w --steps 3 --warmup 3 --no-cpu --no-e2e "$@" > gpurun_out/ab_${v}_$w.log 2>&1
      tail -1 gpurun_out/ab_${v}_$w.log | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v $w', '%.4g'%d['value'], '%.2f'%d['ms_per_step'], d['clocks']['sm_mhz'])" 2>&1 | tail -1
    done
  done
done
