#!/bin/bash
# A/B: run the same bench with two builds of libising.so
for v in ${VARIANTS:-a b}; do
  cp abtest/lib_$v.so paper_2311_09275_b200/lib/libising.so
  touch paper_2311_09275_b200/lib/libising.so
  timeout 600 python bench.py "$@" > gpurun_out/ab_$v.log 2>&1
  echo "$v rc=$?"
done
