#!/bin/bash
# parity of the register-prefetch variants, then A/B
for v in gb gc; do
  cp abtest/lib_$v.so paper_2311_09275_b200/lib/libising.so
  timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "packed" > gpurun_out/pkg_$v.log 2>&1; echo "$v rc=$?"; tail -1 gpurun_out/pkg_$v.log
done
bash abtest/pk.sh ga gb gc gd
