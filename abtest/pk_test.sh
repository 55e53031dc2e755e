#!/bin/bash
# parity tests of the packed kernel on variant lib $1, then A/B of the given variants
v=$1; shift
cp abtest/lib_$v.so paper_2311_09275_b200/lib/libising.so
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "packed" > gpurun_out/pkt_$v.log 2>&1; echo "rc=$?" >> gpurun_out/pkt_$v.log
tail -2 gpurun_out/pkt_$v.log
bash abtest/pk.sh "$@"
