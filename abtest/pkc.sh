#!/bin/bash
cp abtest/lib_cb.so paper_2311_09275_b200/lib/libising.so
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "packed" > gpurun_out/pkc_cb.log 2>&1; echo "cb rc=$?"; tail -1 gpurun_out/pkc_cb.log
bash abtest/pk.sh ca cb
