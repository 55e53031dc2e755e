#!/bin/bash
# ncu captures of both C5 kernels on the final build + per-sweep pipe counts of the packed kernel
mkdir -p gpurun_out
python tools/pipes_profile.py c5:packed > gpurun_out/cap_pipes.log 2>&1
bash tools/prof.sh c5 k_csr_packed 5 c5pk_final
ISING_I8_PACKED=0 bash tools/prof.sh c5 k_csr_i8_ring 5 c5ring_final
echo done
