#!/bin/bash
# ncu --set full capture of one launch of the dominant kernel of a workload (run under gpurun).
# usage: bash tools/prof.sh <workload> <kernel-regex> <skip> <tag> [extra bench args]
w=$1; k=$2; s=$3; tag=$4; shift 4
cmd="python bench.py --workload $w --steps 1 --warmup 3 --no-cpu --no-e2e $*"
$cmd > gpurun_out/plain_$tag.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:$k -s $s -c 1 -o gpurun_out/prof_$tag $cmd > gpurun_out/ncu_$tag.log 2>&1
echo "$tag rc=$?"
