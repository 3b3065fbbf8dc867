#!/bin/bash
# ncu --set full with warm caches (--cache-control none) of the named kernels (usage: tools/gpu_warm.sh TAG "k1 k2")
TAG=$1; KS=$2
for K in $KS; do
  S=30; case $K in *rates*) S=4;; esac
  timeout 600 ncu --set full --cache-control none --clock-control none --import-source on -k regex:$K -s $S -c 1 -o gpurun_out/warm_${K}_$TAG python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
  python tools/ncu_summary.py gpurun_out/wsum_${K}_$TAG.md gpurun_out/warm_${K}_$TAG.ncu-rep > /dev/null 2>&1
done
