#!/bin/bash
# one GPU call: tests, bench, ncu of the top kernels (usage: tools/gpu_round.sh TAG [pytest-args])
TAG=${1:-x}
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
timeout 300 python bench.py --steps 10 --warmup 3 --cpu-n 10 > gpurun_out/bench_$TAG.json 2>gpurun_out/bench_$TAG.err; tail -2 gpurun_out/bench_$TAG.err; cat gpurun_out/bench_$TAG.json
for K in k_mass3d k_cg_node k_rates; do
  S=30; [ $K = k_rates ] && S=4
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$K -s $S -c 1 -o gpurun_out/prof_${K}_$TAG python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
done
ls gpurun_out | tail -5
