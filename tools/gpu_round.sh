#!/bin/bash
# one GPU call: tests, smoke, bench, launch list and ncu of the top kernels (usage: tools/gpu_round.sh TAG)
TAG=${1:-x}
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/tests_$TAG.txt 2>&1; tail -1 gpurun_out/tests_$TAG.txt
python -c 'import __graft_entry__ as g; g.smoke()' 2>&1 | tail -1
timeout 300 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_$TAG.json 2>gpurun_out/bench_$TAG.err; tail -2 gpurun_out/bench_$TAG.err
bash tools/gpu_profile.sh $TAG
