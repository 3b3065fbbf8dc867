#!/bin/bash
# tests + bench for both mass variants + ncu of the chosen kernels (usage: tools/gpu_quick.sh TAG "kernel regexes")
TAG=${1:-x}; KS=${2:-"k_mass3w k_cg_node"}
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for V in line column; do
  HX_MASS_KERNEL=$V timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_${TAG}_$V.json 2>gpurun_out/bench_${TAG}_$V.err
  python -c "import json;d=json.load(open('gpurun_out/bench_${TAG}_$V.json'));print('$V', round(d['value'],1), round(d['ms_per_step'],3), {k:(round(v['avg_us'],1),round(v['share'],3)) for k,v in d['kernels'].items()})" || tail -3 gpurun_out/bench_${TAG}_$V.err
done
for K in $KS; do
  S=30; [ $K = k_rates ] && S=4
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$K -s $S -c 1 -o gpurun_out/prof_${K}_$TAG python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
done
