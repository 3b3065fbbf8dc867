#!/bin/bash
# A/B bench of env-selected variants + ncu --set full of named kernels under the first variant
# usage: tools/gpu_ab.sh TAG "kregex1 kregex2" "ENV=a" "ENV=b" ...
TAG=$1; KS=$2; shift 2
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
i=0
for V in "$@"; do
  i=$((i+1))
  env $V timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_${TAG}_$i.json 2>gpurun_out/bench_${TAG}_$i.err
  python -c "import json;d=json.load(open('gpurun_out/bench_${TAG}_$i.json'));print('$V', round(d['value'],1), round(d['ms_per_step'],3), {k:(round(v['avg_us'],1),round(v['share'],3)) for k,v in d['kernels'].items()})" || tail -3 gpurun_out/bench_${TAG}_$i.err
done
for K in $KS; do
  S=30; case $K in *rates*) S=4;; esac
  env $1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:$K -s $S -c 1 -o gpurun_out/prof_${K}_$TAG python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
  python tools/ncu_summary.py gpurun_out/sum_${K}_$TAG.md gpurun_out/prof_${K}_$TAG.ncu-rep > /dev/null 2>&1
  python tools/ncu_hot.py gpurun_out/prof_${K}_$TAG.ncu-rep 30 > gpurun_out/hot_${K}_$TAG.txt 2>&1
done
ls gpurun_out | tail -8
