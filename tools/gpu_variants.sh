#!/bin/bash
# bench variants selected by environment (usage: tools/gpu_variants.sh TAG "ENV1=a ENV2=b" "ENV1=c" ...)
TAG=$1; shift
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
i=0
for V in "$@"; do
  i=$((i+1))
  env $V timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_${TAG}_$i.json 2>gpurun_out/bench_${TAG}_$i.err
  python -c "import json;d=json.load(open('gpurun_out/bench_${TAG}_$i.json'));print('$V', round(d['value'],1), round(d['ms_per_step'],3), {k:(round(v['avg_us'],1),round(v['share'],3)) for k,v in d['kernels'].items()})" || tail -3 gpurun_out/bench_${TAG}_$i.err
done
