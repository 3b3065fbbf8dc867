#!/bin/bash
O=gpurun_out/${1:-q2ab}; shift; mkdir -p $O
for spec in "$@"; do
  IFS='|' read -r lab lib <<< "$spec"
  L=""; [ -n "$lib" ] && L="HX_LIB=paper_2112_07075_b200/lib_$lib.so"
  env $L timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e --p 2 --n 34 > $O/$lab.json 2> $O/$lab.err
  python -c "import json;d=json.load(open('$O/$lab.json'));print('$lab', round(d['value'],1), {k:round(v['avg_us'],1) for k,v in d['kernels'].items()})"
done
