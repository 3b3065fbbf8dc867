#!/bin/bash
O=gpurun_out/${1:-tmopab}; shift; mkdir -p $O
for spec in "$@"; do
  IFS='|' read -r lab lib <<< "$spec"
  L=""; [ -n "$lib" ] && L="HX_LIB=paper_2112_07075_b200/lib_$lib.so"
  env $L timeout 600 python tools/bench_tmop.py --cpu-n 0 > $O/$lab.json 2> $O/$lab.err
  python -c "import json;d=json.load(open('$O/$lab.json'));print('$lab', {k:round(v['ms']*1e3,1) for k,v in d['calls'].items()})"
done
