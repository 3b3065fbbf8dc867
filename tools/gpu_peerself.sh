#!/bin/bash
# one-rank cost of the multi-GPU exchange protocol: bench.py --peer-self vs the plain step, per library variant
O=gpurun_out/${1:-peerself}; shift; mkdir -p $O
for spec in "$@"; do
  IFS='|' read -r lab lib <<< "$spec"
  L=""; [ -n "$lib" ] && L="HX_LIB=paper_2112_07075_b200/lib_$lib.so"
  for mode in plain peer; do
    F=""; [ $mode = peer ] && F="--peer-self"
    env $L timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e $F > $O/${lab}_$mode.json 2> $O/${lab}_$mode.err
    python -c "import json;d=json.load(open('$O/${lab}_$mode.json'));print('$lab $mode', round(d['value'],1), round(d['ms_per_step'],4))"
  done
done
