#!/bin/bash
# A/B of library variants and env knobs: tools/gpu_ab2.sh OUTDIR "label|ENV=..|libname" ...
O=$1; shift; mkdir -p $O
summ() { python - "$1" "$2" <<'PY'
import json, sys
try:
    d = json.load(open(sys.argv[1]))
except Exception as exc:
    print(sys.argv[2], "no json", exc); sys.exit(0)
ks = " ".join("%s=%.2f" % (k[:6], v["avg_us"]) for k, v in d["kernels"].items())
print("%-14s value %.1f ms %.4f | %s" % (sys.argv[2], d["value"], d["ms_per_step"], ks))
PY
}
for spec in "$@"; do
  IFS='|' read -r lab envs lib <<< "$spec"
  L=""; [ -n "$lib" ] && L="HX_LIB=paper_2112_07075_b200/lib_$lib.so"
  env $envs $L timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e > $O/b_$lab.json 2> $O/b_$lab.err || tail -3 $O/b_$lab.err
  summ $O/b_$lab.json $lab
done
