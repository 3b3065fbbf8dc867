#!/bin/bash
# bench every BASELINE.json config on one GPU (usage: tools/gpu_configs.sh TAG)
TAG=${1:-cfg}; export TAG
mkdir -p gpurun_out/cfg_$TAG
run() { NAME=$1; shift; timeout 400 python bench.py --steps 20 --warmup 5 --no-cpu "$@" > gpurun_out/cfg_$TAG/$NAME.json 2> gpurun_out/cfg_$TAG/$NAME.err; tail -1 gpurun_out/cfg_$TAG/$NAME.err | cut -c1-200; }
run sedov_q3_n23 --p 3 --n 23
run sedov_q2_n34 --p 2 --n 34
run tgv_q4_n17 --p 4 --n 17 --problem tgv
run triple_q3_k8 --p 3 --n 8 --problem triple
run sedov_q3_n30 --p 3 --n 30
python - <<'PY'
import json, glob, os
rows = []
for f in sorted(glob.glob("gpurun_out/cfg_%s/*.json" % os.environ.get("TAG", "cfg"))):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, "failed", e); continue
    k = d["kernels"]
    print(os.path.basename(f), round(d["value"], 1), round(d["ms_per_step"], 3), (d.get("e2e") or {}).get("value"),
          {n: (round(v["avg_us"], 1), round(v["gbs"] or 0)) for n, v in k.items()})
PY
