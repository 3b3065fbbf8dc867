#!/bin/bash
# round-2 lease b: full GPU suite (incl. production-size parity), bench with graph-timed
# kernels, ncu launch list
O=gpurun_out/r2b; mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q -x -p no:cacheprovider --durations=15 > $O/tests.txt 2>&1; tail -25 $O/tests.txt
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"; tail -3 $O/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1; echo "ncu rc=$?"
python - <<'PY'
import json
d = json.load(open("gpurun_out/r2b/bench.json"))
print("value", d["value"], "e2e", d["e2e"]["value"], "ms", d["ms_per_step"], "kpass", d["kernel_pass"]["ms_per_step"])
for k, v in d["kernels"].items():
    print(k, v["launches"], round(v["avg_us"], 2), round(v["share"], 3), round(v["hbm_frac"] or 0, 3))
PY
