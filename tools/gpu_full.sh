#!/bin/bash
# full GPU check: GPU suite, smoke, the driver's bench command, reference arm, launch list
# usage: bash tools/gpu_full.sh <outdir-name>
O=gpurun_out/${1:-full}; mkdir -p $O; export O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/gpu.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=20 > $O/tests.txt 2>&1; tail -30 $O/tests.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; echo "smoke rc=$?"; tail -2 $O/smoke.txt
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"; tail -3 $O/bench.err
[ -n "$NOREF" ] || { timeout 900 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > $O/ref.json 2> $O/ref.err; echo "ref rc=$?"; tail -3 $O/ref.err; }
[ -n "$NONCU" ] || { timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1; echo "ncu rc=$?"; }
python - <<'PY'
import json, os
d = json.load(open(os.environ["O"] + "/bench.json"))
print("value", d["value"], "e2e", d["e2e"]["value"], "ms", d["ms_per_step"])
for k, v in d["kernels"].items():
    print(k, v["launches"], round(v["avg_us"], 2), round(v["share"], 3), round(v["hbm_frac"] or 0, 3))
PY
