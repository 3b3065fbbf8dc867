O=gpurun_out/r2p; mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q -x -p no:cacheprovider > $O/tests.txt 2>&1; tail -5 $O/tests.txt
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"; tail -3 $O/bench.err
python - <<'PY'
import json
d = json.load(open("gpurun_out/r2p/bench.json"))
print("value", d["value"], "e2e", d["e2e"]["value"], "api", d["api"], "ms", d["ms_per_step"])
for k, v in d["kernels"].items():
    print(k, v["launches"], round(v["avg_us"], 2))
PY
