#!/bin/bash
# lease f: TMA mass kernel -- parity suite, A/B bench vs the thread-gather kernel, launch list
O=gpurun_out/r2f; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py tests/test_gpu_properties.py -q -x -p no:cacheprovider > $O/tests.txt 2>&1; tail -5 $O/tests.txt
summ() { python - "$1" <<'PY'
import json, sys
try:
    d = json.load(open(sys.argv[1]))
except Exception as exc:
    print(sys.argv[1], "no json", exc); sys.exit(0)
print(sys.argv[1], "value %.1f ms %.4f" % (d["value"], d["ms_per_step"]), "e2e", d["e2e"] and round(d["e2e"]["value"], 1))
for k, v in d["kernels"].items():
    print("   %-9s n=%4d avg=%7.2f us share=%.3f hbm=%.3f" % (k, v["launches"], v["avg_us"], v["share"], v["hbm_frac"] or 0))
PY
}
for V in 1 0; do
  HX_MASS_TMA=$V timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e > $O/b_tma$V.json 2> $O/b_tma$V.err; tail -2 $O/b_tma$V.err; summ $O/b_tma$V.json
done
HX_GRAPH=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1; echo "ncu rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_mass_tma -s 30 -c 1 -o $O/prof_mass_tma python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1; echo "ncu full rc=$?"
python tools/ncu_summary.py $O/sum_mass_tma.md $O/prof_mass_tma.ncu-rep > /dev/null 2>&1
python tools/ncu_lines.py $O/prof_mass_tma.ncu-rep 30 > $O/lines_mass_tma.txt 2>&1
