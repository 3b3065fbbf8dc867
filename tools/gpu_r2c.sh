#!/bin/bash
# lease c: GPU suite, bench with duplication-timed kernels, mass pipeline variants (A/B)
O=gpurun_out/r2c; mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/tests.txt 2>&1; tail -4 $O/tests.txt
summ() { python - "$1" <<'PY'
import json, sys
d = json.load(open(sys.argv[1]))
print(sys.argv[1], "value %.1f ms %.4f" % (d["value"], d["ms_per_step"]), "e2e", d["e2e"] and round(d["e2e"]["value"], 1))
for k, v in d["kernels"].items():
    print("   %-9s n=%4d avg=%7.2f us share=%.3f hbm=%.3f" % (k, v["launches"], v["avg_us"], v["share"], v["hbm_frac"] or 0))
PY
}
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"; tail -3 $O/bench.err; summ $O/bench.json
for V in pipe128 pipe128d pipe256; do
  HX_LIB=paper_2112_07075_b200/lib_$V.so HX_GRID_CAP= timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "mass_pa or nstep" -p no:cacheprovider > $O/t_$V.txt 2>&1; echo "$V tests: $(tail -1 $O/t_$V.txt)"
  HX_LIB=paper_2112_07075_b200/lib_$V.so timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e > $O/b_$V.json 2> $O/b_$V.err; summ $O/b_$V.json
done
