#!/bin/bash
# committed-evidence capture: launch list + ncu --set full (cold and warm cache) of the top kernels,
# summarised on the box (usage: tools/gpu_profile.sh TAG)
TAG=${1:-r1}
OUT=gpurun_out/prof_$TAG
mkdir -p $OUT
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file $OUT/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
KS="k_mass_brick k_cg_node k_rates_pc k_cg_init k_valid"
for K in $KS; do
  S=30; case $K in *rates*) S=1;; *init*) S=2;; *valid*) S=1;; esac
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$K -s $S -c 1 -o /tmp/full_${K} python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
  timeout 600 ncu --set full --cache-control none --clock-control none --import-source on -k regex:$K -s $S -c 1 -o /tmp/warm_${K} python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
done
python tools/ncu_summary.py $OUT/ncu_summary.md $(for K in $KS; do echo /tmp/full_$K.ncu-rep; done) --launches $OUT/launches.csv
python tools/ncu_summary.py $OUT/ncu_summary_warm.md $(for K in $KS; do echo /tmp/warm_$K.ncu-rep; done)
for K in $KS; do python tools/ncu_lines.py /tmp/full_$K.ncu-rep 30 > $OUT/lines_$K.txt; done
cp /tmp/full_k_mass_brick.ncu-rep /tmp/full_k_rates_pc.ncu-rep $OUT/ 2>/dev/null
timeout 300 python bench.py --steps 10 --warmup 3 > $OUT/bench.json 2> $OUT/bench.err
du -sh gpurun_out
tail -1 $OUT/bench.json | cut -c1-300
