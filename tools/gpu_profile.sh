#!/bin/bash
# committed-evidence capture: launch list + ncu --set full of the top kernels, summarised on the box
# (usage: tools/gpu_profile.sh TAG [keep-rep-regex])
TAG=${1:-r1}; KEEP=${2:-k_mass_pc}
mkdir -p gpurun_out/prof_$TAG
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/prof_$TAG/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
for K in k_mass_pc k_cg_node k_rates k_cg_init; do
  S=30; [ $K = k_rates ] && S=4; [ $K = k_cg_init ] && S=2
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$K -s $S -c 1 -o /tmp/full_${K} python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
done
python tools/ncu_summary.py gpurun_out/prof_$TAG/ncu_summary.md /tmp/full_k_mass_pc.ncu-rep /tmp/full_k_cg_node.ncu-rep /tmp/full_k_rates.ncu-rep /tmp/full_k_cg_init.ncu-rep --launches gpurun_out/prof_$TAG/launches.csv
for K in k_mass_pc k_cg_node k_rates k_cg_init; do python tools/ncu_hot.py /tmp/full_$K.ncu-rep 25 > gpurun_out/prof_$TAG/hot_$K.txt; done
cp /tmp/full_${KEEP}.ncu-rep gpurun_out/prof_$TAG/ 2>/dev/null
timeout 300 python bench.py --steps 10 --warmup 3 > gpurun_out/prof_$TAG/bench.json 2> gpurun_out/prof_$TAG/bench.err
du -sh gpurun_out
tail -1 gpurun_out/prof_$TAG/bench.json | cut -c1-300
