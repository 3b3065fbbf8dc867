#!/bin/bash
# final evidence: GPU suite, smoke, the driver's bench command (twice), reference arm, launch list,
# cold + warm ncu captures of the step kernels with per-line / stall summaries
O=gpurun_out/final; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/gpu.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/tests.txt 2>&1; tail -2 $O/tests.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; echo "smoke rc=$?"
for i in 1 2; do timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > $O/bench_$i.json 2> $O/bench_$i.err; echo "bench rc=$?"; done
timeout 900 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > $O/ref.json 2> $O/ref.err; echo "ref rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 500 --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1; echo "launches rc=$?"
for K in k_mass_brick k_cg_node k_rates_pc; do
  S=30; case $K in *rates*) S=1;; esac
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$K -s $S -c 1 -o /tmp/f_$K python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
  timeout 600 ncu --set full --cache-control none --clock-control none --import-source on -k regex:$K -s $S -c 1 -o /tmp/w_$K python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
  python tools/ncu_summary.py $O/cold_$K.md /tmp/f_$K.ncu-rep > /dev/null 2>&1
  python tools/ncu_summary.py $O/warm_$K.md /tmp/w_$K.ncu-rep > /dev/null 2>&1
  ncu -i /tmp/w_$K.ncu-rep --page raw --csv > $O/raw_warm_$K.csv 2>/dev/null
  ncu -i /tmp/f_$K.ncu-rep --page raw --csv > $O/raw_cold_$K.csv 2>/dev/null
  python tools/ncu_stalls.py $O/raw_warm_$K.csv > $O/stalls_warm_$K.txt 2>&1
  python tools/ncu_lines.py /tmp/w_$K.ncu-rep 30 > $O/lines_warm_$K.txt 2>&1
done
ls $O
