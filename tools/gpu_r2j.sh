#!/bin/bash
O=gpurun_out/r2j; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > $O/tests.txt 2>&1; tail -3 $O/tests.txt
bash tools/gpu_ab2.sh $O "new||" "pp|HX_PAIRS_INPLACE=0|" "invd|HX_INVD_NODE=0|" "old|HX_PAIRS_INPLACE=0 HX_INVD_NODE=0|" "new2||"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_rates_pc -s 2 -c 1 -o /tmp/prof_rates python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1; echo "ncu rc=$?"
python tools/ncu_summary.py $O/sum_rates.md /tmp/prof_rates.ncu-rep > /dev/null 2>&1
python tools/ncu_lines.py /tmp/prof_rates.ncu-rep 40 > $O/lines_rates.txt 2>&1
python tools/ncu_lines.py /tmp/prof_rates.ncu-rep 30 bank > $O/bank_rates.txt 2>&1
ncu -i /tmp/prof_rates.ncu-rep --page raw --csv > $O/raw_rates.csv 2>/dev/null
for K in k_mass_brick k_cg_node; do
timeout 600 ncu --set full --cache-control none --clock-control none --import-source on -k regex:$K -s 30 -c 1 -o /tmp/prof_$K python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1; echo "ncu rc=$?"
python tools/ncu_summary.py $O/sum_warm_$K.md /tmp/prof_$K.ncu-rep > /dev/null 2>&1
ncu -i /tmp/prof_$K.ncu-rep --page raw --csv > $O/raw_warm_$K.csv 2>/dev/null
done
du -sh $O
