#!/bin/bash
O=gpurun_out/r2i; mkdir -p $O
HX_MASS_W2=2 timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py -q -x -p no:cacheprovider > $O/tests.txt 2>&1; tail -3 $O/tests.txt
bash tools/gpu_ab2.sh $O "base||" "w2pf|HX_MASS_W2=2|" "w2pfm5|HX_MASS_W2=2|w2m5" "w2pfm6|HX_MASS_W2=2|w2m6" "w2m6|HX_MASS_W2=1|w2m6" "base2||"
HX_MASS_W2=2 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_mass_w2 -s 30 -c 1 -o $O/prof_w2pf python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1; echo "ncu rc=$?"
python tools/ncu_summary.py $O/sum_w2pf.md $O/prof_w2pf.ncu-rep > /dev/null 2>&1
python tools/ncu_lines.py $O/prof_w2pf.ncu-rep 30 > $O/lines_w2pf.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_rates_pc -s 2 -c 1 -o $O/prof_rates python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1; echo "ncu rc=$?"
python tools/ncu_summary.py $O/sum_rates.md $O/prof_rates.ncu-rep > /dev/null 2>&1
python tools/ncu_lines.py $O/prof_rates.ncu-rep 40 > $O/lines_rates.txt 2>&1
python tools/ncu_lines.py $O/prof_rates.ncu-rep 30 bank > $O/bank_rates.txt 2>&1
