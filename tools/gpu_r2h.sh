#!/bin/bash
O=gpurun_out/r2h; mkdir -p $O
HX_MASS_W2=1 timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py -q -x -p no:cacheprovider > $O/tests.txt 2>&1; tail -3 $O/tests.txt
bash tools/gpu_ab2.sh $O "base||" "w2|HX_MASS_W2=1|" "w2m5|HX_MASS_W2=1|w2m5" "w2m6|HX_MASS_W2=1|w2m6" "w2w8|HX_MASS_W2=1|w2w8"
HX_MASS_W2=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_mass_w2 -s 30 -c 1 -o $O/prof_w2 python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1; echo "ncu full rc=$?"
python tools/ncu_summary.py $O/sum_w2.md $O/prof_w2.ncu-rep > /dev/null 2>&1
python tools/ncu_lines.py $O/prof_w2.ncu-rep 30 > $O/lines_w2.txt 2>&1
