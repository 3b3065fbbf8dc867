#!/bin/bash
O=gpurun_out/r2k; mkdir -p $O
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_rates_pc -s 2 -c 1 -o $O/prof_rates python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1; echo "ncu rc=$?"
python tools/ncu_lines.py $O/prof_rates.ncu-rep 60 ins > $O/ins_rates.txt 2>&1
ls -la $O
