#!/bin/bash
# one ncu --set full capture of a kernel (regex) from the bench, with per-line stall / bank-conflict lists
# usage: bash tools/gpu_prof1.sh OUTNAME KERNEL_REGEX SKIP [extra env assignments...]
O=gpurun_out/$1; K=$2; S=${3:-1}; mkdir -p $O
timeout 600 ncu --set full --clock-control none --import-source on -k regex:$K -s $S -c 1 -o /tmp/p_$1 python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e > $O/ncu.log 2>&1; echo "ncu rc=$?"
python tools/ncu_summary.py $O/sum.md /tmp/p_$1.ncu-rep > /dev/null 2>&1
python tools/ncu_lines.py /tmp/p_$1.ncu-rep 40 > $O/lines.txt 2>&1
python tools/ncu_lines.py /tmp/p_$1.ncu-rep 30 bank > $O/bank.txt 2>&1
python tools/ncu_lines.py /tmp/p_$1.ncu-rep 40 ins > $O/ins.txt 2>&1
ncu -i /tmp/p_$1.ncu-rep --page raw --csv > $O/raw.csv 2>/dev/null
cat $O/sum.md | head -30; head -25 $O/bank.txt
