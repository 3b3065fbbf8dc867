#!/bin/bash
O=gpurun_out/r2g; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py -q -x -p no:cacheprovider > $O/tests.txt 2>&1; tail -3 $O/tests.txt
bash tools/gpu_ab2.sh $O "base||" "norow|HX_NODE_ROW=0|" "notma|HX_MASS_TMA=0|" "old|HX_MASS_TMA=0 HX_NODE_ROW=0|" "e6||e6" "e8n96||e8n96" "g4||g4" "nm4||nm4"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_cg_node_row -s 30 -c 1 -o $O/prof_node_row python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1; echo "ncu full rc=$?"
python tools/ncu_summary.py $O/sum_node_row.md $O/prof_node_row.ncu-rep > /dev/null 2>&1
python tools/ncu_lines.py $O/prof_node_row.ncu-rep 30 > $O/lines_node_row.txt 2>&1
