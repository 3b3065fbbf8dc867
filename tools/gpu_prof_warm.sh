#!/bin/bash
# warm-cache ncu --set full captures of the CG kernels (as in the step graph: L2 holds the CG working set)
O=gpurun_out/${1:-warm}; mkdir -p $O; shift
for K in ${@:-k_mass_brick k_cg_node}; do
  timeout 600 ncu --set full --cache-control none --clock-control none --import-source on -k regex:$K -s 30 -c 1 -o /tmp/w_$K python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e > $O/ncu_$K.log 2>&1; echo "ncu $K rc=$?"
  python tools/ncu_summary.py $O/sum_$K.md /tmp/w_$K.ncu-rep > /dev/null 2>&1
  ncu -i /tmp/w_$K.ncu-rep --page raw --csv > $O/raw_$K.csv 2>/dev/null
  python tools/ncu_stalls.py $O/raw_$K.csv > $O/stalls_$K.txt 2>&1
  python tools/ncu_lines.py /tmp/w_$K.ncu-rep 40 > $O/lines_$K.txt 2>&1
  python tools/ncu_lines.py /tmp/w_$K.ncu-rep 40 ins > $O/ins_$K.txt 2>&1
  head -20 $O/sum_$K.md; cat $O/stalls_$K.txt
done
