#!/bin/bash
# round-2 first lease: GPU tests, smoke, the driver's exact bench commands, the reference arm
mkdir -p gpurun_out/r2a
O=gpurun_out/r2a
timeout 1200 python -m pytest tests -m gpu -q -x > $O/tests.txt 2>&1; tail -1 $O/tests.txt
python -c 'import __graft_entry__ as g; g.smoke()' > $O/smoke.txt 2>&1; tail -1 $O/smoke.txt
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > $O/bench_20_5.json 2> $O/bench_20_5.err; echo "bench 20/5 rc=$?"; tail -3 $O/bench_20_5.err
timeout 900 python bench.py --gpus 1 --steps 50 --warmup 10 > $O/bench_50_10.json 2> $O/bench_50_10.err; echo "bench 50/10 rc=$?"; tail -3 $O/bench_50_10.err
timeout 900 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > $O/ref_20_5.json 2> $O/ref_20_5.err; echo "ref rc=$?"; tail -3 $O/ref_20_5.err
nproc > $O/nproc.txt; lscpu > $O/lscpu.txt
for f in $O/*.json; do echo $f; cut -c1-400 $f; done
