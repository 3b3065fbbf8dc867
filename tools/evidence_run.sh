set -x
mkdir -p gpurun_out/f3
(timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/f3/gpu_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/f3/gpu_tests.txt)
timeout 200 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f3/smoke.txt 2>&1
timeout 500 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/f3/bench.json 2> gpurun_out/f3/bench.err
timeout 500 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/f3/bench_repeat.json 2> gpurun_out/f3/bench_repeat.err
timeout 600 python bench.py --gpus 1 --steps 50 --warmup 10 > gpurun_out/f3/bench_steps50_warmup10.json 2> gpurun_out/f3/bench50.err
timeout 600 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/f3/reference_arm.json 2> gpurun_out/f3/reference_arm.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/f3/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/f3/ncu.log 2>&1
tail -2 gpurun_out/f3/gpu_tests.txt; tail -1 gpurun_out/f3/smoke.txt
for f in bench bench_repeat bench_steps50_warmup10 reference_arm; do python -c "
import json,sys;d=json.load(open('gpurun_out/f3/$f.json'));print('$f',d.get('value'),(d.get('e2e') or {}).get('value'),(d.get('api') or {}).get('value'),d.get('clocks'))"; done
