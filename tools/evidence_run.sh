set -x
mkdir -p gpurun_out/${EVID:-evid}
(timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${EVID:-evid}/gpu_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/${EVID:-evid}/gpu_tests.txt)
timeout 200 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${EVID:-evid}/smoke.txt 2>&1
timeout 500 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/${EVID:-evid}/bench.json 2> gpurun_out/${EVID:-evid}/bench.err
timeout 500 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/${EVID:-evid}/bench_repeat.json 2> gpurun_out/${EVID:-evid}/bench_repeat.err
timeout 600 python bench.py --gpus 1 --steps 50 --warmup 10 > gpurun_out/${EVID:-evid}/bench_steps50_warmup10.json 2> gpurun_out/${EVID:-evid}/bench50.err
timeout 600 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/${EVID:-evid}/reference_arm.json 2> gpurun_out/${EVID:-evid}/reference_arm.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${EVID:-evid}/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/${EVID:-evid}/ncu.log 2>&1
HX_BENCH_ONE_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --steps 3 --warmup 3 --elems 8 > gpurun_out/${EVID:-evid}/n2_one_gpu_functional.json 2> gpurun_out/${EVID:-evid}/n2.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_rates_pc -s 6 -c 1 -o gpurun_out/${EVID:-evid}/rates_full python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/${EVID:-evid}/ncu_full.log 2>&1
tail -2 gpurun_out/${EVID:-evid}/gpu_tests.txt; tail -c 300 gpurun_out/${EVID:-evid}/n2_one_gpu_functional.json; tail -1 gpurun_out/${EVID:-evid}/smoke.txt
for f in bench bench_repeat bench_steps50_warmup10 reference_arm; do python -c "
import json,sys;d=json.load(open('gpurun_out/${EVID:-evid}/$f.json'));print('$f',d.get('value'),(d.get('e2e') or {}).get('value'),(d.get('api') or {}).get('value'),d.get('clocks'))"; done
