#!/bin/bash
# multi-rank functional checks on one B200: 2/4-process step-graph parity, torchrun 4 and 8 ranks
O=gpurun_out/r2r; mkdir -p $O
#timeout 900 python -m pytest tests/test_gpu_distributed.py -m gpu -q -p no:cacheprovider -k graph_step > $O/tests.txt 2>&1; tail -3 $O/tests.txt
for N in ${NS:-4 8}; do
  HX_BENCH_ONE_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus $N --steps 3 --warmup 3 --elems 8 --no-cpu > $O/bench_n$N.json 2> $O/bench_n$N.err
  echo "torchrun N=$N rc=$?"; tail -c 600 $O/bench_n$N.json; tail -3 $O/bench_n$N.err
done
