O=gpurun_out/r2ae; mkdir -p $O
for spec in "cur|" "nt256|HX_LIB=paper_2112_07075_b200/lib_nt256.so"; do
  IFS='|' read -r lab envs <<< "$spec"
  for cfg in "q2|--p 2 --n 34" "tgv|--p 4 --n 17 --problem tgv"; do
    IFS='|' read -r cn args <<< "$cfg"
    env $envs timeout 400 python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e $args > $O/${lab}_$cn.json 2> $O/${lab}_$cn.err
    python -c "import json;d=json.load(open('$O/${lab}_$cn.json'));print('$lab $cn', round(d['value'],1), {k:round(v['avg_us'],1) for k,v in d['kernels'].items()})"
  done
done
