timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for c in c2 c4 c5; do timeout 300 python tools/ktime.py $c tc 5; done
for cp in c2:tc c2:fp64; do
  c=${cp%%:*}; p=${cp##*:}
  for i in 1 2; do
  timeout 300 python bench.py --config $c --precision $p --no-cpu-baseline --steps 20 --warmup 5 > gpurun_out/q.json 2>gpurun_out/q.err
  python -c "import json;d=json.loads(open('gpurun_out/q.json').read().strip().splitlines()[-1]);print('$c $p ms %.4f e2e %.4f launches %d' % (d['ms_per_step'], d['e2e']['ms_per_step'], d['gpu_launches']))"
  done
done
