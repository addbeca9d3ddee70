for v in t0 t1 t2 t3 t123 t0; do
  PGX_LIB=paper_2605_20816_b200/lib/var/$v.so timeout 300 python bench.py --config c2 --no-cpu-baseline --steps 20 --warmup 5 > gpurun_out/q.json 2>gpurun_out/q.err
  python -c "import json;d=json.loads(open('gpurun_out/q.json').read().strip().splitlines()[-1]);print('$v ms %.4f e2e %.4f' % (d['ms_per_step'], d['e2e']['ms_per_step']), d['roofline']['kernels_ms']['tail'])" 2>&1 | tail -1
done
