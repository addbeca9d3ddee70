#!/bin/bash
# A/B of programmatic dependent launch (PGX_PDL=0 / 1) on the bench configs
mkdir -p gpurun_out
for i in 1 2; do
for v in 0 1; do
  for cp in c2:tc c2:fp64 c5:tc; do
    c=${cp%%:*}; p=${cp##*:}
    PGX_PDL=$v timeout 300 python bench.py --config $c --precision $p --no-cpu-baseline --steps 20 --warmup 5 > gpurun_out/pdl$v.json 2>gpurun_out/pdl$v.err
    python -c "import json;d=json.loads(open('gpurun_out/pdl$v.json').read().strip().splitlines()[-1]);print('pdl=$v $c $p ms %.4f e2e %.4f' % (d['ms_per_step'], d['e2e']['ms_per_step']))"
  done
done; done
