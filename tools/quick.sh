#!/bin/bash
# Quick GPU iteration: parity tests (optionally filtered) + short benches.
#   bash tools/quick.sh "<pytest -k expr>" "c5:tc c2:tc"
mkdir -p gpurun_out
K=${1:-}
BENCHES=${2:-"c5:tc"}
if [ -n "$K" ]; then
  timeout 600 python -m pytest tests -m gpu -x -q -k "$K" 2>&1 | tail -15
fi
for cb in $BENCHES; do
  cfg=${cb%%:*}; prec=${cb##*:}
  timeout 300 python bench.py --config $cfg --precision $prec --no-cpu-baseline --also "" --steps 10 --warmup 3 > gpurun_out/q_${cfg}_${prec}.json 2> gpurun_out/q_${cfg}_${prec}.err
  python - "$cfg" "$prec" <<'PY'
import json, sys
cfg, prec = sys.argv[1:3]
try:
    d = json.loads(open(f"gpurun_out/q_{cfg}_{prec}.json").read().strip().splitlines()[-1])
    r = d["roofline"]
    print(cfg, prec, "ms/step %.4f e2e %.4f" % (d["ms_per_step"], d["e2e"]["ms_per_step"]), {k: round(v, 4) for k, v in r["kernels_ms"].items()}, "frac %.3f bound %s" % (r["frac"], r["bound"]), "phi", d["result"]["phi"])
except Exception as e:
    print(cfg, prec, "FAILED", e); print(open(f"gpurun_out/q_{cfg}_{prec}.err").read()[-3000:])
PY
done
