#!/bin/bash
# GPU check: full gpu test suite + default bench line
mkdir -p gpurun_out
TAG=${1:-chk}
timeout 1200 python -m pytest tests -m gpu -x -q ${PYTEST_ARGS:-} > gpurun_out/${TAG}_pytest.txt 2>&1
echo "pytest rc=$?"; tail -15 gpurun_out/${TAG}_pytest.txt
timeout 900 python bench.py ${BENCH_ARGS:-} > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
echo "bench rc=$?"; tail -c 1500 gpurun_out/${TAG}_bench.err
python - "$TAG" <<'PY'
import json, sys
tag = sys.argv[1]
try:
    d = json.loads(open(f"gpurun_out/{tag}_bench.json").read().strip().splitlines()[-1])
    r = d["roofline"]
    print("bench", d["config"]["workload"], d["config"]["precision"], "ms/step %.4f e2e %.4f" % (d["ms_per_step"], d["e2e"]["ms_per_step"]),
          "frac %.3f bound %s" % (r["frac"], r["bound"]), {k: round(v, 4) for k, v in r["kernels_ms"].items()},
          "modes", {k: round(v["ms_per_step"], 3) for k, v in d["modes"].items()},
          "cpu", d["cpu_baseline"] and {k: d["cpu_baseline"][k] for k in ("value", "cores", "cpu_model")},
          "cpu1", d["cpu_baseline"] and d["cpu_baseline"]["single_thread"]["value"],
          "fitcpu", d["cpu_baseline"] and d["cpu_baseline"]["fit_c1"], "fitgpu", d["fit_c1_gpu"], "clocks", d["clocks"])
except Exception as e:
    print("bench parse failed", e)
PY
