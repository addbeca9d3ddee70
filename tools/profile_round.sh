#!/bin/bash
# Round profiling recipe (run under gpurun): bench line, launch list, full-set
# capture of the dominant kernels; text summaries land in gpurun_out/.
set -u
OUT=gpurun_out
mkdir -p $OUT
CFG=${1:-c2}
PREC=${2:-fp64}
TAG=${3:-r01}
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 200 > $OUT/${TAG}_${CFG}_${PREC}_clocks.csv &
SMI=$!
timeout 900 python bench.py --config $CFG --precision $PREC > $OUT/${TAG}_${CFG}_${PREC}_bench.json 2> $OUT/${TAG}_${CFG}_${PREC}_bench.err
RC=$?
kill $SMI
echo "bench rc=$RC"
tail -c 3000 $OUT/${TAG}_${CFG}_${PREC}_bench.json
CMD="python bench.py --config $CFG --precision $PREC --steps 2 --warmup 1 --no-cpu-baseline"
$CMD > $OUT/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/${TAG}_${CFG}_${PREC}_launches.csv $CMD > $OUT/ncu_launch.log 2>&1
python tools/run_eval.py --config $CFG --precision $PREC --iters 2 > $OUT/plain2.log 2>&1 && \
ncu -f --set full --clock-control none --import-source on -k regex:"tc_sweep|tc_grad|tc_coeffs" -s 3 -c 3 \
    -o /tmp/prof_${TAG}_${CFG}_${PREC} python tools/run_eval.py --config $CFG --precision $PREC --iters 2 > $OUT/ncu_full.log 2>&1
python3 tools/ncu_summary.py /tmp/prof_${TAG}_${CFG}_${PREC}.ncu-rep > $OUT/${TAG}_${CFG}_${PREC}_ncu_summary.txt 2>&1
ncu -i /tmp/prof_${TAG}_${CFG}_${PREC}.ncu-rep --page raw --csv > /tmp/raw.csv 2>&1
grep -E "Kernel Name|dram__bytes_(read|write)\.sum|sm__pipe_tensor|sm__inst_executed_pipe_xu|gpu__time_duration\.sum|sm__throughput|launch__registers" /tmp/raw.csv | head -5 > /dev/null
python3 - <<PY > $OUT/${TAG}_${CFG}_${PREC}_ncu_raw_key.txt
import csv
rows = list(csv.reader(open("/tmp/raw.csv")))
hdr = rows[0]
keys = [k for k in hdr if ("issue_stalled" in k and k.endswith("per_issue_active.ratio")) or any(s in k for s in ("Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "sm__pipe_tensor_op", "sm__pipe_tensor_cycles_active.avg.pct", "sm__inst_executed_pipe_tmem", "sm__inst_executed_pipe_xu", "sm__pipe_fp64", "smsp__inst_executed.sum", "sm__warps_active.avg.pct_of_peak", "launch__registers_per_thread", "sm__throughput.avg.pct_of_peak"))]
idx = [hdr.index(k) for k in keys]
for r in rows[2:]:
    print(" | ".join(f"{hdr[i]}={r[i]}" for i in idx))
PY
for k in sweep grad; do python3 tools/sass_hot.py /tmp/prof_${TAG}_${CFG}_${PREC}.ncu-rep $k 30 > $OUT/${TAG}_${CFG}_${PREC}_sass_$k.txt 2>&1; done
cp /tmp/prof_${TAG}_${CFG}_${PREC}.ncu-rep $OUT/ 2>/dev/null
ls $OUT
# DRAM bytes per launch per kernel (bench.py reads the latest profiles/*_traffic.json)
python3 - "$OUT" "$TAG" "$CFG" "$PREC" <<'PY'
import csv, io, json, subprocess, sys
out_dir, tag, cfg, prec = sys.argv[1:5]
raw = subprocess.run(["ncu", "-i", f"/tmp/prof_{tag}_{cfg}_{prec}.ncu-rep", "--page", "raw", "--csv"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
res = {}
if len(rows) > 2:
    h, units = rows[0], rows[1]
    for r in rows[2:]:
        d, u = dict(zip(h, r)), dict(zip(h, units))
        kern = d["Kernel Name"].split("<")[0].replace("void ", "").replace("pgx::", "").replace("k_", "", 1)
        kern = {"tc_sweep": "tc_pass1", "tc_grad": "tc_pass2"}.get(kern, kern)  # bench.py's kernel names
        res[f"{cfg}_{prec}:{kern}"] = {
            "dram_bytes_read": float(d["dram__bytes_read.sum"]) * scale[u["dram__bytes_read.sum"]],
            "dram_bytes_write": float(d["dram__bytes_write.sum"]) * scale[u["dram__bytes_write.sum"]],
            "kernel": d["Kernel Name"], "duration": d["gpu__time_duration.sum"] + " " + u["gpu__time_duration.sum"]}
json.dump(res, open(f"{out_dir}/{tag}_{cfg}_{prec}_traffic.json", "w"), indent=1, sort_keys=True)
PY
