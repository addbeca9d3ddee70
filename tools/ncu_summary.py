"""Key per-kernel metrics from an ncu report:  python tools/ncu_summary.py REPORT [regex]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
args = ["ncu", "-i", rep, "--page", "details", "--csv"]
if len(sys.argv) > 2:
    args += ["-k", f"regex:{sys.argv[2]}"]
out = subprocess.run(args, capture_output=True, text=True).stdout
want = ["Duration", "Registers Per Thread", "Achieved Occupancy", "Theoretical Occupancy",
        "Executed Ipc Active", "Issue Slots Busy", "Eligible Warps Per Scheduler",
        "Warp Cycles Per Issued Instruction", "Waves Per SM", "Grid Size", "DRAM Throughput",
        "Compute (SM) Throughput", "L1/TEX Hit Rate", "L2 Hit Rate", "Block Limit Registers",
        "Block Limit Shared Mem", "Dynamic Shared Memory Per Block",
        "Static Shared Memory Per Block", "SM Frequency"]
seen = {}
for row in csv.DictReader(io.StringIO(out)):
    if row.get("Metric Name") in want:
        key = (row["ID"], row["Kernel Name"][:60])
        seen.setdefault(key, []).append(f'{row["Metric Name"]}={row["Metric Value"]}{row["Metric Unit"]}')
for (i, k), v in seen.items():
    print(f"[{i}] {k}\n    " + "\n    ".join(v))
