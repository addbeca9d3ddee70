"""Summarise the hottest SASS of an ncu report: instructions by executed count
and stall samples.   python tools/sass_hot.py REPORT.ncu-rep KERNEL_REGEX [TOP]"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 60
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                      "-k", f"regex:{kern}"], capture_output=True, text=True).stdout
lines = out.splitlines()
# first kernel block only
start = [i for i, l in enumerate(lines) if l.startswith('"Address"')][0]
end = next((i for i in range(start + 1, len(lines)) if lines[i].startswith('"Kernel Name"')), len(lines))
rows = list(csv.DictReader(io.StringIO("\n".join(lines[start:end]))))
tot = sum(int(r["Instructions Executed"] or 0) for r in rows)
samples = sum(int(r["Warp Stall Sampling (All Samples)"] or 0) for r in rows)
print(f"total warp-instructions {tot}, stall samples {samples}")
mix = {}
for r in rows:
    op = r["Source"].split()[0] if r["Source"].split() else "?"
    if op.startswith("@"):
        op = r["Source"].split()[1]
    op = op.split(".")[0]
    mix[op] = mix.get(op, 0) + int(r["Instructions Executed"] or 0)
for op, n in sorted(mix.items(), key=lambda t: -t[1])[:25]:
    print(f"{op:12s} {n:12d} {100 * n / tot:6.2f}%")
print("--- hottest instructions")
rows.sort(key=lambda r: -int(r["Instructions Executed"] or 0))
for r in rows[:top]:
    print(f'{r["Address"][-5:]} {int(r["Instructions Executed"]):10d} {r["Warp Stall Sampling (All Samples)"]:>6s}  {r["Source"].strip()[:90]}')
print("--- most stalled instructions")
rows.sort(key=lambda r: -int(r["Warp Stall Sampling (All Samples)"] or 0))
for r in rows[:25]:
    print(f'{r["Address"][-5:]} {int(r["Instructions Executed"]):10d} {r["Warp Stall Sampling (All Samples)"]:>6s}  {r["Source"].strip()[:90]}')
