"""Executed warp-instructions per source line: joins an ncu report's SASS
counts with the line table of the local build (same binary).
    python tools/sass_lines.py REPORT KERNEL_REGEX OBJ MANGLED [TOP]"""
import csv
import io
import os
import re
import subprocess
import sys
import tempfile

rep, kern, obj, sym = sys.argv[1:5]
top = int(sys.argv[5]) if len(sys.argv) > 5 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                      "-k", f"regex:{kern}"], capture_output=True, text=True).stdout
lines = out.splitlines()
start = [i for i, l in enumerate(lines) if l.startswith('"Address"')][0]
end = next((i for i in range(start + 1, len(lines)) if lines[i].startswith('"Kernel Name"')), len(lines))
rows = list(csv.DictReader(io.StringIO("\n".join(lines[start:end]))))
base = min(int(r["Address"], 16) for r in rows)
cnt = {int(r["Address"], 16) - base: int(r["Instructions Executed"] or 0) for r in rows}
stall = {int(r["Address"], 16) - base: int(r["Warp Stall Sampling (All Samples)"] or 0) for r in rows}
d = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=d, capture_output=True)
cub = [f for f in os.listdir(d) if f.endswith(".cubin")][0]
sass = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(d, cub)], capture_output=True, text=True).stdout
sec = sass.split(f".text.{sym}:")[1].split(".section")[0]
cur = "?"
per = {}
for l in sec.splitlines():
    m = re.search(r'File "([^"]+)", line (\d+)', l)
    if m:
        cur = f"{os.path.basename(m.group(1))}:{m.group(2)}"
        continue
    m = re.search(r"/\*([0-9a-f]{4,})\*/", l)
    if m:
        off = int(m.group(1), 16)
        c, s = per.get(cur, (0, 0))
        per[cur] = (c + cnt.get(off, 0), s + stall.get(off, 0))
tot = sum(c for c, _ in per.values())
print(f"total {tot} warp-instructions")
for k, (c, s) in sorted(per.items(), key=lambda t: -t[1][0])[:top]:
    print(f"{k:32s} {c:11d} {100 * c / max(tot, 1):6.2f}%  stalls {s}")
