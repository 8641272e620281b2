"""Aggregate ncu warp-stall samples of one kernel by CUDA source line.

usage: python scripts/ncu_lines.py REPORT.ncu-rep OBJ.o KERNEL_MANGLED [top]
Maps each SASS instruction's offset in the ncu source page to the line info
nvdisasm -g prints for the same cubin (compile with -lineinfo)."""
import csv
import os
import re
import subprocess
import sys
import tempfile
from collections import Counter, defaultdict

rep, obj, kern = sys.argv[1:4]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()[1:]))
h = rows[0]
ix = {n: i for i, n in enumerate(h)}
data = [r for r in rows[1:] if r and r[0].startswith("0x")]
base = min(int(r[0], 16) for r in data)
samp = {int(r[0], 16) - base: int(r[ix["Warp Stall Sampling (All Samples)"]] or 0) for r in data}
stalls = [n for n in h if n.startswith("stall_") and "Not Issued" not in n]
sdet = {int(r[0], 16) - base: {n: int(r[ix[n]] or 0) for n in stalls} for r in data}
with tempfile.TemporaryDirectory() as d:
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=d, capture_output=True)
    cub = [f for f in os.listdir(d) if f.endswith(".cubin")][0]
    dis = subprocess.run(["nvdisasm", "-g", os.path.join(d, cub)], capture_output=True, text=True).stdout
lines = dis.splitlines()
cur, started = None, False
off2line = {}
for l in lines:
    if l.startswith(".text."):
        if started:
            break
        started = kern in l
        continue
    if not started:
        continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        cur = f"{m.group(1).split('/')[-1]}:{m.group(2)}"
        continue
    mo = re.search(r"/\*([0-9a-f]{4,})\*/", l)
    if mo and cur:
        off2line[int(mo.group(1), 16)] = cur
agg, det = Counter(), defaultdict(Counter)
for off, s in samp.items():
    ln = off2line.get(off, "?")
    agg[ln] += s
    for n, c in sdet[off].items():
        det[ln][n[6:]] += c
tot = sum(agg.values())
print(f"total samples {tot}")
for ln, s in agg.most_common(top):
    br = " ".join(f"{n}:{c}" for n, c in det[ln].most_common(3) if c)
    print(f"{100 * s / tot:5.1f}%  {ln:28s} {br}")
