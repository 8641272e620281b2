"""Top SASS instructions by warp-stall samples from an ncu report (source page)."""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()[1:]))
h = rows[0]
idx = {n: i for i, n in enumerate(h)}
stalls = [n for n in h if n.startswith("stall_") and "Not Issued" not in n]
data = rows[1:]
tot = sum(int(r[idx["Warp Stall Sampling (All Samples)"]] or 0) for r in data)
print(f"total samples {tot}")
order = sorted(range(len(data)), key=lambda i: -int(data[i][idx["Warp Stall Sampling (All Samples)"]] or 0))
for i in order[:top]:
    r = data[i]
    s = int(r[idx["Warp Stall Sampling (All Samples)"]] or 0)
    br = sorted(((int(r[idx[n]] or 0), n[6:]) for n in stalls), reverse=True)[:3]
    print(f"{i:5d} {100*s/tot:5.1f}%  {r[idx['Source']].strip()[:60]:60s} {' '.join(f'{n}:{c}' for c, n in br if c)}")
