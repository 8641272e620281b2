"""Summarise an ncu --metrics gpu__time_duration.sum CSV log (our kernels only)."""
import csv
import sys
from collections import defaultdict

path = sys.argv[1]
lines = [l for l in open(path) if l.startswith('"')]
rows = list(csv.reader(lines))
h = rows[0]
ours = ("sample_", "encode_kernel", "mlp_kernel", "kf32", "reduce_partials", "adam_train", "adam_", "tc_train", "tc_prep")
agg = defaultdict(list)
for r in rows[1:]:
    d = dict(zip(h, r))
    name = d["Kernel Name"]
    if not any(o in name for o in ours):
        continue
    short = name.split("(")[0].replace("void ", "")[:70]
    agg[(short, d["Grid Size"], d["Block Size"])].append(float(d["Metric Value"]))
tot = sum(sum(v) for v in agg.values())
for (n, g, b), v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    print(f"{sum(v)/len(v)/1e3:9.1f} us x{len(v):3d}  {100*sum(v)/tot:5.1f}%  {n} grid{g} block{b}")
