"""Executed-instruction mix of one kernel by CUDA source line (ncu source page
+ nvdisasm -g line info).  usage: python scripts/ncu_mix.py REP OBJ KERNEL [top]"""
import csv, collections, os, re, subprocess, sys, tempfile
rep, obj, kern = sys.argv[1:4]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
for i, r in enumerate(rows):
    if "Source" in r and "Address" in r:
        h, start = r, i + 1
        break
ix = {n: i for i, n in enumerate(h)}
data = [r for r in rows[start:] if len(r) == len(h) and r[0].startswith("0x")]
base = min(int(r[0], 16) for r in data)
with tempfile.TemporaryDirectory() as d:
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=d, capture_output=True)
    cub = [f for f in os.listdir(d) if f.endswith(".cubin")][0]
    dis = subprocess.run(["nvdisasm", "-g", os.path.join(d, cub)], capture_output=True, text=True).stdout
cur, started, off2line = None, False, {}
for l in dis.splitlines():
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
byline = collections.defaultdict(collections.Counter)
tot = 0
for r in data:
    src = r[ix["Source"]].strip().split()
    if not src:
        continue
    op = src[1] if src[0].startswith("@") else src[0]
    op = op.split(".")[0]
    n = int(float(r[ix["Instructions Executed"]] or 0))
    byline[off2line.get(int(r[0], 16) - base, "?")][op] += n
    tot += n
lines = sorted(byline.items(), key=lambda kv: -sum(kv[1].values()))
print(f"total warp instructions {tot}")
for ln, c in lines[:top]:
    s = sum(c.values())
    print(f"{100 * s / tot:5.1f}%  {ln:26s} " + " ".join(f"{o}:{n // 1000}k" for o, n in c.most_common(5)))
