"""Summarise an ncu source page (cuda lines): top lines by stall samples / instructions."""
import csv
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows, path, hdr = [], None, None
for rec in csv.reader(out.splitlines()):
    if not rec:
        continue
    if rec[0] == "File Path":
        path = rec[1].split("/")[-1]
        continue
    if rec[0] == "Function Name":
        continue
    if rec[0] == "Line No":
        hdr = rec
        continue
    if hdr is None or len(rec) < len(hdr) or not rec[0]:
        continue
    d = dict(zip(hdr, rec))
    try:
        samp = int(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
        inst = int(d.get("Instructions Executed", "0") or 0)
    except ValueError:
        continue
    rows.append((samp, inst, path, d["Line No"], d["Source"].strip()[:110]))
tot_s = sum(r[0] for r in rows) or 1
tot_i = sum(r[1] for r in rows) or 1
print(f"total samples {tot_s}  total warp-instructions {tot_i}")
for r in sorted(rows, reverse=True)[:n]:
    print(f"{100*r[0]/tot_s:5.1f}% smp {100*r[1]/tot_i:5.1f}% inst  {r[2]}:{r[3]}  {r[4]}")
