"""Write profiles/<tag>_summary.md (+ traffic.json) from ncu reports in gpurun_out/."""
import csv
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
out = ROOT / "profiles"
out.mkdir(exist_ok=True)
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "smsp__sass_thread_inst_executed_op_ffma_pred_on.sum.per_cycle_elapsed",
        "sm__sass_thread_inst_executed_op_ffma_pred_on.sum.peak_sustained",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smsp__sass_inst_executed_op_shared_ld.sum",
        "smsp__inst_executed.sum", "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic",
        "launch__grid_size", "launch__block_size", "lts__t_sector_hit_rate.pct",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_uniform.avg.pct_of_peak_sustained_active"]


def raw(rep, launch=0):
    txt = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    hdr, units, vals = rows[0], rows[1], rows[2 + launch]
    return {k: (v, u) for k, u, v in zip(hdr, units, vals)}


def stalls(d):
    st = [(float(v.replace(",", "")), k) for k, (v, u) in d.items()
          if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")]
    tot = sum(v for v, _ in st) or 1
    return [(k[33:], 100 * v / tot) for v, k in sorted(st, reverse=True)[:8]]


lines = [f"# ncu summary ({tag})", "",
         "Captured with `ncu --set full --clock-control none --import-source on` on one B200 under gpurun,",
         "command `python bench.py --steps 2 --warmup 3 --no-cpu-baseline` (config 2), one launch per kernel",
         "(KT and KF normally run concurrently on two streams; ncu serialises them).",
         "ncu flushes caches before each replay: durations are cold-cache and serialised.", ""]
traffic = {}
for name, rep, launch in (("tensor-core MLP train (KT, tc_train_kernel, hidden-128 background)", "prof_tc", 0),
                          ("FFMA MLP train (KF32, kf32_train_kernel, hidden-32 objects)", "prof_kf32", 0),
                          ("FFMA MLP train (KF, mlp_kernel, generic)", "prof_mlp", 0),
                          ("opt-in tensor path for the objects (KH32, kh32_train_kernel, 3xTF32 mma.sync)",
                           "prof_kh32", 0),
                          ("partial-gradient reduce (reduce_partials_kernel)", "prof_red", 0),
                          ("sampler prep, objects (KS, sample_prep_kernel grid 50)", "prof_prep", 0),
                          ("sampler prep, background (KS, sample_prep_kernel grid 1)", "prof_prep", 1),
                          ("sampler rays (KS)", "prof_rays", 0), ("Adam (KA)", "prof_adam", 0)):
    p = ROOT / "gpurun_out" / f"{rep}.ncu-rep"
    if not p.exists():
        continue
    try:
        d = raw(p, launch)
    except IndexError:
        continue
    lines += [f"## {name}", "", "| metric | value | unit |", "|---|---|---|"]
    for k in KEYS:
        if k in d:
            lines.append(f"| {k} | {d[k][0]} | {d[k][1]} |")
    lines += ["", "Top warp stall reasons (share of samples): " +
              ", ".join(f"{k} {v:.1f}%" for k, v in stalls(d)), ""]
    mb = lambda k: float(d[k][0].replace(",", "")) * (1e9 if d[k][1] == "Gbyte" else 1e6 if d[k][1] == "Mbyte"
                                                      else 1e3 if d[k][1] == "Kbyte" else 1)
    if rep in ("prof_kf32", "prof_tc"):
        key = "mlp_kernel_dram_bytes_per_launch" if rep == "prof_kf32" else "tc_train_kernel_dram_bytes_per_launch"
        traffic[key] = mb("dram__bytes_read.sum") + mb("dram__bytes_write.sum")
        traffic["source"] = f"profiles/{tag}_summary.md (ncu --set full, cold cache)"
summ = ROOT / "gpurun_out" / f"{tag}_launches.txt"
if summ.exists():
    lines += ["## Launch list (ncu --metrics gpu__time_duration.sum, per-step kernels)", "", "```",
              summ.read_text().rstrip(), "```", ""]
(out / f"{tag}_summary.md").write_text("\n".join(lines) + "\n")
if traffic:
    (out / "traffic.json").write_text(json.dumps(traffic, indent=1) + "\n")
print("\n".join(lines))
