"""Secondary measurements (one JSON object on stdout), each next to the
reference's own CPU code on the same box where that finishes in seconds:

* fig6: train-only step time (trainer.py:609-642 `benchmark`, synthetic
  batches) for K objects x hidden h -- the paper's Fig. 6 axes;
* infer: query_grid (64^3 per object, 256^3 background) and render_view
  throughput (meshing.py:64-97, :485-579);
* ingest: process_frame on a 1200x680 frame with 50 instances
  (trainer.py:226-265).
usage: python scripts/bench_sweep.py [--quick]
"""
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2302_01838_b200 import TrainConfig  # noqa: E402
from paper_2302_01838_b200.trainer import benchmark  # noqa: E402

quick = "--quick" in sys.argv
out = {"device": torch.cuda.get_device_name(0)}
vobj = bench.import_reference_pkg()

# ---------------- Fig. 6: train-only ----------------
ks, hs = [1, 50, 200, 1000], [16, 32, 64, 128]
rows = benchmark(ks, hs, timed_steps=20 if quick else 50, warmup_steps=5, modes=("vectorised",))
fig6 = [{"k": r.k, "hidden": r.hidden, "ms": r.ms, "object_steps_per_s": r.k / (r.ms * 1e-3)} for r in rows]
if vobj is not None:
    from vobj.trainer import benchmark as ref_benchmark
    for r in ref_benchmark([1, 50, 200], [32, 128], timed_steps=2, warmup_steps=1, modes=("vectorised",)):
        for f in fig6:
            if f["k"] == r.k and f["hidden"] == r.hidden:
                f["reference_cpu_ms"] = r.ms
                f["speedup"] = r.ms / f["ms"]
out["fig6_train_only"] = fig6
out["fig6_paper_rtx3090_ms"] = {"k50": 5.11, "k200": 14.70, "note": "PAPER.md:489/504, vMAP vectorised, hidden 32"}

# ---------------- Fig. 6 (right): hidden widths beyond the fused kernels (layered path) ----------------
paper_h = {16: 5.34, 32: 5.31, 64: 6.63, 128: 9.37, 256: 18.53, 512: 44.73, 1024: 155.88}
cfg6 = TrainConfig()
wide = benchmark([50], [256, 512, 1024], timed_steps=5 if quick else 20, warmup_steps=3, modes=("vectorised",))
fig6h = []
for r in [x for x in rows if x.k == 50] + wide:
    arch = cfg6.arch_object
    d = 3 * arch.include_input + 6 * arch.n_freq
    h = r.hidden
    macs = d * h + (arch.n_layers - 2) * h * h + 4 * h  # per sample
    flop = 6.0 * cfg6.rays_per_object * cfg6.points_per_ray * macs * r.k  # forward + dW + dx
    fig6h.append({"k": r.k, "hidden": h, "ms": r.ms, "tflops": flop / (r.ms * 1e-3) / 1e12,
                  "paper_rtx3090_ms": paper_h.get(h), "path": "layered" if h > 128 else "fused"})
if vobj is not None:
    from vobj.trainer import benchmark as ref_benchmark
    for r in ref_benchmark([50], [256], timed_steps=1, warmup_steps=1, modes=("vectorised",)):
        for f in fig6h:
            if f["hidden"] == r.hidden:
                f["reference_cpu_ms"] = r.ms
                f["speedup"] = r.ms / f["ms"]
out["fig6_hidden_k50"] = fig6h
out["fig6_hidden_note"] = ("PAPER.md:550-556 (K unstated; K=50 here), R=120, S=10, 4 layers; tflops = "
                           "6 x samples x MACs per sample / step time (FP32 FFMA peak ~74)")

# ---------------- inference ----------------
from paper_2302_01838_b200.mapper import Mapper  # noqa: E402
from paper_2302_01838_b200.meshing import query_grid, render_view  # noqa: E402
from paper_2302_01838_b200.scenes import make_scene, populate  # noqa: E402

scene = make_scene(50, n_kf=5, seed=0)
cfg = TrainConfig()
m = Mapper(scene["intrinsics"], cfg)
populate(m, scene)
for _ in range(5):
    m.train_step()
torch.cuda.synchronize()


def timed(fn, n=3):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / n


inst = m.instance_for_model(0)
t_obj = timed(lambda: query_grid(m.obj_params, 0, inst.aabb.padded(0.1), inst.pe_scale, 64, as_tensor=True))
bg = m.map.background
t_bg = timed(lambda: query_grid(m.bg_params, bg.model_index, bg.aabb.padded(0.1), bg.pe_scale, 256, as_tensor=True),
             n=1)
pose = scene["background"]["keyframes"][0]["pose"]
t_view = timed(lambda: render_view(m.obj_params, m.bg_params, m.map, scene["intrinsics"], pose), n=1)
inf = {"query_grid_obj_64^3_ms": t_obj * 1e3, "query_grid_obj_points_per_s": 64 ** 3 / t_obj,
       "query_grid_bg_256^3_ms": t_bg * 1e3, "query_grid_bg_points_per_s": 256 ** 3 / t_bg,
       "render_view_1200x680_50_objects_ms": t_view * 1e3}
if vobj is not None:
    from vobj.meshing import query_grid as rq
    rm = bench.reference_mapper(vobj, scene, cfg)
    ri = rm.instance_for_model(0)
    t0 = time.perf_counter()
    rq(rm.obj_params, 0, ri.aabb.padded(0.1), ri.pe_scale, 64)
    inf["reference_cpu_query_grid_obj_64^3_ms"] = (time.perf_counter() - t0) * 1e3
    inf["query_grid_obj_speedup"] = inf["reference_cpu_query_grid_obj_64^3_ms"] / inf["query_grid_obj_64^3_ms"]
out["inference"] = inf

# ---------------- ingestion ----------------
from paper_2302_01838_b200.ingest import Frame  # noqa: E402

g = np.random.default_rng(1)
H, W = 680, 1200
mask = np.zeros((H, W), np.int32)
for i in range(50):
    h, w = (int(x) for x in g.integers(40, 140, 2))
    v0, u0 = int(g.integers(0, H - h)), int(g.integers(0, W - w))
    mask[v0:v0 + h, u0:u0 + w] = i + 1
frames = [Frame(j, scene["rgb"], scene["depth"], mask, scene["background"]["keyframes"][j]["pose"]) for j in range(5)]
mi = Mapper(scene["intrinsics"], cfg)
mi.process_frame(frames[0])
torch.cuda.synchronize()
t0 = time.perf_counter()
for fr in frames[1:]:
    mi.process_frame(fr)
torch.cuda.synchronize()
ing = {"process_frame_1200x680_50_instances_ms": (time.perf_counter() - t0) / 4 * 1e3,
       "objects_after": mi.obj_params.count}
if vobj is not None:
    from vobj.datasets import Frame as RF
    from vobj.render import CameraIntrinsics
    from vobj.trainer import Mapper as RM
    intr = scene["intrinsics"]
    rmi = RM(CameraIntrinsics(intr.fx, intr.fy, intr.cx, intr.cy, intr.width, intr.height))
    rfr = [RF(f.frame_id, f.rgb, f.depth, f.mask, f.pose) for f in frames]
    rmi.process_frame(rfr[0])
    t0 = time.perf_counter()
    for fr in rfr[1:]:
        rmi.process_frame(fr)
    ing["reference_cpu_process_frame_ms"] = (time.perf_counter() - t0) / 4 * 1e3
    ing["speedup"] = ing["reference_cpu_process_frame_ms"] / ing["process_frame_1200x680_50_instances_ms"]
    ing["same_objects"] = rmi.obj_params.count == mi.obj_params.count
out["ingest"] = ing
print(json.dumps(out))
