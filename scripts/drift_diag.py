"""Drift diagnostics: GPU f32 vs reference-order f32 vs f64 truth, per step."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

from oracle import vobj_oracle as O
from paper_2302_01838_b200 import LossWeights, ModelArch, TrainConfig, init_stacked, train_on_batch
from paper_2302_01838_b200.mapper import Mapper
from paper_2302_01838_b200.scenes import config, populate
from paper_2302_01838_b200.trainer import RaySampleBatch, _synthetic_batch
from tests.helpers import host_layers, oracle_arch, oracle_mapstate


def flat_gpu(p):
    W, B = host_layers(p)
    k = p.count
    return np.concatenate([np.concatenate([W[l].reshape(k, -1), B[l]], 1) for l in range(len(W))], 1).astype(np.float64)


def flat_o(st):
    k = st.count
    return np.concatenate([np.concatenate([st.W[l][:k].reshape(k, -1), st.b[l][:k]], 1) for l in range(len(st.W))], 1).astype(np.float64)


def f64_copy(st):
    c = st.copy()
    for name in ("W", "b", "mW", "vW", "mb", "vb"):
        setattr(c, name, [a.astype(np.float64) for a in getattr(c, name)])
    return c


def report(tag, s, g, r, t):
    rl = lambda a, b: (np.linalg.norm(a - b, axis=1) / np.linalg.norm(b, axis=1)).max()
    print(f"{tag} step {s:2d}: max|gpu-ref| {np.abs(g-r).max():.2e}  relL2(gpu,ref) {rl(g,r):.2e}  "
          f"relL2(gpu,f64) {rl(g,t):.2e}  relL2(ref,f64) {rl(r,t):.2e}  "
          f"frac>tol {np.mean(np.abs(g-r) > 1e-5 + 1e-4*np.abs(r)):.4%}")


def synthetic(hidden, k, rays, steps):
    arch = ModelArch(hidden=hidden)
    p, s = init_stacked(arch, k, seed=11)
    o = O.new_stack(oracle_arch(arch), k, 11)
    t = f64_copy(o)
    b = _synthetic_batch(arch, k, rays, 10, seed=7)
    hb = {kk: getattr(b, kk).cpu().numpy() for kk in ("encoded", "t", "target_depth", "target_colour",
                                                       "target_mask", "valid_depth", "ray_ok")}
    hb64 = {kk: (v.astype(np.float64) if v.dtype == np.float32 else v) for kk, v in hb.items()}
    for i in range(steps):
        train_on_batch(p, s, b, LossWeights())
        O.train_on_batch(o, hb)
        O.train_on_batch(t, hb64)
        if i in (0, 4, 9, 19, 29, 49) or i == steps - 1:
            report(f"synthetic h{hidden} K{k} R{rays}", i + 1, flat_gpu(p), flat_o(o), flat_o(t))


def mapper_cfg1(steps):
    scene = config("1")
    cfg = TrainConfig(train_background=False)
    m = Mapper(scene["intrinsics"], cfg)
    populate(m, scene)
    ms = oracle_mapstate(scene, cfg)
    t = f64_copy(ms.obj)
    for i in range(steps):
        m.train_step()
        bs = [O.assemble_batch(inst, ms.intr, ms.obj.arch, ms.rays_object, ms.global_step, ms.seed, ms.sampling,
                               ms.bound_pad) for inst in ms.objects]
        hb = O.stack_batches(bs)
        O.train_on_batch(ms.obj, hb)
        O.train_on_batch(t, {kk: (v.astype(np.float64) if v.dtype == np.float32 else v) for kk, v in hb.items()})
        ms.global_step += 1
        if i in (0, 4, 9, 19, 29) or i == steps - 1:
            report("mapper cfg1 objects", i + 1, flat_gpu(m.obj_params), flat_o(ms.obj), flat_o(t))


mapper_cfg1(30)
synthetic(32, 5, 120, 30)
synthetic(128, 1, 300, 30)
