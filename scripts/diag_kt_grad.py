"""Step-0 background gradient accuracy (config 1): KT vs the f32 reference vs f64."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
from oracle import vobj_oracle as O
from paper_2302_01838_b200 import TrainConfig
from paper_2302_01838_b200.mapper import Mapper
from paper_2302_01838_b200.scenes import config, populate
from tests.helpers import oracle_mapstate, host_state, f64_stack, f64_batch

scene = config(sys.argv[1] if len(sys.argv) > 1 else "1"); cfg = TrainConfig()
m = Mapper(scene["intrinsics"], cfg, use_graphs=False); populate(m, scene)
ms = oracle_mapstate(scene, cfg)
b = O.stack_batches([O.assemble_batch(ms.background, ms.intr, ms.bg.arch, ms.rays_background, 0, ms.seed, ms.sampling, ms.bound_pad)])
t = f64_stack(ms.bg); r = ms.bg.copy()
O.train_on_batch(t, f64_batch(b)); O.train_on_batch(r, b)
m.train_step()
mw, vw, mb, vb, st = host_state(m.bg_state, 1)
for l in range(4):
    for nm, g, rr, tt in (("W", mw[l][0], r.mW[l][0], t.mW[l][0]), ("b", mb[l][0], r.mb[l][0], t.mb[l][0])):
        g, rr, tt = g.astype(np.float64) * 10, rr.astype(np.float64) * 10, tt * 10
        eg, er = np.abs(g - tt), np.abs(rr - tt)
        scale = np.abs(tt).max()
        rel_g = eg / (np.abs(tt) + 1e-30); rel_r = er / (np.abs(tt) + 1e-30)
        print(f"{nm}{l}: |g| max {scale:.3e}; gpu err/max|g|: max {eg.max()/scale:.2e} p99 {np.quantile(eg, .99)/scale:.2e}; "
              f"ref err/max|g|: max {er.max()/scale:.2e} p99 {np.quantile(er, .99)/scale:.2e}; rel err >1e-4: gpu {(rel_g > 1e-4).sum()} ref {(rel_r > 1e-4).sum()} of {g.size}")
