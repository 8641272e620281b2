"""Step 1 from the Mapper's own state: oracle step from the GPU state vs the GPU step."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
from oracle import vobj_oracle as O
from paper_2302_01838_b200 import TrainConfig
from paper_2302_01838_b200.mapper import Mapper
from paper_2302_01838_b200.scenes import config, populate
from tests.helpers import oracle_mapstate, host_state, host_layers, flat_params, flat_oracle, rel_l2

scene = config("2"); cfg = TrainConfig(train_background=False)
m = Mapper(scene["intrinsics"], cfg, use_graphs=False); populate(m, scene)
ms = oracle_mapstate(scene, cfg)
m.train_step(); O.map_update_step(ms)
# oracle stack loaded with the GPU state
g = ms.obj.copy()
W, B = host_layers(m.obj_params); mw, vw, mb, vb, st = host_state(m.obj_state, 50)
for l in range(4):
    g.W[l][:50], g.b[l][:50], g.mW[l][:50], g.vW[l][:50], g.mb[l][:50], g.vb[l][:50] = W[l], B[l], mw[l], vw[l], mb[l], vb[l]
g.step[:50] = st
bs = [O.assemble_batch(inst, ms.intr, ms.obj.arch, ms.rays_object, 1, ms.seed, ms.sampling, ms.bound_pad) for inst in ms.objects]
b = O.stack_batches(bs)
O.train_on_batch(g, b)
m.train_step(); O.map_update_step(ms)
e_gg = rel_l2(flat_params(m.obj_params), flat_oracle(g)); e_gr = rel_l2(flat_params(m.obj_params), flat_oracle(ms.obj))
e_rr = rel_l2(flat_oracle(g), flat_oracle(ms.obj))
print(f"GPU step vs oracle step from the GPU state: {e_gg.max():.2e} (obj {e_gg.argmax()}); GPU vs oracle trajectory {e_gr.max():.2e} (obj {e_gr.argmax()}); "
      f"oracle-from-GPU-state vs oracle trajectory {e_rr.max():.2e} (obj {e_rr.argmax()})")
k = 20
for l in range(4):
    d = np.abs(g.W[l][k] - ms.obj.W[l][k]); i = np.unravel_index(d.argmax(), d.shape)
    print(f"obj20 W{l}: oracle(GPU state) vs oracle max |d| {d.max():.2e} at {i}; m0 gpu {mw[l][k][i]:.3e} ref_m0 ?")
