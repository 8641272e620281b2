import sys, time
sys.path.insert(0, '.')
import torch
from paper_2302_01838_b200 import TrainConfig, ModelArch, init_stacked
from paper_2302_01838_b200.meshing import query_grid
from paper_2302_01838_b200.geometry import AABB
import numpy as np
p, s = init_stacked(ModelArch(hidden=128), 1, seed=0, stream=2)
box = AABB(np.array([-2., -2., -2.]), np.array([2., 2., 2.]))
for res in (64, 128, 256):
    for chunk in (1 << 21, 1 << 23):
        f = lambda: query_grid(p, 0, box, 8.0, res, chunk=chunk, as_tensor=True)
        f(); torch.cuda.synchronize()
        t0 = time.perf_counter(); f(); torch.cuda.synchronize()
        print(res, chunk, f"{(time.perf_counter()-t0)*1e3:.2f} ms")
