"""cProfile of Mapper.process_frame (1200x680, 50 instances; the sweep's ingestion case)."""
import cProfile
import pstats
import sys
import time
sys.path.insert(0, '.')
import numpy as np
import torch
from paper_2302_01838_b200 import TrainConfig
from paper_2302_01838_b200.ingest import Frame
from paper_2302_01838_b200.mapper import Mapper
from paper_2302_01838_b200.scenes import make_scene

scene = make_scene(50, n_kf=5, seed=0)
g = np.random.default_rng(1)
H, W = 680, 1200
mask = np.zeros((H, W), np.int32)
for i in range(50):
    h, w = (int(x) for x in g.integers(40, 140, 2))
    v0, u0 = int(g.integers(0, H - h)), int(g.integers(0, W - w))
    mask[v0:v0 + h, u0:u0 + w] = i + 1
frames = [Frame(j, scene["rgb"], scene["depth"], mask, scene["background"]["keyframes"][j]["pose"]) for j in range(5)]
mi = Mapper(scene["intrinsics"], TrainConfig())
mi.process_frame(frames[0])
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
t0 = time.perf_counter()
for fr in frames[1:]:
    mi.process_frame(fr)
torch.cuda.synchronize()
pr.disable()
print(f"process_frame {(time.perf_counter() - t0) / 4 * 1e3:.1f} ms, objects {mi.obj_params.count}")
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
