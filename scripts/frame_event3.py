"""Fine-grained cost of one frame event (5 new keyframes) in the e2e loop."""
import sys
import time
sys.path.insert(0, '.')
import cProfile
import pstats
import torch
from paper_2302_01838_b200 import TrainConfig
from paper_2302_01838_b200.mapper import Mapper
from paper_2302_01838_b200.scenes import make_scene, populate

scene = make_scene(50, n_kf=5, seed=0)
m = Mapper(scene["intrinsics"], TrainConfig())
populate(m, scene)
for _ in range(5):
    m.train_step()
torch.cuda.synchronize()
local = [m.instance_for_model(j) for j in range(m.obj_params.count)]
fid = 10 ** 6
pr = cProfile.Profile()
T = []
for rep in range(20):
    fid += 1
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    pr.enable()
    for j in range(5):
        inst = local[(fid * 5 + j) % len(local)]
        kf = inst.keyframes[0]
        m.add_keyframe(inst, fid, kf.pose, kf.bbox, kf.mask, scene["rgb"], scene["depth"])
    t1 = time.perf_counter()
    m.train_step()
    t2 = time.perf_counter()
    pr.disable()
    m.train_step()
    t3 = time.perf_counter()
    T.append((t1 - t0, t2 - t1, t3 - t2))
import numpy as np
a = np.median(np.array(T), axis=0) * 1e3
print(f"add_keyframe x5 {a[0]:.3f} ms, train_step after growth {a[1]:.3f} ms, next train_step {a[2]:.3f} ms")
pstats.Stats(pr).sort_stats("tottime").print_stats(22)
