"""Cost of one frame's map growth in the e2e loop (5 new keyframes)."""
import sys
import time
sys.path.insert(0, '.')
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
builds = [0]
orig = m._build_graphs
def counted():
    builds[0] += 1
    return orig()
m._build_graphs = counted
local = [m.instance_for_model(j) for j in range(m.obj_params.count)]
fid = 10 ** 6
for rep in range(6):
    fid += 1
    t0 = time.perf_counter()
    for j in range(5):
        inst = local[(fid * 5 + j) % len(local)]
        kf = inst.keyframes[0]
        m.add_keyframe(inst, fid, kf.pose, kf.bbox, kf.mask, scene["rgb"], scene["depth"])
    t1 = time.perf_counter()
    m._sync()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    m.train_step()
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    m.train_step()
    torch.cuda.synchronize()
    t4 = time.perf_counter()
    print(f"add_keyframe x5 {1e3*(t1-t0):.3f} ms  _sync {1e3*(t2-t1):.3f} ms  first step {1e3*(t3-t2):.3f} ms  "
          f"next step {1e3*(t4-t3):.3f} ms  graph builds {builds[0]}")
import cProfile
import pstats
pr = cProfile.Profile()
for rep in range(5):
    fid += 1
    for j in range(5):
        inst = local[(fid * 5 + j) % len(local)]
        kf = inst.keyframes[0]
        m.add_keyframe(inst, fid, kf.pose, kf.bbox, kf.mask, scene["rgb"], scene["depth"])
    pr.enable()
    m._sync()
    torch.cuda.synchronize()
    pr.disable()
    m.train_step()
pstats.Stats(pr).sort_stats("tottime").print_stats(14)
