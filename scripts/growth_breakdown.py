"""Wall-clock breakdown of one frame's map growth (5 new keyframes) in the
e2e loop, then a cProfile of the post-growth table rebuild (_sync)."""
import sys, time
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2302_01838_b200 import TrainConfig
from paper_2302_01838_b200.mapper import Mapper
from paper_2302_01838_b200.scenes import make_scene, populate
scene = make_scene(50, n_kf=5, seed=0)
m = Mapper(scene["intrinsics"], TrainConfig()); populate(m, scene)
for _ in range(5): m.train_step()
torch.cuda.synchronize()
local = [m.instance_for_model(j) for j in range(m.obj_params.count)]
fid = 10 ** 6; T = []
import paper_2302_01838_b200.keyframes as KF
for rep in range(30):
    fid += 1
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for j in range(5):
        inst = local[(fid * 5 + j) % len(local)]; kf = inst.keyframes[0]
        m.add_keyframe(inst, fid, kf.pose, kf.bbox, kf.mask, scene["rgb"], scene["depth"])
    t1 = time.perf_counter()
    m._sync(); t2 = time.perf_counter()
    torch.cuda.synchronize(); t3 = time.perf_counter()
    g = m._g; rebuilt = g is None or g.get("key") != m._graph_key()
    st = m.global_step
    m.enqueue_graph_step(st); t4 = time.perf_counter()
    torch.cuda.synchronize(); t5 = time.perf_counter()
    m.global_step += 1
    m.train_step(); t6 = time.perf_counter()
    T.append((t1-t0, t2-t1, t3-t2, t4-t3, t5-t4, t6-t5, rebuilt))
a = np.array([t[:6] for t in T]) * 1e3
print("add_kf x5 | _sync host | sync wait | enqueue(host) | step wait | next train_step  (median ms)")
print(np.round(np.median(a, axis=0), 3), "graph rebuilds:", sum(t[6] for t in T))
print("max", np.round(a.max(axis=0), 3))

import cProfile, pstats
pr = cProfile.Profile()
for rep in range(30):
    fid += 1
    for j in range(5):
        inst = local[(fid * 5 + j) % len(local)]; kf = inst.keyframes[0]
        m.add_keyframe(inst, fid, kf.pose, kf.bbox, kf.mask, scene["rgb"], scene["depth"])
    torch.cuda.synchronize()
    pr.enable(); m._sync(); pr.disable()
    m.train_step()
pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
