import sys, time
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2302_01838_b200 import TrainConfig
from paper_2302_01838_b200.mapper import Mapper
from paper_2302_01838_b200.scenes import make_scene, populate
import paper_2302_01838_b200.keyframes as K
scene = make_scene(50, n_kf=5, seed=0)
m = Mapper(scene["intrinsics"], TrainConfig())
populate(m, scene)
for _ in range(5): m.train_step()
torch.cuda.synchronize()
local = [m.instance_for_model(j) for j in range(m.obj_params.count)]
ar = m.arena
print("arena cap", ar.rgbd.shape[0], "used", ar.used)
fid = 10**6
for rep in range(4):
    fid += 1
    kfs = []
    for j in range(5):
        inst = local[(fid * 5 + j) % len(local)]
        kf = inst.keyframes[0]
        kfs.append(m.add_keyframe(inst, fid, kf.pose, kf.bbox, kf.mask, scene["rgb"], scene["depth"]))
    torch.cuda.synchronize()
    t0 = time.perf_counter(); ar.add_many(kfs); torch.cuda.synchronize(); t1 = time.perf_counter()
    m._sync(); torch.cuda.synchronize(); t2 = time.perf_counter()
    print(f"add_many {1e3*(t1-t0):.3f} ms (texels {sum(k.mask.size for k in kfs)}), rest of _sync {1e3*(t2-t1):.3f} ms")
    m.train_step()
# pieces of a _sync without keyframe changes but forced table change
t0 = time.perf_counter()
for _ in range(20):
    m._dev_tables[0][0].last = None
    m.invalidate(); m._sync()
torch.cuda.synchronize()
print("forced table reupload _sync", (time.perf_counter() - t0) / 20 * 1e3, "ms")
