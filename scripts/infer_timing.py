import sys, time
sys.path.insert(0, '.')
import torch
from paper_2302_01838_b200 import TrainConfig
from paper_2302_01838_b200.mapper import Mapper
from paper_2302_01838_b200.meshing import query_grid, render_view
from paper_2302_01838_b200.scenes import make_scene, populate
scene = make_scene(50, n_kf=5, seed=0)
m = Mapper(scene["intrinsics"], TrainConfig())
populate(m, scene)
for _ in range(5): m.train_step()
torch.cuda.synchronize()
bg = m.map.background
def timed(fn, n=2):
    fn(); torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(n): fn()
    torch.cuda.synchronize(); return (time.perf_counter() - t0) / n
g = lambda: query_grid(m.bg_params, bg.model_index, bg.aabb.padded(0.1), bg.pe_scale, 256, as_tensor=True)
print("bg 256^3 ms", timed(g) * 1e3)
pose = scene["background"]["keyframes"][0]["pose"]
print("render_view ms", timed(lambda: render_view(m.obj_params, m.bg_params, m.map, scene["intrinsics"], pose), 1) * 1e3)
a = query_grid(m.bg_params, bg.model_index, bg.aabb.padded(0.1), bg.pe_scale, 64, as_tensor=True)
print("grid mean", float(a.values.mean()), float(a.values.std()))
