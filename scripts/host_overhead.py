"""Where does Mapper.train_step spend host time (config 2)?  cProfile over
100 graph-replayed steps; prints the top functions by cumulative time."""
import cProfile
import pstats
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
t0 = time.perf_counter()
for _ in range(100):
    m.train_step()
dt = (time.perf_counter() - t0) / 100
print(f"train_step wall {dt*1e6:.1f} us")
pr = cProfile.Profile()
pr.enable()
for _ in range(100):
    m.train_step()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)

# with the bench's frame cadence: tables rebuilt every steps_per_frame steps
torch.cuda.synchronize()
t0 = time.perf_counter()
for i in range(100):
    if i % 10 == 0:
        m.invalidate()
    m.train_step()
torch.cuda.synchronize()
print(f"train_step wall with invalidate/10: {(time.perf_counter() - t0) / 100 * 1e6:.1f} us")
t0 = time.perf_counter()
for _ in range(20):
    m.invalidate()
    m._sync()
print(f"_sync (table rebuild + upload) {(time.perf_counter() - t0) / 20 * 1e6:.1f} us")
pr = cProfile.Profile()
pr.enable()
for _ in range(20):
    m.invalidate()
    m._sync()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(8)
