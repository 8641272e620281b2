"""Small eager map-update run for compute-sanitizer (memcheck / racecheck /
synccheck): config-1 scene, objects (KF32) + background (KT + partial reduce),
sampler (KS) and Adam, plus the generic FFMA kernel (VM_KF32=0 runs)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_2302_01838_b200 import TrainConfig
from paper_2302_01838_b200.mapper import Mapper
from paper_2302_01838_b200.scenes import config, populate

scene = config("1")
cfg = TrainConfig(rays_background=240)
m = Mapper(scene["intrinsics"], cfg, use_graphs=False)
populate(m, scene)
for _ in range(2):
    rep = m.train_step()
torch.cuda.synchronize()
print("ok", rep.step, len(rep.losses))
