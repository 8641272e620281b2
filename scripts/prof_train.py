"""Profiling driver: a few fused train steps at config-2 shapes (objects and/or bg)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_2302_01838_b200 import LossWeights, ModelArch, init_stacked
from paper_2302_01838_b200.trainer import _synthetic_batch, launch_train

which = sys.argv[1] if len(sys.argv) > 1 else "both"
ao, ab = ModelArch(hidden=32), ModelArch(hidden=128)
stacks = []
if which in ("obj", "both"):
    po, so = init_stacked(ao, 50, seed=0)
    stacks.append((po, so, _synthetic_batch(ao, 50, 120, 10, seed=3)))
if which in ("bg", "both"):
    pb, sb = init_stacked(ab, 1, seed=0, stream=2)
    stacks.append((pb, sb, _synthetic_batch(ab, 1, 1200, 10, seed=4)))
for _ in range(4):
    launch_train(stacks, LossWeights())
torch.cuda.synchronize()
