"""Dev timing: the fused train step at config-2 shapes, per phase (CUDA events
inside vm_train_step: tag 1 = FFMA kernel KF, 2 = tensor-core branch KT,
3 = reduce + Adam).  usage: python scripts/kf_exp.py [obj|bg|both] [steps]"""
import ctypes as C
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_2302_01838_b200 import LossWeights, ModelArch, _lib, init_stacked
from paper_2302_01838_b200.trainer import _synthetic_batch, launch_train

class PointsBatch:
    """Config-2 style batch on the fused-PE (points) path the Mapper uses."""

    def __init__(self, enc_batch, scale):
        k, r, s, d = enc_batch.encoded.shape
        g = torch.Generator(device="cuda").manual_seed(1)
        self.b, self.d = enc_batch, d
        self.points = torch.rand((k, r, s, 3), device="cuda", generator=g) * 2 - 1
        self.pe_scale = torch.full((k,), scale, device="cuda")

    def vm(self):
        out = self.b.vm()
        out.encoded = None
        out.points = self.points.data_ptr()
        out.pe_scale = self.pe_scale.data_ptr()
        return out


which = sys.argv[1] if len(sys.argv) > 1 else "both"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
K = int(sys.argv[3]) if len(sys.argv) > 3 else 50
lib = _lib.load()
ao, ab = ModelArch(hidden=32), ModelArch(hidden=128)
stacks = []
if which in ("obj", "both"):
    po, so = init_stacked(ao, K, seed=0)
    stacks.append((po, so, PointsBatch(_synthetic_batch(ao, K, 120, 10, seed=3), 10.0)))
if which in ("bg", "both"):
    pb, sb = init_stacked(ab, 1, seed=0, stream=2)
    stacks.append((pb, sb, PointsBatch(_synthetic_batch(ab, 1, 1200, 10, seed=4), 15.0)))
w = LossWeights()
for _ in range(5):
    launch_train(stacks, w)
torch.cuda.synchronize()
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
tot = {1: 0.0, 2: 0.0, 3: 0.0, 0: 0.0}
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
wall = 0.0
for _ in range(n):
    flush.fill_(1.0)
    lib.vm_profile_enable(1)
    e0.record()
    launch_train(stacks, w)
    e1.record()
    torch.cuda.synchronize()
    wall += e0.elapsed_time(e1)
    for tag in tot:
        cnt, ms = C.c_int(), C.c_double()
        lib.vm_profile_read_tag(tag, C.byref(cnt), C.byref(ms))
        tot[tag] += ms.value
    lib.vm_profile_enable(0)
flop = 0
for p, s, b in stacks:
    h = p.arch.hidden
    per = 2 * (2 * (h * 33 + 2 * h * h + 4 * h) + (2 * h * h + 4 * h))
    flop += per * b.points.shape[0] * b.points.shape[1] * b.points.shape[2]
kf = tot[1] / n
print(f"{which} K={K}: step {wall / n * 1e3:.1f} us | KF {kf * 1e3:.1f} us | KT {tot[2] / n * 1e3:.1f} us | "
      f"reduce+adam {tot[3] / n * 1e3:.1f} us | MLP phase {tot[0] / n * 1e3:.1f} us")
if which == "obj":
    print(f"  KF algorithmic {flop / (kf * 1e-3) / 1e12:.2f} TFLOP/s")
