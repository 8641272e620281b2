"""Warm-cache CUDA-event timing of the fused train kernel for objects-only,
background-only and both stacks (config-2 shapes)."""
import ctypes as C
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_2302_01838_b200 import LossWeights, ModelArch, _lib, init_stacked
from paper_2302_01838_b200.trainer import _synthetic_batch, launch_train

lib = _lib.load()
ao, ab = ModelArch(hidden=32), ModelArch(hidden=128)
po, so = init_stacked(ao, 50, seed=0)
pb, sb = init_stacked(ab, 1, seed=0, stream=2)
bo = _synthetic_batch(ao, 50, 120, 10, seed=3)
bb = _synthetic_batch(ab, 1, 1200, 10, seed=4)
w = LossWeights()
for name, stacks in (("objects", [(po, so, bo)]), ("background", [(pb, sb, bb)]),
                     ("both", [(po, so, bo), (pb, sb, bb)])):
    for _ in range(3):
        launch_train(stacks, w)
    torch.cuda.synchronize()
    lib.vm_profile_enable(1)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        launch_train(stacks, w)
    e1.record()
    torch.cuda.synchronize()
    n, ms = C.c_int(), C.c_double()
    lib.vm_profile_read(C.byref(n), C.byref(ms))
    lib.vm_profile_enable(0)
    vs = (_lib.VmStack * len(stacks))(*[__import__("paper_2302_01838_b200.models", fromlist=["vm_stack"]).vm_stack(p, s) for p, s, _ in stacks])
    vb = (_lib.VmBatch * len(stacks))(*[b.vm() for _, _, b in stacks])
    ctas, smem = C.c_int(), C.c_int()
    lib.vm_train_grid(vs, vb, len(stacks), C.byref(ctas), C.byref(smem))
    print(f"{name:10s}: step {e0.elapsed_time(e1)/20*1e3:7.1f} us   fused kernel {ms.value/n.value*1e3:7.1f} us"
          f"   ctas {ctas.value} smem {smem.value}")
