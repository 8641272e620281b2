"""Dev timing helper: FFMA peak probe + fused train step at config-2 shapes."""
import ctypes as C
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_2302_01838_b200 import LossWeights, ModelArch, _lib, init_stacked
from paper_2302_01838_b200.trainer import _synthetic_batch, launch_train

lib = _lib.load()
tf = C.c_float()
for it in (4096, 16384):
    _lib.check(lib.vm_ffma_peak(it, C.byref(tf), _lib.stream_ptr()), "ffma")
    print(f"ffma peak probe iters={it}: {tf.value:.1f} TFLOP/s")

ao, ab = ModelArch(hidden=32), ModelArch(hidden=128)
po, so = init_stacked(ao, 50, seed=0)
pb, sb = init_stacked(ab, 1, seed=0, stream=2)
bo = _synthetic_batch(ao, 50, 120, 10, seed=3)
bb = _synthetic_batch(ab, 1, 1200, 10, seed=4)
w = LossWeights()
for name, stacks in (("objects only", [(po, so, bo)]), ("bg only", [(pb, sb, bb)]),
                     ("objects+bg", [(po, so, bo), (pb, sb, bb)])):
    for _ in range(5):
        launch_train(stacks, w)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 50
    e0.record()
    for _ in range(n):
        launch_train(stacks, w)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / n
    flop = 0
    for p, s, b in stacks:
        h = p.arch.hidden
        per = 2 * (2 * (h * 33 + 2 * h * h + 4 * h) + (2 * h * h + 4 * h))
        flop += per * b.encoded.shape[0] * b.encoded.shape[1] * b.encoded.shape[2]
    print(f"{name}: {ms*1e3:.1f} us/step  {flop/ms/1e9:.2f} TFLOP/s algorithmic")
