"""KT per-tile timeline (CTA 0) from a VM_TC_DEBUG build:
  REBUILD=vm_mlp.o scripts/build_variant.sh ktdbg -DVM_TC_DEBUG
  VM_LIB=scripts/bin/ktdbg/libvmap_b200.so python scripts/kt_timeline.py
Prints, in SM cycles from the CTA's start: compute-warp waits on the MMA
accumulator (before -> after), the MMA thread's per-chunk operand-ready and
weight-ready times, and the compute warps' slot acquisitions."""
import ctypes as C
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2302_01838_b200 import LossWeights, ModelArch, _lib, init_stacked  # noqa: E402
from paper_2302_01838_b200.trainer import _synthetic_batch, launch_train  # noqa: E402

lib = _lib.load()
ab = ModelArch(hidden=128)
pb, sb = init_stacked(ab, 1, seed=0, stream=2)
bb = _synthetic_batch(ab, 1, 1200, 10, seed=4)
for _ in range(3):
    launch_train([(pb, sb, bb)], LossWeights())
torch.cuda.synchronize()
buf = (C.c_int * 512)()
assert lib.vm_tc_debug_read(buf) == 0
d = np.frombuffer(buf, dtype=np.int32)
ev = d[96:96 + 64]
print("markers 26..30 (fwd end, out, render start, render end, bwd start):", list(d[96 + 26:96 + 31]))
print("wait_acc (before, after, stall):")
for i in range(0, 26, 2):
    if ev[i] or ev[i + 1]:
        print(f"  acc#{i // 2:2d} {ev[i]:8d} {ev[i + 1]:8d} {ev[i + 1] - ev[i]:7d}")
print("last bwd marker", ev[31:40])
full = d[320:384]
wr = d[256:320]
acq = d[384:448]
print("chunk: operands-ready, weights-ready(+issue), compute-acquire")
for j in range(64):
    if full[j] or wr[j] or acq[j]:
        print(f"  {j:2d} {full[j]:8d} {wr[j]:8d} {acq[j]:8d}")
