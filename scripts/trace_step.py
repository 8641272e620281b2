"""Schedule of one config-2 step (VM_TRACE=1): when each FFMA work item (KF32)
and each KT tile ran, on which SM.
usage: VM_TRACE=1 python scripts/trace_step.py [env knobs as usual]"""
import ctypes as C
import os
import sys
sys.path.insert(0, '.')
import numpy as np
import torch
from paper_2302_01838_b200 import TrainConfig, _lib
from paper_2302_01838_b200.mapper import Mapper
from paper_2302_01838_b200.scenes import make_scene, populate

assert os.environ.get("VM_TRACE") == "1"
scene = make_scene(50, n_kf=5, seed=0)
m = Mapper(scene["intrinsics"], TrainConfig())
populate(m, scene)
for _ in range(5):
    m.train_step()
lib = _lib.load()
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
KIND = {1: "KF item", 2: "KT tile", 3: "reduce", 4: "Adam", 5: "sample prep", 6: "sample rays", 7: "loss sums", 8: "step init", 9: "step advance", 10: "ls staged", 11: "ls leaves"}
buf = (C.c_ulonglong * (4 << 16))()
n = C.c_int()
for rep in range(3):
    flush.fill_(rep)
    torch.cuda.synchronize()
    lib.vm_trace_read(buf, 1 << 16, C.byref(n))  # drop older records
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    m.enqueue_graph_step(m.global_step)
    e1.record()
    m.global_step += 1
    torch.cuda.synchronize()
    assert lib.vm_trace_read(buf, 1 << 16, C.byref(n)) == 0
    r = np.frombuffer(buf, dtype=np.uint64)[:4 * n.value].reshape(-1, 4).astype(np.int64)
    t0 = r[:, 2].min()
    r[:, 2:] -= t0
    kf, kt = r[r[:, 0] == 1], r[r[:, 0] == 2]
    print(f"--- step {rep}: graph {e0.elapsed_time(e1) * 1e3:.1f} us (events); records from the first CTA start (us):")
    for kd, name in KIND.items():
        q = r[r[:, 0] == kd]
        if len(q):
            print(f"  {name:12s} n={len(q):4d} start {q[:,2].min()/1e3:7.1f}..{q[:,2].max()/1e3:7.1f}"
                  f"  end {q[:,3].min()/1e3:7.1f}..{q[:,3].max()/1e3:7.1f}")
    if len(kf):
        d = (kf[:, 3] - kf[:, 2]) / 1e3
        print(f"  KF items: start {kf[:,2].min()/1e3:.1f}..{kf[:,2].max()/1e3:.1f}  end {kf[:,3].min()/1e3:.1f}..{kf[:,3].max()/1e3:.1f}"
              f"  duration med {np.median(d):.1f} min {d.min():.1f} max {d.max():.1f}  SMs {len(set(kf[:,1]))}")
    if len(kt):
        d = (kt[:, 3] - kt[:, 2]) / 1e3
        print(f"  KT tiles: start {kt[:,2].min()/1e3:.1f}..{kt[:,2].max()/1e3:.1f}  end {kt[:,3].min()/1e3:.1f}..{kt[:,3].max()/1e3:.1f}"
              f"  duration med {np.median(d):.1f} min {d.min():.1f} max {d.max():.1f}  SMs {len(set(kt[:,1]))}")
        st = np.sort(kt[:, 2]) / 1e3
        print("  KT start deciles:", [round(float(x), 1) for x in st[::10]])
    if len(kf):
        en = np.sort(kf[:, 3]) / 1e3
        print("  KF end deciles:", [round(float(x), 1) for x in en[::25]])
