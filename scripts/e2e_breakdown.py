"""Where does the end-to-end Mapper.train_step time go (config 2)?"""
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
N = 200


def t(label, fn):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i in range(N):
        fn(i)
    torch.cuda.synchronize()
    print(f"{label:48s} {(time.perf_counter() - t0) / N * 1e6:8.1f} us")


s = torch.cuda.current_stream()
t("graph replay back to back (no host sync)", lambda i: (m.enqueue_graph_step(m.global_step), setattr(m, "global_step", m.global_step + 1)))
t("graph replay + stream sync", lambda i: (m.enqueue_graph_step(m.global_step), s.synchronize(), setattr(m, "global_step", m.global_step + 1)))
t("_graph_step (replay, sync, host views)", lambda i: (m._graph_step(m.global_step), setattr(m, "global_step", m.global_step + 1)))
t("train_step", lambda i: m.train_step())
t("train_step + invalidate every 10", lambda i: (m.invalidate() if i % 10 == 0 else None, m.train_step()))
t("invalidate + _sync (table rebuild)", lambda i: (m.invalidate(), m._sync()))
t("_graph_key()", lambda i: m._graph_key())
t("_sync() fast path", lambda i: m._sync())
