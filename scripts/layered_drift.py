"""Drift of the layered path vs the f32 reference, both measured against an
f64 run of the same algorithm, per step and over seeds (is a gap chaotic
knife-edge noise or systematic?)."""
import sys

import numpy as np

sys.path.insert(0, ".")
from oracle import vobj_oracle as O  # noqa: E402
from paper_2302_01838_b200 import LossWeights, ModelArch, init_stacked, train_on_batch  # noqa: E402
from paper_2302_01838_b200.trainer import _synthetic_batch  # noqa: E402
from tests.helpers import f64_batch, f64_stack, flat_oracle, flat_params, oracle_arch, rel_l2, to_host_batch  # noqa: E402

for hidden, rays in ((1024, 120), (256, 64)):
    for seed in range(4):
        arch = ModelArch(n_layers=4, hidden=hidden, n_freq=5)
        p, s = init_stacked(arch, 1, seed=11 + seed)
        ost = O.new_stack(oracle_arch(arch), 1, 11 + seed)
        tru = f64_stack(ost)
        b = _synthetic_batch(arch, 1, rays, 10, seed=7 + seed)
        hb = to_host_batch(b)
        h64 = f64_batch(hb)
        row = []
        for step in range(5):
            train_on_batch(p, s, b, LossWeights())
            O.train_on_batch(ost, hb)
            O.train_on_batch(tru, h64)
            g, r, t = flat_params(p), flat_oracle(ost), flat_oracle(tru)
            row.append(f"{rel_l2(g, t).max():.1e}/{rel_l2(r, t).max():.1e}")
        print(f"h{hidden} seed {seed}: gpu/ref rel-L2 to f64 per step: " + "  ".join(row), flush=True)
