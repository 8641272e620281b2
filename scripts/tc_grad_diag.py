"""One training step of the two-stack scenario; compares the background
gradient (recovered from Adam's first moment m = (1 - b1) g) with the f64
oracle gradient, per layer, and prints where the largest errors sit."""
import sys
sys.path.insert(0, '.')
import numpy as np
from oracle import vobj_oracle as O
from paper_2302_01838_b200 import LossWeights, ModelArch, init_stacked
from paper_2302_01838_b200.trainer import _synthetic_batch, launch_train
from tests.helpers import f64_stack, f64_batch, oracle_arch, to_host_batch, host_state

rays = int(sys.argv[1]) if len(sys.argv) > 1 else 1200
ab = ModelArch(hidden=128)
pb, sb = init_stacked(ab, 1, seed=0, stream=2)
ob = f64_stack(O.new_stack(oracle_arch(ab), 1, 0, stream=2))
bb = _synthetic_batch(ab, 1, rays, 10, seed=4)
launch_train([(pb, sb, bb)], LossWeights())
O.train_on_batch(ob, f64_batch(to_host_batch(bb)))
mW, vW, mb, vb, step = host_state(sb, 1)
for l in range(4):
    g = mW[l][0].astype(np.float64) / 0.1
    t = ob.mW[l][0] / 0.1
    err = np.abs(g - t)
    scale = np.abs(t).max()
    print(f"W{l}: max err {err.max():.3e} (max|g| {scale:.3e}) relL2 {np.linalg.norm(g-t)/np.linalg.norm(t):.2e}")
    rows = err.max(axis=1)
    worst = np.argsort(-rows)[:5]
    print("   worst rows", [(int(r), f"{rows[r]:.2e}") for r in worst], " row-median", f"{np.median(rows):.2e}")
    cols = err.max(axis=0)
    wc = np.argsort(-cols)[:5]
    print("   worst cols", [(int(c), f"{cols[c]:.2e}") for c in wc])
    gb = mb[l][0].astype(np.float64) / 0.1
    tbb = ob.mb[l][0] / 0.1
    print(f"   b{l}: max err {np.abs(gb-tbb).max():.3e} (max|g| {np.abs(tbb).max():.3e})")
