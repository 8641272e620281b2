"""Where does the tensor-core (3xTF32) path stand numerically?  Runs the
two-stack scenario of tests/test_gpu_train.py::test_two_stacks_one_launch for
N steps and compares the background stack against the f32 oracle and an f64
run of the same algorithm (truth).  Run once with VM_TC=1 and once with VM_TC=0."""
import sys
sys.path.insert(0, '.')
import numpy as np
from oracle import vobj_oracle as O
from paper_2302_01838_b200 import LossWeights, ModelArch, init_stacked
from paper_2302_01838_b200.trainer import _synthetic_batch, launch_train
from tests.helpers import f64_stack, f64_batch, oracle_arch, to_host_batch, host_layers

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
ao, ab = ModelArch(hidden=32), ModelArch(hidden=128)
po, so = init_stacked(ao, 6, seed=0)
pb, sb = init_stacked(ab, 1, seed=0, stream=2)
ob = O.new_stack(oracle_arch(ab), 1, 0, stream=2)
tb = f64_stack(ob)
bo = _synthetic_batch(ao, 6, 120, 10, seed=3)
bb = _synthetic_batch(ab, 1, 1200, 10, seed=4)
hb = to_host_batch(bb)
hb64 = f64_batch(hb)
for _ in range(steps):
    launch_train([(po, so, bo), (pb, sb, bb)], LossWeights())
    O.train_on_batch(ob, hb)
    O.train_on_batch(tb, hb64)
W, B = host_layers(pb)
for l in range(len(W)):
    g, r, t = W[l][0].astype(np.float64), ob.W[l][0].astype(np.float64), tb.W[l][0]
    viol = np.abs(g - r) > (1e-5 + 1e-4 * np.abs(r))
    print(f"W{l}: max|gpu-ref| {np.abs(g-r).max():.2e}  max|gpu-f64| {np.abs(g-t).max():.2e}  "
          f"max|ref-f64| {np.abs(r-t).max():.2e}  violations(rtol1e-4,atol1e-5) {int(viol.sum())}  "
          f"relL2 gpu-f64 {np.linalg.norm(g-t)/np.linalg.norm(t):.2e} ref-f64 {np.linalg.norm(r-t)/np.linalg.norm(t):.2e}")
    if viol.any():
        for idx in np.argwhere(viol)[:4]:
            idx = tuple(idx)
            print(f"    {idx}: gpu {g[idx]:.7f} ref {r[idx]:.7f} f64 {t[idx]:.7f}")
