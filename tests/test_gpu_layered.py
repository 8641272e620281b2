"""GPU parity of the layered path (vm_layered.cu): the architectures and
batches the fused kernels do not take -- hidden widths above 128 (PAPER.md
Fig. 6 sweeps hidden sizes up to 1024), encodings wider than 40, layer counts
without a fused instantiation, more than 32 samples per ray -- against the
oracle's train_on_batch (trainer.py:480-506).

Contract: losses within rtol 1e-4 of the oracle at every step; one step's
gradient within relative L2 1e-5 (per layer) of an f64 run of the same
algorithm; parameters after N = 5 steps within per-object relative L2 1e-4 of
the oracle, or else at least as close to the f64 run as the f32 reference
itself (within 2x).
Per-component bands are not used here: with 10^4-10^5 parameters per model a
few components whose gradient is ~0 (Adam divides by its magnitude) leave
any rtol band for two f32 summation orders (measured on a B200: 1 of 8192 at
hidden 64, 1 of 131072 at hidden 256), while the models as a whole agree to
~1e-6.
"""

import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest
import torch

from oracle import vobj_oracle as O
from paper_2302_01838_b200 import LossWeights, ModelArch, init_stacked, train_on_batch
from paper_2302_01838_b200.models import backward, forward
from paper_2302_01838_b200.trainer import _synthetic_batch, launch_train, train_on_batch_sequential

from .helpers import (assert_as_close_to_truth, assert_params_close, assert_params_rel_l2, f64_batch, f64_stack,
                      flat_oracle, flat_params, oracle_arch, rel_l2, to_host_batch)

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("hidden,n_layers,n_freq,k,rays,points", [
    (256, 4, 5, 2, 64, 10),   # wide hidden (the paper's sweep)
    (200, 3, 5, 2, 40, 7),    # width not a multiple of 32 (padded arena rows)
    (1024, 4, 5, 1, 120, 10), # the widest Fig. 6 model
    (32, 6, 5, 2, 50, 10),    # six layers: no fused instantiation
    (32, 4, 8, 2, 40, 10),    # 51-wide encoding (> 40)
    (64, 4, 5, 2, 30, 40),    # 40 samples per ray (> 32)
])
def test_layered_train_vs_oracle(cuda, hidden, n_layers, n_freq, k, rays, points):
    arch = ModelArch(n_layers=n_layers, hidden=hidden, n_freq=n_freq)
    params, state = init_stacked(arch, k, seed=11)
    ost = O.new_stack(oracle_arch(arch), k, 11)
    truth = f64_stack(ost)
    batch = _synthetic_batch(arch, k, rays, points, seed=7)
    hb = to_host_batch(batch)
    hb64 = f64_batch(hb)
    w = LossWeights()
    # hidden 1024 on 1200 samples: both f32 trajectories leave the f64 one
    # chaotically after ~2 steps (profiles/r02i_layered_drift.txt), so the
    # trajectory is compared over 2 steps there (N = 5 elsewhere)
    for step in range(2 if hidden >= 1024 else 5):
        ld, lc, lo = train_on_batch(params, state, batch, w)
        ed, ec, eo = O.train_on_batch(ost, hb)
        O.train_on_batch(truth, hb64)
        np.testing.assert_allclose(ld, ed, rtol=1e-4, atol=1e-6)
        np.testing.assert_allclose(lc, ec, rtol=1e-4, atol=1e-6)
        np.testing.assert_allclose(lo, eo, rtol=1e-4, atol=1e-6)
    gpu, ref, f64 = flat_params(params), flat_oracle(ost), flat_oracle(truth)
    if rel_l2(gpu, ref).max() > 1e-4:
        # a ReLU knife-edge flip of a rarely active unit moves all its fan-in
        # weights by ~lr: then hold the chaotic-drift contract instead
        assert_as_close_to_truth(gpu, ref, f64)
    np.testing.assert_array_equal(state.step[:k].cpu().numpy(), ost.step[:k])


@pytest.mark.parametrize("hidden,n_layers,n_freq,k,rays,points", [
    (256, 4, 5, 2, 64, 10), (1024, 4, 5, 1, 24, 10), (32, 6, 5, 2, 50, 10), (64, 4, 5, 2, 30, 40)])
def test_layered_gradient_accuracy(cuda, hidden, n_layers, n_freq, k, rays, points):
    """One step's gradient, recovered from Adam's first moment
    (m = (1 - b1) g after step 1), against an f64 run: relative L2 per layer."""
    arch = ModelArch(n_layers=n_layers, hidden=hidden, n_freq=n_freq)
    params, state = init_stacked(arch, k, seed=3)
    truth = f64_stack(O.new_stack(oracle_arch(arch), k, 3))
    batch = _synthetic_batch(arch, k, rays, points, seed=5)
    train_on_batch(params, state, batch, LossWeights())
    O.train_on_batch(truth, f64_batch(to_host_batch(batch)))
    for l in range(n_layers):
        for got, ref, name in ((state.m_weights[l], truth.mW[l], "W"), (state.m_biases[l], truth.mb[l], "b")):
            g = got[:k].cpu().numpy().astype(np.float64).reshape(k, -1)
            t = ref[:k].reshape(k, -1)
            rel = np.linalg.norm(g - t, axis=1) / np.maximum(np.linalg.norm(t, axis=1), 1e-30)
            assert rel.max() < 1e-5, f"layer {l} {name}: relative L2 {rel.max():.2e}"


def test_layered_vectorised_matches_sequential(cuda):
    """test_trainer.py:117-132 on the layered path: the weight-gradient sample
    split depends only on a model's own shape, so bits match."""
    arch = ModelArch(n_layers=4, hidden=256, n_freq=5)
    k = 3
    pv, sv = init_stacked(arch, k, seed=11)
    ps, ss = init_stacked(arch, k, seed=11)
    batch = _synthetic_batch(arch, k, 100, 10, seed=7)
    for _ in range(3):
        lv = train_on_batch(pv, sv, batch, LossWeights())
        ls = train_on_batch_sequential(ps, ss, batch, LossWeights())
        for a, b in zip(lv, ls):
            np.testing.assert_array_equal(a, b.astype(np.float32))
    assert torch.equal(pv.arena[:k], ps.arena[:k])


def test_fused_objects_with_wide_background(cuda):
    """Mapper.train_step's two stacks (trainer.py:364-390) when the background
    is wider than the fused kernels: objects on KF32, background layered, in
    one vm_train_step call."""
    ao, ab = ModelArch(hidden=32), ModelArch(hidden=256)
    po, so = init_stacked(ao, 4, seed=0)
    pb, sb = init_stacked(ab, 1, seed=0, stream=2)
    oo, ob = O.new_stack(oracle_arch(ao), 4, 0), O.new_stack(oracle_arch(ab), 1, 0, stream=2)
    bo = _synthetic_batch(ao, 4, 120, 10, seed=3)
    bb = _synthetic_batch(ab, 1, 600, 10, seed=4)
    for _ in range(5):
        losses, status = launch_train([(po, so, bo), (pb, sb, bb)], LossWeights())
        l = losses.cpu().numpy()
        st = status.cpu().numpy()
        assert st[2] == 1 and st[6] == 1
        e1 = O.train_on_batch(oo, to_host_batch(bo))
        e2 = O.train_on_batch(ob, to_host_batch(bb))
        np.testing.assert_allclose(l[:4], np.stack(e1, 1), rtol=1e-4, atol=1e-6)
        np.testing.assert_allclose(l[4:], np.stack(e2, 1), rtol=1e-4, atol=1e-6)
    assert_params_close(po, oo)
    assert_params_rel_l2(pb, ob)


def test_layered_nonfinite_gradient_and_stack_skip(cuda):
    """models.py:423-428 on the layered path (the offending model named,
    nothing updated), and a later stack skipped after an earlier stack's
    failure (the reference raises before training it)."""
    arch = ModelArch(n_layers=4, hidden=256, n_freq=5)
    params, state = init_stacked(arch, 3, seed=1)
    batch = _synthetic_batch(arch, 3, 30, 10, seed=2)
    batch.encoded[2, 0, 0, 0] = float("inf")
    before = params.arena.clone()
    with pytest.raises(FloatingPointError, match="model index 2"):
        train_on_batch(params, state, batch, LossWeights())
    assert torch.equal(before, params.arena)
    # stack 0 (fused objects) fails -> the wide background (stack 1) is skipped
    ao = ModelArch(hidden=32)
    po, so = init_stacked(ao, 2, seed=0)
    bo = _synthetic_batch(ao, 2, 40, 10, seed=3)
    bo.encoded[1, 0, 0, 0] = float("nan")
    pb, sb = init_stacked(arch, 1, seed=0, stream=2)
    bb = _synthetic_batch(arch, 1, 60, 10, seed=4)
    snap = pb.arena.clone()
    _, status = launch_train([(po, so, bo), (pb, sb, bb)], LossWeights())
    st = status.cpu().numpy()
    assert st[0] == 1 and st[6] == 0
    assert torch.equal(pb.arena, snap)
    assert sb.step[:1].cpu().tolist() == [0]


@pytest.mark.parametrize("hidden,n_layers,n_freq", [(256, 4, 5), (160, 3, 8)])
def test_layered_forward_backward_vs_oracle(cuda, hidden, n_layers, n_freq):
    """vm_forward / vm_backward (models.py:311-398) for wide models."""
    arch = ModelArch(n_layers=n_layers, hidden=hidden, n_freq=n_freq)
    k, n = 2, 333
    params, _ = init_stacked(arch, k, seed=7)
    ost = O.new_stack(oracle_arch(arch), k, 7)
    g = np.random.default_rng(hidden)
    enc = g.uniform(-1, 1, (k, n, arch.input_dim)).astype(np.float32)
    out, cache = forward(params, torch.from_numpy(enc))
    occ, col, xs, ms = O.mlp_forward(ost, enc)
    np.testing.assert_allclose(out.occupancy.cpu().numpy(), occ, rtol=1e-5, atol=1e-6)
    np.testing.assert_allclose(out.colour.cpu().numpy(), col, rtol=1e-5, atol=1e-6)
    go = g.standard_normal((k, n)).astype(np.float32)
    gc = g.standard_normal((k, n, 3)).astype(np.float32)
    grads = backward(params, cache, torch.from_numpy(go), torch.from_numpy(gc))
    dW, db = O.mlp_backward(ost, occ, col, xs, ms, go, gc)
    for l in range(n_layers):
        scale = np.abs(dW[l]).max() + 1e-6
        np.testing.assert_allclose(grads.d_weights[l].cpu().numpy(), dW[l], rtol=1e-4, atol=1e-5 * scale)
        scale = np.abs(db[l]).max() + 1e-6
        np.testing.assert_allclose(grads.d_biases[l].cpu().numpy(), db[l], rtol=1e-4, atol=1e-5 * scale)


FORCED_SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
from oracle import vobj_oracle as O
from paper_2302_01838_b200 import LossWeights, ModelArch, init_stacked
from paper_2302_01838_b200.trainer import _synthetic_batch, launch_train
from tests.helpers import assert_params_close, assert_params_rel_l2, oracle_arch, to_host_batch
ao, ab = ModelArch(hidden=32), ModelArch(hidden=128)
po, so = init_stacked(ao, 3, seed=0)
pb, sb = init_stacked(ab, 1, seed=0, stream=2)
oo, ob = O.new_stack(oracle_arch(ao), 3, 0), O.new_stack(oracle_arch(ab), 1, 0, stream=2)
bo = _synthetic_batch(ao, 3, 120, 10, seed=3)
bb = _synthetic_batch(ab, 1, 600, 10, seed=4)
for _ in range(5):
    losses, status = launch_train([(po, so, bo), (pb, sb, bb)], LossWeights())
    l = losses.cpu().numpy()
    e1 = O.train_on_batch(oo, to_host_batch(bo))
    e2 = O.train_on_batch(ob, to_host_batch(bb))
    np.testing.assert_allclose(l[:3], np.stack(e1, 1), rtol=1e-4, atol=1e-6)
    np.testing.assert_allclose(l[3:], np.stack(e2, 1), rtol=1e-4, atol=1e-6)
assert_params_rel_l2(po, oo)
assert_params_rel_l2(pb, ob)
print("layered ok")
"""


def test_layered_forced_on_the_bench_architectures(cuda):
    """VM_LAYERED=1: the config-2 architectures (h32 objects + h128
    background) through the layered path only -- an FP32 cross-check of what
    KF32 / KT compute, held to the layered contract."""
    root = Path(__file__).resolve().parents[1]
    env = dict(os.environ, VM_LAYERED="1")
    r = subprocess.run([sys.executable, "-c", FORCED_SCRIPT, str(root)], env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    assert "layered ok" in r.stdout


def test_layered_query_grid_vs_oracle(cuda):
    """meshing.py:64-97 query_grid for a hidden-256 model (inference on the
    layered forward, several chunks)."""
    from paper_2302_01838_b200.geometry import AABB
    from paper_2302_01838_b200.meshing import query_grid
    arch = ModelArch(n_layers=4, hidden=256, n_freq=5)
    params, _ = init_stacked(arch, 2, seed=9)
    ost = O.new_stack(oracle_arch(arch), 2, 9)
    box = AABB(np.array([-0.4, -0.3, -0.5]), np.array([0.5, 0.6, 0.2]))
    g = query_grid(params, 1, box, 0.8, 24, chunk=5000)
    exp = O.query_grid(ost, 1, box.min, box.max, 0.8, 24)
    np.testing.assert_allclose(g.values, exp, rtol=1e-4, atol=1e-6)
