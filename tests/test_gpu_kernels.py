"""GPU parity of the standalone kernels against the CPU oracle.

Bit-exact where the reference's float32 op order is reproducible (render,
losses, Adam given identical gradients); tolerance-bounded where
the reference uses OpenBLAS sgemm / scipy expit (MLP forward/backward).
"""

import numpy as np
import pytest
import torch

from oracle import vobj_oracle as O
from paper_2302_01838_b200 import (Gradients, LossWeights, ModelArch, adam_step, backward, compute_losses,
                                   forward, init_stacked, loss_output_grads, render_backward, render_rays,
                                   set_frozen)

from .helpers import host_layers, host_state, oracle_arch

pytestmark = pytest.mark.gpu


def _rng(seed):
    return np.random.default_rng(seed)


@pytest.mark.parametrize("S", [10, 6, 3])
def test_render_forward_backward_bit_exact(cuda, S):
    g = _rng(S)
    R = 400
    occ = g.uniform(0, 1, (R, S)).astype(np.float32)
    occ[0, 0] = 1.0  # o = 1 edge (clamped denominator)
    occ[1, :] = 0.0
    col = g.uniform(0, 1, (R, S, 3)).astype(np.float32)
    t = np.sort(g.uniform(0.1, 8, (R, S)), axis=1).astype(np.float32)
    res = render_rays(torch.from_numpy(occ), torch.from_numpy(col), torch.from_numpy(t))
    Oo, Do, Co, w, T = O.render_forward(occ, col, t)
    np.testing.assert_array_equal(res.opacity.cpu().numpy(), Oo)
    np.testing.assert_array_equal(res.depth.cpu().numpy(), Do)
    np.testing.assert_array_equal(res.colour.cpu().numpy(), Co)
    np.testing.assert_array_equal(res.weights.cpu().numpy(), w)
    np.testing.assert_array_equal(res.transmittance.cpu().numpy(), T)
    gO = g.standard_normal(R).astype(np.float32)
    gD = g.standard_normal(R).astype(np.float32)
    gC = g.standard_normal((R, 3)).astype(np.float32)
    d_occ, d_col = render_backward(torch.from_numpy(occ), torch.from_numpy(col), torch.from_numpy(t), res,
                                   torch.from_numpy(gO), torch.from_numpy(gD), torch.from_numpy(gC))
    e_occ, e_col = O.render_backward(occ, col, t, w, T, gO, gD, gC)
    np.testing.assert_array_equal(d_occ.cpu().numpy(), e_occ)
    np.testing.assert_array_equal(d_col.cpu().numpy(), e_col)


@pytest.mark.parametrize("K,R", [(3, 120), (2, 1200), (1, 7)])
def test_losses_and_grads_bit_exact(cuda, K, R):
    g = _rng(K * R)
    Oa = g.uniform(0, 1, (K, R)).astype(np.float32)
    Da = g.uniform(0, 4, (K, R)).astype(np.float32)
    Ca = g.uniform(0, 1, (K, R, 3)).astype(np.float32)
    tD = g.uniform(0, 4, (K, R)).astype(np.float32)
    tC = g.uniform(0, 1, (K, R, 3)).astype(np.float32)
    m, v, ok = g.random((K, R)) < 0.6, g.random((K, R)) < 0.8, g.random((K, R)) < 0.9
    Da[0, :3] = tD[0, :3]  # sign(0) = 0
    w = LossWeights()
    from paper_2302_01838_b200.render import RenderResult
    res = RenderResult(torch.from_numpy(Oa), torch.from_numpy(Da), torch.from_numpy(Ca), None, None)
    got = compute_losses(res, tD, tC, m, v, ok, w)
    exp = O.losses(Oa, Da, Ca, tD, tC, m, v, ok)
    for a, b in zip(got, exp):
        np.testing.assert_array_equal(a.cpu().numpy(), b)
    got = loss_output_grads(res, tD, tC, m, v, ok, w)
    exp = O.loss_grads(Oa, Da, Ca, tD, tC, m, v, ok)
    for a, b in zip(got, exp):
        np.testing.assert_array_equal(a.cpu().numpy(), b)


def test_init_matches_reference_streams(cuda):
    arch = ModelArch(n_layers=4, hidden=32, n_freq=5)
    params, _ = init_stacked(arch, 5, seed=42)
    ost = O.new_stack(oracle_arch(arch), 5, 42)
    W, B = host_layers(params)
    for l in range(4):
        np.testing.assert_array_equal(W[l], ost.W[l][:5])
        np.testing.assert_array_equal(B[l], ost.b[l][:5])


def _grads_for(arch, k, g):
    return ([g.standard_normal((k,) + (fo, fi)).astype(np.float32) * 0.1 for fo, fi in arch.layer_dims()],
            [g.standard_normal((k, fo)).astype(np.float32) * 0.1 for fo, _ in arch.layer_dims()])


@pytest.mark.parametrize("hidden,n_layers", [(32, 4), (128, 4), (16, 3)])
def test_adam_bit_exact_with_masks_and_frozen(cuda, hidden, n_layers):
    arch = ModelArch(n_layers=n_layers, hidden=hidden, n_freq=5)
    k = 5
    params, state = init_stacked(arch, k, seed=3)
    ost = O.new_stack(oracle_arch(arch), k, 3)
    set_frozen(params, 1, True)
    ost.frozen[1] = True
    g = _rng(hidden)
    for step in range(30):
        dW, db = _grads_for(arch, k, g)
        mask = g.random(k) < 0.7 if step % 3 else None
        adam_step(params, state, Gradients(dW, db), update_mask=mask)
        O.adam_update(ost, dW, db, update_mask=mask)
    W, B = host_layers(params)
    mW, vW, mb, vb, st = host_state(state, k)
    for l in range(n_layers):
        np.testing.assert_array_equal(W[l], ost.W[l][:k])
        np.testing.assert_array_equal(B[l], ost.b[l][:k])
        np.testing.assert_array_equal(mW[l], ost.mW[l][:k])
        np.testing.assert_array_equal(vW[l], ost.vW[l][:k])
    np.testing.assert_array_equal(st, ost.step[:k])


def test_adam_non_finite_names_model_and_updates_nothing(cuda):
    arch = ModelArch(n_layers=3, hidden=8, n_freq=1)
    params, state = init_stacked(arch, 3, seed=0)
    before = params.arena.clone()
    dW, db = _grads_for(arch, 3, _rng(1))
    dW[1][2, 0, 0] = np.nan
    with pytest.raises(FloatingPointError, match="model index 2"):
        adam_step(params, state, Gradients(dW, db))
    assert torch.equal(before, params.arena)
    # masked-out model's NaN is ignored
    adam_step(params, state, Gradients(dW, db), update_mask=np.array([True, True, False]))
    assert state.step.cpu().tolist()[:3] == [1, 1, 0]


@pytest.mark.parametrize("hidden,n_layers,n_freq", [(32, 4, 5), (128, 4, 5), (16, 3, 3), (64, 2, 2)])
def test_forward_backward_vs_oracle(cuda, hidden, n_layers, n_freq):
    arch = ModelArch(n_layers=n_layers, hidden=hidden, n_freq=n_freq)
    k, n = 3, 333
    params, _ = init_stacked(arch, k, seed=7)
    ost = O.new_stack(oracle_arch(arch), k, 7)
    g = _rng(hidden + n_layers)
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


def test_backward_stale_cache_rejected(cuda):
    arch = ModelArch(n_layers=3, hidden=8, n_freq=1)
    params, state = init_stacked(arch, 2, seed=0)
    enc = torch.zeros((2, 4, arch.input_dim))
    _, cache = forward(params, enc)
    grads = backward(params, cache, torch.ones((2, 4)), torch.ones((2, 4, 3)))
    adam_step(params, state, grads)
    with pytest.raises(ValueError, match="stale"):
        backward(params, cache, torch.ones((2, 4)), torch.ones((2, 4, 3)))
