"""Shared helpers for parity tests (host copies, oracle conversions)."""

from __future__ import annotations

import numpy as np

from oracle import vobj_oracle as O


def host_layers(params):
    k = params.count
    return ([w[:k].cpu().numpy().copy() for w in params.weights],
            [b[:k].cpu().numpy().copy() for b in params.biases])


def host_state(state, k):
    return ([m[:k].cpu().numpy().copy() for m in state.m_weights],
            [v[:k].cpu().numpy().copy() for v in state.v_weights],
            [m[:k].cpu().numpy().copy() for m in state.m_biases],
            [v[:k].cpu().numpy().copy() for v in state.v_biases],
            state.step[:k].cpu().numpy().copy())


def oracle_arch(arch):
    return O.Arch(arch.n_layers, arch.hidden, arch.n_freq, arch.include_input)


def assert_params_close(params, ost: O.Stack, rtol=1e-4, atol=1e-5, rel_l2=1e-4):
    """SURVEY hard-part-4 contract: per component rtol/atol + per-object rel L2."""
    W, B = host_layers(params)
    k = params.count
    for l in range(len(W)):
        np.testing.assert_allclose(W[l], ost.W[l][:k], rtol=rtol, atol=atol)
        np.testing.assert_allclose(B[l], ost.b[l][:k], rtol=rtol, atol=atol)
    mine = np.concatenate([np.concatenate([W[l].reshape(k, -1), B[l]], 1) for l in range(len(W))], 1)
    ref = np.concatenate([np.concatenate([ost.W[l][:k].reshape(k, -1), ost.b[l][:k]], 1)
                          for l in range(len(W))], 1)
    rel = np.linalg.norm(mine - ref, axis=1) / np.maximum(np.linalg.norm(ref, axis=1), 1e-30)
    assert rel.max() <= rel_l2, f"per-object relative L2 {rel.max():.3e} > {rel_l2}"


def to_host_batch(b):
    return {k: getattr(b, k).cpu().numpy() for k in
            ("encoded", "t", "target_depth", "target_colour", "target_mask", "valid_depth", "ray_ok")}
