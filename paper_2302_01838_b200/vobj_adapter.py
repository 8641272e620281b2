"""The binding a `vobj` maintainer adds to route the reference's
`train_on_batch` (trainer.py:480-506) through this package (INTEGRATION.md
"Python drop-in"): the reference keeps its numpy stacks; each call mirrors
them onto the device, runs the fused B200 step and writes the update back.

    # vobj/trainer.py, in Mapper.train_step's vectorised branch
    from paper_2302_01838_b200.vobj_adapter import b200_train_on_batch
    ld, lc, lo = b200_train_on_batch(self.obj_params, self.obj_state, batch, self.cfg.loss_weights)

This path pays a host<->device copy of the stack per call; for full speed the
stacks stay device-resident (`paper_2302_01838_b200.mapper.Mapper`).
"""

from __future__ import annotations

import numpy as np
import torch

from .models import ModelArch, init_stacked
from .render import LossWeights
from .trainer import RaySampleBatch, train_on_batch

_mirrors: dict = {}


def _mirror(params, state):
    """Device stack holding the reference stack's live models (weights,
    biases, Adam moments, step counters, frozen flags)."""
    a = params.arch
    arch = ModelArch(n_layers=a.n_layers, hidden=a.hidden, n_freq=a.n_freq, include_input=a.include_input)
    k = params.count
    key = id(params)
    hit = _mirrors.get(key)
    if hit is None or hit[0].count != k or hit[0].arch != arch:
        p, s = init_stacked(arch, k, seed=0, lr=state.lr, beta1=state.beta1, beta2=state.beta2, eps=state.eps)
        _mirrors[key] = (p, s)
    p, s = _mirrors[key]
    for l in range(arch.n_layers):
        p.weights[l][:k].copy_(torch.from_numpy(np.ascontiguousarray(params.weights[l][:k])))
        p.biases[l][:k].copy_(torch.from_numpy(np.ascontiguousarray(params.biases[l][:k])))
        s.m_weights[l][:k].copy_(torch.from_numpy(np.ascontiguousarray(state.m_weights[l][:k])))
        s.v_weights[l][:k].copy_(torch.from_numpy(np.ascontiguousarray(state.v_weights[l][:k])))
        s.m_biases[l][:k].copy_(torch.from_numpy(np.ascontiguousarray(state.m_biases[l][:k])))
        s.v_biases[l][:k].copy_(torch.from_numpy(np.ascontiguousarray(state.v_biases[l][:k])))
    s.step[:k].copy_(torch.from_numpy(np.asarray(state.step[:k], np.int64)))
    p.frozen[:k] = params.frozen[:k]
    p.version += 1
    return p, s


def b200_train_on_batch(params, state, batch, weights):
    """trainer.py:480-506 on the B200: same arguments (the reference's numpy
    StackedModelParams / OptimState / RaySampleBatch / LossWeights), same
    return value (per-model L_depth, L_colour, L_occ), same in-place update
    of the reference stack and the same exceptions."""
    p, s = _mirror(params, state)
    b = RaySampleBatch.from_arrays(batch.encoded, batch.t, batch.target_depth, batch.target_colour,
                                   batch.target_mask, batch.valid_depth, batch.ray_ok, batch.has_rays)
    out = train_on_batch(p, s, b, LossWeights(weights.colour, weights.occupancy))
    k = params.count
    for l in range(len(params.weights)):
        params.weights[l][:k] = p.weights[l][:k].cpu().numpy()
        params.biases[l][:k] = p.biases[l][:k].cpu().numpy()
        state.m_weights[l][:k] = s.m_weights[l][:k].cpu().numpy()
        state.v_weights[l][:k] = s.v_weights[l][:k].cpu().numpy()
        state.m_biases[l][:k] = s.m_biases[l][:k].cpu().numpy()
        state.v_biases[l][:k] = s.v_biases[l][:k].cpu().numpy()
    state.step[:k] = s.step[:k].cpu().numpy()
    params.version += 1
    return out
