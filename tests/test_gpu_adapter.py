"""The drop-in binding of INTEGRATION.md, exercised against the unmodified
reference package (baseline/_ref, the copy the reference arm runs): the
reference's numpy stack trained through vobj_adapter.b200_train_on_batch
tracks the reference's own train_on_batch (trainer.py:480-506) -- losses
within rtol 1e-4 every step, parameters and Adam moments within the
per-component contract after 5 steps -- and the update lands in the
reference's arrays in place."""

import copy
import sys
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


def _vobj():
    sys.path.insert(0, str(ROOT))
    import bench
    v = bench.import_reference_pkg()
    if v is None:
        pytest.skip("reference package not installed in baseline/_ref")
    return v


def test_adapter_tracks_reference_train_on_batch(cuda):
    _vobj()
    from vobj import models as RM
    from vobj import render as RR
    from vobj import trainer as RT

    from paper_2302_01838_b200.vobj_adapter import b200_train_on_batch

    arch = RM.ModelArch(hidden=32)
    ref_p, ref_s = RM.init_stacked(arch, 5, seed=11)
    gpu_p, gpu_s = copy.deepcopy(ref_p), copy.deepcopy(ref_s)
    batch = RT._synthetic_batch(arch, 5, 120, 10, seed=7)
    w = RR.LossWeights()
    for _ in range(5):
        exp = RT.train_on_batch(ref_p, ref_s, batch, w)
        got = b200_train_on_batch(gpu_p, gpu_s, batch, w)
        for a, e in zip(got, exp):
            np.testing.assert_allclose(a, e, rtol=1e-4, atol=1e-6)
    for l in range(arch.n_layers):
        np.testing.assert_allclose(gpu_p.weights[l][:5], ref_p.weights[l][:5], rtol=1e-4, atol=1e-5)
        np.testing.assert_allclose(gpu_p.biases[l][:5], ref_p.biases[l][:5], rtol=1e-4, atol=1e-5)
        np.testing.assert_allclose(gpu_s.m_weights[l][:5], ref_s.m_weights[l][:5], rtol=1e-4, atol=1e-6)
    np.testing.assert_array_equal(gpu_s.step[:5], ref_s.step[:5])
    assert gpu_p.version == 5
