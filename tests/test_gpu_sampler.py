"""GPU sampler (KS) parity: pixel draws, rays, samples bit-exact vs the oracle.

kf index / u / v / mask bit, sorted f64 sample distances, ray_ok, targets and
the f32 t are compared with array_equal.  The positional encoding uses device
f64 sin/cos (<= 2 ulp vs libm) before the f32 cast, so it is compared to 1e-6
and the number of differing f32 values is reported (expected ~0).
"""

import numpy as np
import pytest
import torch

from oracle import vobj_oracle as O
from paper_2302_01838_b200 import TrainConfig
from paper_2302_01838_b200.mapper import Mapper
from paper_2302_01838_b200.scenes import make_scene, populate

from .helpers import oracle_mapstate

pytestmark = pytest.mark.gpu


def _check_stack(mapper, ms, step, background):
    buf = mapper.assemble(step, background=background, encode=True, aux=True)
    insts = [ms.background] if background else ms.objects
    arch = ms.bg.arch if background else ms.obj.arch
    R = ms.rays_background if background else ms.rays_object
    enc_mismatch = 0
    for k, inst in enumerate(insts):
        nr = O.object_rays(inst, R)  # config 3: rows >= nr are zero padding
        exp, aux = O.assemble_batch(inst, ms.intr, arch, nr, step, ms.seed, ms.sampling, ms.bound_pad,
                                    with_aux=True)
        exp = O.pad_batch(exp, R, ms.sampling.n_stratified + ms.sampling.n_surface, arch.input_dim)
        if nr < R:
            for key in ("kf_idx", "u", "v", "t64"):
                assert not buf.aux[key][k][nr:].any()
            aux = dict(aux, t64=np.concatenate([aux["t64"], np.zeros((R - nr,) + aux["t64"].shape[1:])]))
            for key in ("kf_idx", "u", "v"):
                aux[key] = np.concatenate([aux[key], np.zeros(R - nr, aux[key].dtype)])
        np.testing.assert_array_equal(buf.aux["kf_idx"][k].cpu().numpy(), aux["kf_idx"])
        np.testing.assert_array_equal(buf.aux["u"][k].cpu().numpy(), aux["u"])
        np.testing.assert_array_equal(buf.aux["v"][k].cpu().numpy(), aux["v"])
        np.testing.assert_array_equal(buf.target_mask[k].cpu().numpy(), exp["target_mask"])
        np.testing.assert_array_equal(buf.valid_depth[k].cpu().numpy(), exp["valid_depth"])
        np.testing.assert_array_equal(buf.target_depth[k].cpu().numpy(), exp["target_depth"])
        np.testing.assert_array_equal(buf.target_colour[k].cpu().numpy(), exp["target_colour"])
        np.testing.assert_array_equal(buf.aux["t64"][k].cpu().numpy(), aux["t64"])
        np.testing.assert_array_equal(buf.t[k].cpu().numpy(), exp["t"])
        np.testing.assert_array_equal(buf.ray_ok[k].cpu().numpy(), exp["ray_ok"])
        enc = buf.encoded[k].cpu().numpy()
        np.testing.assert_allclose(enc, exp["encoded"], rtol=0, atol=1e-6)
        enc_mismatch += int((enc != exp["encoded"]).sum())
    return enc_mismatch


@pytest.mark.parametrize("n_obj,w,h,step", [(3, 160, 120, 0), (3, 160, 120, 5), (12, 640, 480, 3)])
def test_sampler_bit_exact(cuda, n_obj, w, h, step):
    scene = make_scene(n_obj, n_kf=3, width=w, height=h, focal=w / 2, crop=(20, min(w, h) // 2),
                       n_kf_bg=2, seed=n_obj + step)
    cfg = TrainConfig(seed=5)
    m = Mapper(scene["intrinsics"], cfg)
    populate(m, scene)
    ms = oracle_mapstate(scene, cfg)
    bad = _check_stack(m, ms, step, background=False)
    bad += _check_stack(m, ms, step, background=True)
    print("encoded f32 values differing from the oracle:", bad)


def test_single_keyframe_consumes_no_index_words(cuda):
    scene = make_scene(4, n_kf=1, width=160, height=120, focal=80, crop=(20, 50), n_kf_bg=1, seed=9)
    cfg = TrainConfig(seed=2)
    m = Mapper(scene["intrinsics"], cfg)
    populate(m, scene)
    ms = oracle_mapstate(scene, cfg)
    _check_stack(m, ms, 4, background=False)
    _check_stack(m, ms, 4, background=True)


def test_inactive_and_frozen_get_zero_batch(cuda):
    scene = make_scene(3, n_kf=2, width=160, height=120, focal=80, crop=(20, 50), n_kf_bg=1, seed=4)
    m = Mapper(scene["intrinsics"], TrainConfig())
    populate(m, scene)
    m.map.instances[2].active = False
    m.invalidate()
    m.freeze_object(3)
    buf = m.assemble(0, encode=True)
    for k in (1, 2):
        assert not buf.ray_ok[k].any() and float(buf.encoded[k].abs().sum()) == 0.0
    assert buf.ray_ok[0].any()
