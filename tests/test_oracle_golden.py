"""Pin the CPU oracle (oracle/vobj_oracle.py) to golden vectors produced by the
real reference (tests/golden/make_golden.py).  CPU only.

Integer draws, f64 geometry/sampling, render, losses and Adam are compared
bit-exactly; OpenBLAS-backed matmuls (forward/backward/train) bit-exactly on
the golden host and within 1e-6 relative elsewhere (kernel choice is CPU
dependent)."""

from pathlib import Path

import numpy as np
import pytest

from oracle import vobj_oracle as O
from paper_2302_01838_b200 import TrainConfig
from paper_2302_01838_b200.scenes import config

from .helpers import oracle_mapstate

G = Path(__file__).resolve().parent / "golden"


@pytest.fixture(scope="module")
def ops():
    return np.load(G / "ops.npz")


def _flat(st):
    k = st.count
    return np.concatenate([np.concatenate([st.W[l][:k].reshape(k, -1), st.b[l][:k]], 1)
                           for l in range(len(st.W))], 1)


def _blas_close(a, b):
    np.testing.assert_allclose(a, b, rtol=1e-6, atol=1e-7)


@pytest.mark.parametrize("tag,arch,k", [("h32", O.Arch(4, 32, 5), 3), ("h16l3", O.Arch(3, 16, 3), 2)])
def test_models_init_forward_backward_adam(ops, tag, arch, k):
    st = O.new_stack(arch, k, 42)
    np.testing.assert_array_equal(_flat(st), ops[f"{tag}_init"])
    occ, col, xs, ms = O.mlp_forward(st, ops[f"{tag}_enc"])
    _blas_close(occ, ops[f"{tag}_occ"])
    _blas_close(col, ops[f"{tag}_col"])
    dW, db = O.mlp_backward(st, occ, col, xs, ms, ops[f"{tag}_go"], ops[f"{tag}_gc"])
    g = np.concatenate([np.concatenate([dW[l].reshape(k, -1), db[l]], 1) for l in range(arch.n_layers)], 1)
    _blas_close(g, ops[f"{tag}_dW"])
    # Adam on the golden gradients is exact (element-wise f32 ops)
    gold = ops[f"{tag}_dW"]
    off, gw, gb = 0, [], []
    for fo, fi in arch.dims():
        gw.append(gold[:, off:off + fo * fi].reshape(k, fo, fi)); off += fo * fi
        gb.append(gold[:, off:off + fo]); off += fo
    st.frozen[0] = k > 2
    for _ in range(3):
        O.adam_update(st, gw, gb, update_mask=np.array([True, False, True][:k]))
    np.testing.assert_array_equal(_flat(st), ops[f"{tag}_adam3"])
    np.testing.assert_array_equal(st.step[:k], ops[f"{tag}_adam3_step"])


def test_render_and_losses_exact(ops):
    O_, D, C, w, T = O.render_forward(ops["r_occ"], ops["r_col"], ops["r_t"])
    for a, b in ((O_, "r_O"), (D, "r_D"), (C, "r_C"), (w, "r_w"), (T, "r_T")):
        np.testing.assert_array_equal(a, ops[b])
    d_occ, d_col = O.render_backward(ops["r_occ"], ops["r_col"], ops["r_t"], w, T, ops["r_gO"], ops["r_gD"],
                                     ops["r_gC"])
    np.testing.assert_array_equal(d_occ, ops["r_docc"])
    np.testing.assert_array_equal(d_col, ops["r_dcol"])
    args = (ops["l_tD"], ops["l_tC"], ops["l_m"], ops["l_v"], ops["l_ok"])
    for a, b in zip(O.losses(O_, D, C, *args), ("l_ld", "l_lc", "l_lo", "l_lt")):
        np.testing.assert_array_equal(a, ops[b])
    for a, b in zip(O.loss_grads(O_, D, C, *args), ("l_dO", "l_dD", "l_dC")):
        np.testing.assert_array_equal(a, ops[b])


@pytest.fixture(scope="module")
def cfg1():
    scene = config("1")
    return scene, oracle_mapstate(scene, TrainConfig())


@pytest.mark.parametrize("step", [0, 3])
def test_sampler_matches_reference_bit_exact(cfg1, step):
    scene, ms = cfg1
    gold = np.load(G / "sampler_cfg1.npz")
    for k, inst in enumerate(ms.objects):
        b, aux = O.assemble_batch(inst, ms.intr, ms.obj.arch, ms.rays_object, step, ms.seed, ms.sampling,
                                  ms.bound_pad, with_aux=True)
        pre = f"s{step}_o{k}_"
        np.testing.assert_array_equal(aux["kf_idx"], gold[pre + "kf"])
        np.testing.assert_array_equal(aux["u"], gold[pre + "u"])
        np.testing.assert_array_equal(aux["v"], gold[pre + "v"])
        np.testing.assert_array_equal(aux["in_mask"], gold[pre + "mask"])
        np.testing.assert_array_equal(b["t"], gold[pre + "t"])
        np.testing.assert_array_equal(b["ray_ok"], gold[pre + "ok"])
        np.testing.assert_array_equal(b["valid_depth"], gold[pre + "valid"])
        np.testing.assert_array_equal(b["target_depth"], gold[pre + "tdepth"])
        np.testing.assert_array_equal(b["target_colour"], gold[pre + "tcol"])
        if step == 0:
            np.testing.assert_array_equal(b["encoded"], gold[pre + "enc"])
    b = O.assemble_batch(ms.background, ms.intr, ms.bg.arch, ms.rays_background, step, ms.seed, ms.sampling,
                         ms.bound_pad)
    np.testing.assert_array_equal(b["t"], gold[f"s{step}_bg_t"])
    np.testing.assert_array_equal(b["ray_ok"], gold[f"s{step}_bg_ok"])
    np.testing.assert_array_equal(b["target_depth"], gold[f"s{step}_bg_tdepth"])
    np.testing.assert_array_equal(b["target_mask"], gold[f"s{step}_bg_tmask"])
    if step == 0:
        np.testing.assert_array_equal(b["encoded"][:200], gold["s0_bg_enc200"])


def test_map_update_20_steps_matches_reference():
    scene = config("1")
    ms = oracle_mapstate(scene, TrainConfig())
    gold = np.load(G / "train_cfg1.npz")
    for step in range(20):
        rep = O.map_update_step(ms)
        got = np.array([rep[oid] for oid in sorted(rep)])
        np.testing.assert_allclose(got, gold["losses"][step], rtol=1e-6, atol=1e-7)
    _blas_close(_flat(ms.obj), gold["obj_params"])
    _blas_close(_flat(ms.bg), gold["bg_params"])


@pytest.mark.parametrize("tag,arch,k,rays,pts", [("syn32", O.Arch(4, 32, 5), 5, 120, 10),
                                                 ("syn16", O.Arch(3, 16, 3), 3, 24, 6)])
def test_train_on_batch_matches_reference(tag, arch, k, rays, pts):
    gold = np.load(G / "train_cfg1.npz")
    st = O.new_stack(arch, k, 11)
    b = O.synthetic_batch(arch, k, rays, pts, 7)
    ls = np.array([O.train_on_batch(st, b) for _ in range(20)])
    np.testing.assert_allclose(ls, gold[f"{tag}_losses"], rtol=1e-6, atol=1e-7)
    _blas_close(_flat(st), gold[f"{tag}_params"])


def test_padding_rows_are_inert():
    """Config 3 semantics: zero-batch rows (ray_ok = False) appended to an
    object's batch change neither its losses nor its parameter update
    (render.py:301-333 masks them out of every term)."""
    from paper_2302_01838_b200 import TrainConfig
    from paper_2302_01838_b200.scenes import make_scene
    from tests.helpers import oracle_mapstate
    sc = make_scene(2, n_kf=2, width=160, height=120, focal=100.0, crop=(20, 60), n_kf_bg=1, seed=4)
    cfg = TrainConfig(rays_per_object=40, train_background=False)
    a, b = oracle_mapstate(sc, cfg), oracle_mapstate(sc, cfg)
    for inst in b.objects:
        inst.n_rays = 25
    b.rays_object = 40
    a.rays_object = 25
    la, lb = O.map_update_step(a), O.map_update_step(b)
    for oid in la:
        np.testing.assert_allclose(la[oid], lb[oid], rtol=1e-6, atol=1e-7)
    for l in range(len(a.obj.W)):
        np.testing.assert_allclose(a.obj.W[l][:2], b.obj.W[l][:2], rtol=1e-6, atol=1e-7)


def test_inference_matches_reference():
    """query_grid (meshing.py:64-97) and render_view (meshing.py:485-579) of
    the oracle on the reference's trained config-1 map vs the reference."""
    from tests.helpers import trained_config1_oracle
    scene, ms, _ = trained_config1_oracle()
    gold = np.load(G / "infer_cfg1.npz")
    o0 = ms.objects[0]
    bmin, bmax = O._padded(o0.aabb.min, o0.aabb.max, 0.10)
    _blas_close(O.query_grid(ms.obj, 0, bmin, bmax, o0.pe_scale, (9, 10, 11)), gold["grid_obj0"])
    bg = ms.background
    bmin, bmax = O._padded(bg.aabb.min, bg.aabb.max, 0.10)
    _blas_close(O.query_grid(ms.bg, 0, bmin, bmax, bg.pe_scale, 8), gold["grid_bg"])
    pose = scene["background"]["keyframes"][0]["pose"]
    for tag, thr in (("v", 0.5), ("v0", 0.0)):
        rgb, depth, inst = O.render_view(ms.obj, ms.bg, ms.objects, bg, ms.intr, pose, samples_object=16,
                                         samples_background=16, samples_refine=8, threshold=thr)
        _blas_close(rgb, gold[tag + "_rgb"])
        _blas_close(depth, gold[tag + "_depth"])
        np.testing.assert_array_equal(inst, gold[tag + "_inst"])
