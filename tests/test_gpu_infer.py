"""Forward-only inference on the GPU vs the reference's own
outputs (tests/golden/infer_cfg1.npz, made by running vobj's meshing.py on
its trained config-1 map) and vs the oracle at a mesh-sized grid.

query_grid (meshing.py:64-97) and render_view (meshing.py:485-579) evaluate
the MLP in f32 on f32-encoded points (numpy's f32 sin/cos vs CUDA sincosf:
a few ulp), so occupancy / colour / depth are compared at rtol 1e-4; the
per-pixel instance ids (depth competition with threshold) exactly.
"""

from pathlib import Path

import numpy as np
import pytest

from oracle import vobj_oracle as O
from paper_2302_01838_b200 import TrainConfig
from paper_2302_01838_b200.mapper import Mapper
from paper_2302_01838_b200.meshing import query_grid, render_view
from paper_2302_01838_b200.scenes import populate

from .helpers import load_flat_params, trained_config1_oracle

pytestmark = pytest.mark.gpu
G = Path(__file__).resolve().parent / "golden"


@pytest.fixture(scope="module")
def trained():
    scene, ms, gold = trained_config1_oracle()
    m = Mapper(scene["intrinsics"], TrainConfig())
    populate(m, scene)
    load_flat_params(m.obj_params, gold["obj_params"])
    load_flat_params(m.bg_params, gold["bg_params"])
    return scene, m, ms


def test_query_grid_matches_reference(cuda, trained):
    scene, m, ms = trained
    gold = np.load(G / "infer_cfg1.npz")
    o0 = m.instance_for_model(0)
    g = query_grid(m.obj_params, 0, o0.aabb.padded(0.10), o0.pe_scale, (9, 10, 11))
    np.testing.assert_allclose(g.values, gold["grid_obj0"], rtol=1e-4, atol=1e-6)
    bg = m.map.background
    g = query_grid(m.bg_params, bg.model_index, bg.aabb.padded(0.10), bg.pe_scale, 8)
    np.testing.assert_allclose(g.values, gold["grid_bg"], rtol=1e-4, atol=1e-6)


def test_query_grid_mesh_resolution_vs_oracle(cuda, trained):
    """64^3 object grid (TrainConfig.mesh_resolution_object) in several chunks."""
    scene, m, ms = trained
    for k in range(m.obj_params.count):
        inst = m.instance_for_model(k)
        box = inst.aabb.padded(0.10)
        g = query_grid(m.obj_params, k, box, inst.pe_scale, 64, chunk=100_000)
        exp = O.query_grid(ms.obj, k, box.min, box.max, inst.pe_scale, 64)
        np.testing.assert_allclose(g.values, exp, rtol=1e-4, atol=1e-6)


@pytest.mark.parametrize("tag,thr", [("v", 0.5), ("v0", 0.0)])
def test_render_view_matches_reference(cuda, trained, tag, thr):
    scene, m, ms = trained
    gold = np.load(G / "infer_cfg1.npz")
    pose = scene["background"]["keyframes"][0]["pose"]
    view = render_view(m.obj_params, m.bg_params, m.map, scene["intrinsics"], pose, samples_object=16,
                       samples_background=16, samples_refine=8, threshold=thr, chunk=5000)
    np.testing.assert_array_equal(view.instance, gold[tag + "_inst"])
    np.testing.assert_allclose(view.rgb, gold[tag + "_rgb"], rtol=1e-4, atol=1e-6)
    np.testing.assert_allclose(view.depth, gold[tag + "_depth"], rtol=1e-4, atol=1e-6)


def test_render_view_default_samples_vs_oracle(cuda, trained):
    """Default sample counts (48 / 48 / 32) from a second keyframe pose."""
    scene, m, ms = trained
    pose = scene["background"]["keyframes"][1]["pose"]
    view = render_view(m.obj_params, m.bg_params, m.map, scene["intrinsics"], pose)
    rgb, depth, inst = O.render_view(ms.obj, ms.bg, ms.objects, ms.background, ms.intr, pose)
    np.testing.assert_array_equal(view.instance, inst)
    np.testing.assert_allclose(view.rgb, rgb, rtol=1e-4, atol=1e-6)
    np.testing.assert_allclose(view.depth, depth, rtol=1e-4, atol=1e-6)


def test_query_grid_rejects_bad_resolution(cuda, trained):
    scene, m, ms = trained
    o0 = m.instance_for_model(0)
    with pytest.raises(ValueError, match="resolution"):
        query_grid(m.obj_params, 0, o0.aabb, o0.pe_scale, 1)
    with pytest.raises(IndexError):
        query_grid(m.obj_params, 99, o0.aabb, o0.pe_scale, 4)
