"""Host-side logic on CPU: arena layout views, config validation, scenes,
sharding plans.  No GPU."""

import numpy as np
import pytest
import torch

from paper_2302_01838_b200 import AssociationConfig, ModelArch, SamplingConfig, TrainConfig
from paper_2302_01838_b200.models import _Arena, _init_model_arrays
from paper_2302_01838_b200.scenes import config, make_scene
from paper_2302_01838_b200.sharding import ObjectSharding, object_cost, pack_model, plan_by_cost, unpack_model


@pytest.mark.parametrize("arch", [ModelArch(4, 32, 5), ModelArch(3, 16, 3), ModelArch(2, 5, 1, False),
                                  ModelArch(4, 128, 5)])
def test_arena_views_roundtrip(arch):
    lay = _Arena(arch)
    ws, bs = _init_model_arrays(arch, 3, 1, 1)
    host = lay.pack([w[None] for w in ws], [b[None] for b in bs])
    arena = torch.from_numpy(np.concatenate([host, np.zeros_like(host)]))
    for l in range(arch.n_layers):
        v = lay.weight_view(arena, l)
        assert tuple(v.shape) == (2,) + ws[l].shape
        np.testing.assert_array_equal(v[0].numpy(), ws[l])
        np.testing.assert_array_equal(lay.bias_view(arena, l)[0].numpy(), bs[l])
        assert not v[1].any()
    # padding outside the views is zero
    mask = np.zeros(lay.block, bool)
    for l in range(arch.n_layers):
        mask[lay.weight_view(torch.from_numpy(np.arange(lay.block, dtype=np.float32)[None]), l).numpy().astype(int).ravel()] = True
        mask[lay.bias_view(torch.from_numpy(np.arange(lay.block, dtype=np.float32)[None]), l).numpy().astype(int).ravel()] = True
    assert mask.sum() == lay.n_params
    assert not host[0][~mask].any()


def test_config_validation():
    with pytest.raises(ValueError):
        TrainConfig(steps_per_frame=0)
    with pytest.raises(ValueError):
        SamplingConfig(t_near=2.0, t_far=1.0)
    with pytest.raises(ValueError):
        AssociationConfig(iou_threshold=0.0)
    with pytest.raises(ValueError):
        ModelArch(n_layers=1)
    c = TrainConfig()
    assert (c.rays_per_object, c.rays_background, c.points_per_ray) == (120, 1200, 10)
    assert c.arch_background.hidden == 128 and c.arch_object.input_dim == 33


def test_config2_scene_shapes():
    s = config("2")
    assert len(s["objects"]) == 50 and len(s["background"]["keyframes"]) == 5
    for ob in s["objects"]:
        assert len(ob["keyframes"]) == 5
        for kf in ob["keyframes"]:
            u0, v0, u1, v1 = kf["bbox"]
            assert 60 <= u1 - u0 < 140 and 60 <= v1 - v0 < 140 and kf["mask"].shape == (v1 - v0, u1 - u0)
            assert 0 <= u0 and u1 <= 1200 and 0 <= v0 and v1 <= 680


def test_lpt_plan_balances_and_is_deterministic():
    costs = [object_cost(120, 10, 32)] * 100 + [object_cost(1200, 10, 128)]
    own = plan_by_cost(costs, 4)
    assert own == plan_by_cost(costs, 4)
    load = [sum(c for c, o in zip(costs, own) if o == r) for r in range(4)]
    # LPT bound: makespan <= max(largest item, 4/3 x ideal); the background
    # (125 objects' worth of FLOPs) is indivisible and gets a rank of its own
    assert max(load) <= max(max(costs), 4 / 3 * sum(costs) / 4) * (1 + 1e-9)
    assert sorted(load)[2] - sorted(load)[0] <= costs[0]   # object-only ranks level within one object
    sh = ObjectSharding.plan(make_scene(20, n_kf=1, width=64, height=48, focal=40, crop=(10, 20)), 3)
    assert sorted(sum((sh.objects_of(r) for r in range(3)), [])) == list(range(20))


def test_pack_unpack_model():
    arena = torch.randn(4, 37)
    m, v = torch.randn(4, 37), torch.rand(4, 37)
    step = torch.tensor([0, 5, 123456789, 7], dtype=torch.int64)
    buf = pack_model(arena, m, v, step, 2)
    a2, m2, v2, s2 = torch.zeros_like(arena), torch.zeros_like(m), torch.zeros_like(v), torch.zeros_like(step)
    unpack_model(buf, a2, m2, v2, s2, 1)
    assert torch.equal(a2[1], arena[2]) and torch.equal(m2[1], m[2]) and torch.equal(v2[1], v[2])
    assert int(s2[1]) == 123456789


def test_associate_vectorised_matches_pairwise_loop():
    """ingest.associate (one IoU matrix) == the pairwise loop of
    objects.py:233-259 on random boxes with shared classes and exact ties."""
    from types import SimpleNamespace

    from paper_2302_01838_b200.geometry import AABB, aabb_iou
    from paper_2302_01838_b200.ingest import associate
    from paper_2302_01838_b200.objects import AssociationConfig

    def loop(dets, objs, thr):
        cand = []
        for di, d in enumerate(dets):
            for o in objs:
                if o.semantic_class != d.semantic_class:
                    continue
                iou = aabb_iou(d.aabb, o.aabb)
                if iou >= thr:
                    cand.append((-iou, o.object_id, di))
        cand.sort()
        out, used = [None] * len(dets), set()
        for _, oid, di in cand:
            if out[di] is None and oid not in used:
                out[di] = oid
                used.add(oid)
        return out

    g = np.random.default_rng(3)
    for trial in range(20):
        def box():
            lo = g.uniform(-2, 2, 3)
            return AABB(lo, lo + g.uniform(0.05, 1.5, 3))
        objs = [SimpleNamespace(object_id=int(i * 3 + 1), semantic_class=int(g.integers(1, 3)), aabb=box())
                for i in range(int(g.integers(0, 40)))]
        dets = [SimpleNamespace(semantic_class=int(g.integers(1, 3)), aabb=box()) for _ in range(int(g.integers(0, 30)))]
        if objs and dets:  # an exact duplicate box: tie on IoU
            dets[0].aabb = AABB(objs[0].aabb.min.copy(), objs[0].aabb.max.copy())
            dets[0].semantic_class = objs[0].semantic_class
        omap = SimpleNamespace(objects=lambda objs=objs: iter(objs))
        cfg = AssociationConfig()
        for thr in (cfg.iou_threshold, 0.01):
            c = AssociationConfig(iou_threshold=thr)
            assert associate(dets, omap, c) == loop(dets, objs, thr), trial
