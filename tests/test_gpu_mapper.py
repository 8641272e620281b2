"""Mapper.train_step (sampler + fused train, points path with in-kernel PE)
against the oracle's Mapper.train_step restatement on config 1."""

import numpy as np
import pytest

from oracle import vobj_oracle as O
from paper_2302_01838_b200 import TrainConfig
from paper_2302_01838_b200.mapper import Mapper
from paper_2302_01838_b200.scenes import config, make_scene, populate

from .helpers import (assert_as_close_to_truth, assert_params_close, f64_batch, f64_stack, flat_oracle,
                      flat_params, oracle_mapstate, rel_l2)

pytestmark = pytest.mark.gpu


def _run(scene, cfg, steps, strict_at=5, truth=None):
    m = Mapper(scene["intrinsics"], cfg)
    populate(m, scene)
    ms = oracle_mapstate(scene, cfg)
    worst = 0.0
    for s in range(steps):
        rep = m.train_step()
        if truth is not None:  # f64 run of the objects stack on the same batches
            bs = [O.assemble_batch(inst, ms.intr, ms.obj.arch, ms.rays_object, ms.global_step, ms.seed,
                                   ms.sampling, ms.bound_pad) for inst in ms.objects]
            O.train_on_batch(truth, f64_batch(O.stack_batches(bs)))
        exp = O.map_update_step(ms)
        if s + 1 == strict_at:
            assert_params_close(m.obj_params, ms.obj)
        assert sorted(rep.losses) == sorted(exp)
        for oid, trip in exp.items():
            got = np.array(rep.losses[oid])
            ref = np.array(trip)
            np.testing.assert_allclose(got, ref, rtol=1e-4, atol=1e-5, err_msg=f"step {s} object {oid}")
            worst = max(worst, float(np.max(np.abs(got - ref) / np.maximum(np.abs(ref), 1e-6))))
    return m, ms, worst


def test_config1_objects_20_steps(cuda):
    """Objects only (h32): parameter contract after N=20 steps."""
    scene = config("1")
    cfg = TrainConfig(train_background=False)
    truth = f64_stack(oracle_mapstate(scene, cfg).obj)
    m, ms, worst = _run(scene, cfg, 20, truth=truth)
    print("worst per-step loss rel diff", worst)
    # north star: per-object parameters within relative tolerance 1e-4
    assert rel_l2(flat_params(m.obj_params), flat_oracle(ms.obj)).max() <= 1e-4
    assert_as_close_to_truth(flat_params(m.obj_params), flat_oracle(ms.obj), flat_oracle(truth))


def test_config1_with_background_losses(cuda):
    """Objects + h128 background, per-step losses over 10 steps."""
    scene = config("1")
    m, ms, worst = _run(scene, TrainConfig(), 10)
    print("worst per-step loss rel diff", worst)


def test_config1_wide_background(cuda):
    """Mapper.train_step (graph-replayed) with a hidden-256 background: the
    objects on KF32 and the background on the layered path inside the same
    captured step; per-step losses over 5 steps and the background's
    parameters against the oracle's map_update_step."""
    from paper_2302_01838_b200 import ModelArch
    from .helpers import assert_params_rel_l2
    scene = config("1")
    cfg = TrainConfig(arch_background=ModelArch(n_layers=4, hidden=256, n_freq=5))
    m, ms, worst = _run(scene, cfg, 5)
    print("worst per-step loss rel diff", worst)
    assert_params_rel_l2(m.bg_params, ms.bg)


def test_frozen_background_reports_zero_loss(cuda):
    scene = make_scene(2, n_kf=1, width=160, height=120, focal=80, crop=(20, 50), n_kf_bg=1, seed=2)
    m = Mapper(scene["intrinsics"], TrainConfig())
    populate(m, scene)
    m.train_step()
    before = m.bg_params.arena.clone()
    m.freeze_object(0)
    rep = m.train_step()
    assert rep.losses[0] == (0.0, 0.0, 0.0)
    assert (m.bg_params.arena == before).all()
    assert rep.k_models == 3 and rep.step == 1


def test_unknown_mode_rejected(cuda):
    scene = make_scene(1, n_kf=1, width=64, height=48, focal=40, crop=(10, 20), n_kf_bg=1, seed=0)
    m = Mapper(scene["intrinsics"], TrainConfig())
    with pytest.raises(ValueError, match="mode"):
        m.train_step(mode="turbo")


def test_sharded_shard_matches_oracle_shard(cuda):
    """One rank's share of a cost-planned 2-rank map (global ids, global init
    keys, background on the plan's rank) on this GPU reproduces the oracle's
    shard, which the gloo test shows equals the unsharded map update."""
    from paper_2302_01838_b200.sharding import ObjectSharding
    scene = make_scene(7, n_kf=2, width=160, height=120, focal=100.0, crop=(20, 60), n_kf_bg=1, seed=5)
    cfg = TrainConfig(rays_per_object=24, rays_background=40)
    shard = ObjectSharding.plan(scene, 2, cfg.rays_per_object, cfg.rays_background, cfg.points_per_ray)
    for rank in (0, 1):
        mine = set(shard.objects_of(rank))
        m = Mapper(scene["intrinsics"], cfg)
        populate(m, scene, objects=mine, with_background=(rank == shard.background_rank))
        ms = oracle_mapstate(scene, cfg, objects=mine, with_background=(rank == shard.background_rank))
        for s in range(3):
            rep = m.train_step()
            exp = O.map_update_step(ms)
            assert sorted(rep.losses) == sorted(exp) == sorted([i + 1 for i in mine] +
                                                               ([0] if rank == shard.background_rank else []))
            for oid, trip in exp.items():
                np.testing.assert_allclose(np.array(rep.losses[oid]), np.array(trip), rtol=1e-4, atol=1e-5)
        if m.obj_params.count:  # the background's rank may own no objects
            assert_params_close(m.obj_params, ms.obj)


def test_report_total_and_nonfinite_errors(cuda):
    """StepReport.total is the reference's left-to-right sum over
    report.losses.values() (trainer.py:395-400); a non-finite model raises
    FloatingPointError through the graph-replayed step."""
    scene = config("1")
    cfg = TrainConfig()
    m = Mapper(scene["intrinsics"], cfg)
    populate(m, scene)
    for _ in range(3):
        rep = m.train_step()
        w = cfg.loss_weights
        total = 0
        for d, c, o in rep.losses.values():
            total += d + w.colour * c + w.occupancy * o
        assert rep.total == float(total)
        assert rep.k_models == len(rep.losses)
    m.obj_params.arena[2].fill_(float("nan"))
    with pytest.raises(FloatingPointError, match="non-finite"):
        m.train_step()
