"""World-size-2 gloo runs of the object-sharding collectives on CPU:
per-step loss gather and object migration (send/recv of params + Adam)."""

import os
import socket
from types import SimpleNamespace

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2302_01838_b200.sharding import ObjectSharding, migrate


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        owner = [0, 1, 0, 1, 1]
        sh = ObjectSharding(world, owner)
        mine = sh.objects_of(rank)
        rep = SimpleNamespace(losses={i + 1: (float(i), 2.0 * i, rank + 0.5) for i in mine})
        merged = sh.gather_losses(rep)
        losses = torch.tensor([[float(i), 1.0, 2.0] for i in mine])
        buf = sh.gather_losses_device(losses)
        # migrate model slot 1 of rank 0 into slot 3 of rank 1
        arena = torch.full((4, 10), float(rank))
        arena[1] = torch.arange(10.0) + 100 * rank
        m, v = arena * 2, arena * 3
        step = torch.tensor([1, 42 + rank, 3, 4])
        migrate(arena, m, v, step, 1, 0, 1, rank, k_dst=3)
        q.put((rank, merged, buf.tolist(), arena.tolist(), int(step[3])))
    finally:
        dist.destroy_process_group()


def test_gather_and_migrate_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(2):
        r = q.get(timeout=120)
        res[r[0]] = r
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in (0, 1):
        merged = res[r][1]
        assert sorted(merged) == [1, 2, 3, 4, 5]
        assert merged[2] == (1.0, 2.0, 1.5) and merged[1] == (0.0, 0.0, 0.5)
        buf = torch.tensor(res[r][2])
        assert buf.shape[0] == 2 and buf[1, 0, 0] == 1.0 and buf[0, 1, 0] == 2.0
    assert res[1][3][3] == [float(x) for x in range(10)]   # rank 0's model 1 arrived in slot 3
    assert res[1][4] == 42                                  # with its Adam step counter


def _shard_worker(rank, world, port, q):
    """One rank of a sharded config-2-style map: build only the objects the
    cost plan gives this rank (global ids and init keys), run the reference
    step on them, all-gather the losses."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import vobj_oracle as O
        from paper_2302_01838_b200 import TrainConfig
        from paper_2302_01838_b200.scenes import make_scene
        from tests.helpers import oracle_mapstate
        scene = make_scene(7, n_kf=2, width=160, height=120, focal=100.0, crop=(20, 60), n_kf_bg=1, seed=5)
        cfg = TrainConfig(rays_per_object=24, rays_background=40)
        shard = ObjectSharding.plan(scene, world, cfg.rays_per_object, cfg.rays_background, cfg.points_per_ray)
        ms = oracle_mapstate(scene, cfg, objects=set(shard.objects_of(rank)),
                             with_background=(rank == shard.background_rank))
        merged = []
        for _ in range(2):
            merged.append(shard.gather_losses(SimpleNamespace(losses=O.map_update_step(ms))))
        q.put((rank, shard.objects_of(rank), shard.background_rank, merged))
    finally:
        dist.destroy_process_group()


def test_sharded_map_matches_single_stack_world2():
    """objects are independent models, so a map sharded by cost
    over two ranks (global ids + global init keys) reproduces the unsharded
    map update exactly, with only the per-object losses crossing ranks."""
    from oracle import vobj_oracle as O
    from paper_2302_01838_b200 import TrainConfig
    from paper_2302_01838_b200.scenes import make_scene
    from tests.helpers import oracle_mapstate
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_shard_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(2):
        r = q.get(timeout=180)
        res[r[0]] = r
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    scene = make_scene(7, n_kf=2, width=160, height=120, focal=100.0, crop=(20, 60), n_kf_bg=1, seed=5)
    ms = oracle_mapstate(scene, TrainConfig(rays_per_object=24, rays_background=40))
    full = [O.map_update_step(ms) for _ in range(2)]
    assert sorted(res[0][1] + res[1][1]) == list(range(7))       # every object on exactly one rank
    assert res[0][2] == res[1][2]
    for r in (0, 1):
        for step in range(2):
            assert res[r][3][step] == full[step]                  # bit-identical losses, every rank


def test_bench_self_launch_world2():
    """`bench.py --gpus 2` without WORLD_SIZE re-launches itself under
    torch.distributed.run; only rank 0 prints (reference arm: CPU only)."""
    import json
    import subprocess
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    env["OMP_NUM_THREADS"] = "1"
    out = subprocess.run([sys.executable, str(root / "bench.py"), "--impl", "reference", "--gpus", "2", "--steps",
                          "1", "--warmup", "1"], capture_output=True, text=True, env=env, timeout=600, cwd=root)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [json.loads(l) for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1 and lines[0]["n_gpus"] == 2 and lines[0]["impl"] == "reference"
