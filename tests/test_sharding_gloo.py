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
