"""Object-parallel multi-GPU plumbing.

Every object is an independent model with its own keyframes, RNG streams
(keyed by object id) and Adam state, so objects shard across ranks with no
gradient collective.  What crosses ranks:
  * per step: the per-object loss triples (+ object ids) -> one all_gather
    (NCCL over NVLink on GPUs, gloo in the CPU tests);
  * on rebalance: an object's parameter block + Adam moments + step counter
    (point-to-point send/recv of one packed tensor).
Placement is longest-processing-time greedy on a per-object cost (rays x
samples x FLOP/sample), so a heavy background model gets its own share.
Model initialisation keys stay the object's global append index (SURVEY 8e
"init-key caveat"), so a sharded run starts from the same weights as a
single-stack run.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch


def plan_by_cost(costs, world: int) -> list[int]:
    """LPT greedy: returns owner rank per item (deterministic tie-breaks)."""
    order = sorted(range(len(costs)), key=lambda i: (-float(costs[i]), i))
    load = [0.0] * world
    owner = [0] * len(costs)
    for i in order:
        r = min(range(world), key=lambda q: (load[q], q))
        owner[i] = r
        load[r] += float(costs[i])
    return owner


def object_cost(rays: int, points: int, hidden: int, input_dim: int = 33) -> float:
    mac_fwd = hidden * input_dim + 2 * hidden * hidden + 4 * hidden
    mac_dx = 2 * hidden * hidden + 4 * hidden
    return float(rays * points * 2 * (2 * mac_fwd + mac_dx))


@dataclass
class ObjectSharding:
    world: int
    owner: list            # owner rank per global object index
    background_rank: int = 0
    rooms: bool = False    # one independent map per rank (weak scaling) instead of one sharded map
    _gather_buf: torch.Tensor | None = field(default=None, repr=False)

    @staticmethod
    def plan(scene: dict, world: int, rays_object: int = 120, rays_background: int = 1200, points: int = 10,
             hidden_object: int = 32, hidden_background: int = 128) -> "ObjectSharding":
        n = len(scene["objects"])
        costs = [object_cost(rays_object, points, hidden_object)] * n
        bg = scene.get("background") is not None
        if bg:
            costs = costs + [object_cost(rays_background, points, hidden_background)]
        owner = plan_by_cost(costs, world) if world > 1 else [0] * len(costs)
        bg_rank = owner[-1] if bg else 0
        return ObjectSharding(world, owner[:n], bg_rank)

    def objects_of(self, rank: int) -> list[int]:
        return [i for i, r in enumerate(self.owner) if r == rank]

    # -------------------------------------------------------- loss gather
    def gather_losses_device(self, losses: torch.Tensor) -> torch.Tensor | None:
        """All-gather a [k_local, 3] loss tensor (padded to the max shard) on the
        current stream; no host sync.  Returns the gathered [world, kmax, 3]."""
        if self.world == 1:
            return None
        import torch.distributed as dist
        kmax = max(sum(1 for r in self.owner if r == q) for q in range(self.world)) + 1
        if self._gather_buf is None or self._gather_buf.shape[1] != kmax or self._gather_buf.device != losses.device:
            self._gather_buf = torch.zeros((self.world, kmax, 3), dtype=losses.dtype, device=losses.device)
            self._send = torch.zeros((kmax, 3), dtype=losses.dtype, device=losses.device)
        self._send.zero_()
        self._send[:losses.shape[0]] = losses
        _all_gather(self._gather_buf.view(self.world, -1), self._send.view(-1))
        return self._gather_buf

    def gather_losses(self, report) -> dict | None:
        """Host-level gather of StepReport.losses (object id -> triple) to every
        rank; returns the merged dict.  With `rooms` (independent maps per
        rank, each with its own background id 0) the keys are (rank, id)."""
        if self.world == 1:
            return dict(report.losses)
        import torch.distributed as dist
        ids = sorted(report.losses)
        kmax = max(sum(1 for r in self.owner if r == q) for q in range(self.world)) + 1
        dev = (torch.device("cuda", torch.cuda.current_device()) if dist.get_backend() == "nccl"
               else torch.device("cpu"))
        rank = dist.get_rank()
        rows = np.full((kmax, 5), -1.0, dtype=np.float64)
        for j, oid in enumerate(ids):
            rows[j] = (rank, oid, *report.losses[oid])
        send = torch.from_numpy(rows).to(dev)
        out = torch.empty((self.world * kmax, 5), dtype=torch.float64, device=dev)
        _all_gather(out.view(self.world, -1), send.view(-1))
        merged = {}
        for row in out.cpu().numpy():
            if row[0] >= 0:
                key = (int(row[0]), int(row[1])) if self.rooms else int(row[1])
                merged[key] = (float(row[2]), float(row[3]), float(row[4]))
        return merged


def _all_gather(out2d: torch.Tensor, send: torch.Tensor) -> None:
    """out2d[r] <- send of rank r (NCCL all_gather_into_tensor; list form on gloo)."""
    import torch.distributed as dist
    if dist.get_backend() == "nccl":
        dist.all_gather_into_tensor(out2d.view(-1), send)
    else:
        parts = list(out2d.unbind(0))
        dist.all_gather(parts, send)


# ------------------------------------------------------------ migration


def pack_model(arena: torch.Tensor, m: torch.Tensor, v: torch.Tensor, step: torch.Tensor, k: int) -> torch.Tensor:
    """One object's parameter block, Adam moments and step counter as a flat
    float32 tensor (step stored as two exact float32 halves)."""
    s = int(step[k].item())
    meta = torch.tensor([float(s & 0xFFFFFF), float(s >> 24)], dtype=torch.float32, device=arena.device)
    return torch.cat([arena[k], m[k], v[k], meta])


def unpack_model(buf: torch.Tensor, arena: torch.Tensor, m: torch.Tensor, v: torch.Tensor, step: torch.Tensor,
                 k: int) -> None:
    b = arena.shape[1]
    arena[k] = buf[:b]
    m[k] = buf[b:2 * b]
    v[k] = buf[2 * b:3 * b]
    lo, hi = (int(x) for x in buf[3 * b:3 * b + 2].tolist())
    step[k] = lo + (hi << 24)


def migrate(arena, m, v, step, k_src: int, src: int, dst: int, rank: int, k_dst: int | None = None) -> None:
    """Move model `k_src` of rank `src` into slot `k_dst` of rank `dst`
    (point-to-point; collective over the pair)."""
    import torch.distributed as dist
    b = arena.shape[1]
    if rank == src:
        dist.send(pack_model(arena, m, v, step, k_src).contiguous(), dst)
    elif rank == dst:
        buf = torch.empty(3 * b + 2, dtype=torch.float32, device=arena.device)
        dist.recv(buf, src)
        unpack_model(buf, arena, m, v, step, k_src if k_dst is None else k_dst)
