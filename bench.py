"""Benchmark: vMAP map update (BASELINE.json config 2) on B200.

Workload (a "step"): one full Mapper.train_step on the config-2 synthetic scene
-- 50 objects x 5 keyframes (hidden-32 MLPs, 120 rays x 10 samples each) plus
the hidden-128 background (1200 rays) -- i.e. CUDA sampling (KS), the fused
MLP fwd/render/loss/bwd kernel (KF) and batched Adam (KA).

  python bench.py [--gpus N --steps K --warmup W]      # this framework
  python bench.py --impl reference [...]               # reference CPU path

N > 1: one process per GPU.  Without WORLD_SIZE in the environment,
`--gpus N` re-launches itself under torch.distributed.run (127.0.0.1); under
the driver's own torchrun WORLD_SIZE must equal N.  Workloads:
  --workload 2 (default)  weak scaling: every rank maps one config-2 room
                          (50 objects + its background, globally unique ids);
  --workload 4            strong scaling: BASELINE config 4, one 1000-object
                          map + background placed over the ranks by
                          ObjectSharding.plan (cost-greedy), each object on
                          exactly one rank with its global id and init key.
Per step the per-object loss triples are all-gathered over NCCL (the only
cross-rank traffic: objects are independent models).  Timing: CUDA events per
step on the launch stream with an L2 flush (256 MiB write) between steps, max
over ranks.
"""

from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "object-model training steps/sec (×objects) and ray-samples/sec at 50 objects"
UNIT = "object-steps/s"
OBJ_PER_RANK = 50


def kt_alone_ms(rays: int, points: int, reps: int = 20) -> float:
    """Device time of one background-only train call (KT's weight-image prep,
    KT, partial reduce, Adam) on an otherwise idle GPU: a config-2-shaped
    hidden-128 model on a synthetic batch (trainer.py:594-606), launches
    back to back between two CUDA events after a warm-up."""
    import torch
    from paper_2302_01838_b200 import LossWeights, ModelArch, init_stacked
    from paper_2302_01838_b200.trainer import TrainWorkspace, _synthetic_batch, launch_train
    ab = ModelArch(hidden=128)
    pb, sb = init_stacked(ab, 1, seed=0, stream=2)
    bb = _synthetic_batch(ab, 1, rays, points, seed=4)
    ws = TrainWorkspace()
    for _ in range(5):
        launch_train([(pb, sb, bb)], LossWeights(), ws)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        launch_train([(pb, sb, bb)], LossWeights(), ws)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def flop_per_sample(hidden: int, input_dim: int = 33) -> int:
    """Algorithmic GEMM FLOPs per sample: 2*(2*MAC_fwd + MAC_dx)."""
    mac_fwd = hidden * input_dim + 2 * hidden * hidden + 4 * hidden
    mac_dx = 2 * hidden * hidden + 4 * hidden
    return 2 * (2 * mac_fwd + mac_dx)


def _free_port() -> int:
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def self_launch(args) -> None:
    """--gpus N > 1 outside torchrun: re-exec under torch.distributed.run so the
    driver's plain `python bench.py --gpus N` measures N ranks."""
    env_world = os.environ.get("WORLD_SIZE")
    if env_world is not None:
        if args.gpus is not None and int(env_world) != args.gpus:
            sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={env_world}")
        return
    if args.gpus is not None and args.gpus > 1:
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr=127.0.0.1", f"--master-port={_free_port()}", str(Path(__file__).resolve())]
        cmd += sys.argv[1:]
        os.execv(sys.executable, cmd)


def dist_setup():
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return rank, world


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except FileNotFoundError:
            self.proc = None
        time.sleep(0.3)
        return self

    def __exit__(self, *a):
        self.lines = []
        if self.proc is not None:
            time.sleep(0.25)
            self.proc.terminate()
            out, _ = self.proc.communicate(timeout=10)
            self.lines = [l for l in out.splitlines() if l.strip()]

    def summary(self):
        if not self.lines:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in self.lines:
            f = [x.strip() for x in l.split(",")]
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except (ValueError, IndexError):
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def import_reference_pkg():
    """The unmodified reference package installed once into baseline/_ref
    (pip install --no-index --target baseline/_ref /root/reference/pkg).  Its
    meshing module imports scikit-image at import time, which this image
    lacks; the map-update path never calls it, so a stub module stands in."""
    import types
    ref = ROOT / "baseline" / "_ref"
    if not (ref / "vobj").is_dir():
        return None
    try:
        import skimage  # noqa: F401
    except ImportError:
        sk = types.ModuleType("skimage")
        meas, met = types.ModuleType("skimage.measure"), types.ModuleType("skimage.metrics")
        meas.marching_cubes = lambda *a, **k: (_ for _ in ()).throw(RuntimeError("skimage stub"))
        met.structural_similarity = lambda *a, **k: 0.0
        sk.measure, sk.metrics = meas, met
        sys.modules.update({"skimage": sk, "skimage.measure": meas, "skimage.metrics": met})
    sys.path.insert(0, str(ref))
    try:
        import vobj
    except Exception:
        return None
    return vobj


def reference_mapper(vobj, scene: dict, cfg):
    """The reference's Mapper populated with the scene exactly as
    scenes.populate does for this package (append order = init keys)."""
    from vobj import trainer as T
    from vobj.geometry import AABB
    from vobj.models import append_model
    from vobj.objects import add_keyframe
    from vobj.render import CameraIntrinsics
    from vobj.rng import PURPOSE_INIT_BACKGROUND, PURPOSE_INIT_OBJECT
    intr = scene["intrinsics"]
    rc = T.TrainConfig(seed=cfg.seed, rays_per_object=cfg.rays_per_object, rays_background=cfg.rays_background)
    m = T.Mapper(CameraIntrinsics(intr.fx, intr.fy, intr.cx, intr.cy, intr.width, intr.height), rc)
    if scene["background"] is not None:
        b = scene["background"]
        idx = append_model(m.bg_params, m.bg_state, rc.seed, PURPOSE_INIT_BACKGROUND)
        inst = m.map.add_background(AABB(b["aabb"].min, b["aabb"].max), rc.pe_scale_background, idx)
        for kf in b["keyframes"]:
            add_keyframe(inst, kf["frame_id"], kf["pose"], kf["bbox"], kf["mask"], scene["rgb"], scene["depth"])
    for ob in scene["objects"]:
        idx = append_model(m.obj_params, m.obj_state, rc.seed, PURPOSE_INIT_OBJECT)
        inst = m.map.add_object(1, AABB(ob["aabb"].min, ob["aabb"].max), rc.pe_scale_object, idx)
        m.model_to_object.append(inst.object_id)
        for kf in ob["keyframes"]:
            add_keyframe(inst, kf["frame_id"], kf["pose"], kf["bbox"], kf["mask"], scene["rgb"], scene["depth"])
    return m


def reference_stepper(scene: dict, cfg, workload: str):
    """(step(), kind, description) of the reference's CPU map update: the
    unmodified reference package when installed (configs 2 and 4), else the
    oracle port (config 3's per-object ray counts have no reference API)."""
    vobj = import_reference_pkg() if workload != "3" else None
    if vobj is not None:
        m = reference_mapper(vobj, scene, cfg)
        return m.train_step, "reference", "vobj Mapper.train_step (baseline/_ref, unmodified reference package)"
    from oracle import vobj_oracle as O
    from tests.helpers import oracle_mapstate
    ms = oracle_mapstate(scene, cfg)
    return (lambda: O.map_update_step(ms)), "port", "oracle/vobj_oracle.py map_update_step (numpy port)"


def cpu_sample(scene, seconds: float, cfg, workload: str, min_steps: int = 3):
    """Time the reference's CPU map update on the workload (bounded sample)."""
    step, kind, desc = reference_stepper(scene, cfg, workload)
    step()  # warm-up (BLAS threads, page faults)
    n, t0 = 0, time.perf_counter()
    while n < min_steps or time.perf_counter() - t0 < seconds:
        step()
        n += 1
    dt = (time.perf_counter() - t0) / n
    k = len(scene["objects"])
    one = None
    try:  # the same on one BLAS thread, a short bounded sample
        from threadpoolctl import threadpool_limits
        with threadpool_limits(1):
            t1 = time.perf_counter()
            for _ in range(2):
                step()
            one = k / ((time.perf_counter() - t1) / 2)
    except Exception:
        pass
    return k / dt, n, dt, kind, desc, one


def blas_threads():
    try:
        from threadpoolctl import threadpool_info
        return max([i.get("num_threads", 1) for i in threadpool_info()] or [1])
    except Exception:
        return os.cpu_count() or 1


def run_reference(args, rank, world):
    """--impl reference: the reference's own CPU map update (the unmodified
    package from baseline/_ref; the oracle port when it is absent) on the
    box's host cores, rank 0 only."""
    if rank != 0:
        return
    scene = workload_scene(args.workload, 0)
    import numpy as np
    step, kind, desc = reference_stepper(scene, workload_cfg(args.workload), args.workload)
    for _ in range(max(args.warmup, 1)):
        step()
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        step()
        times.append(time.perf_counter() - t0)
    dt = sum(times) / len(times)
    k = len(scene["objects"])
    if args.workload == "2":  # N rooms, as the GPU arm (timed on one host: N x the work)
        k, dt = k * world, dt * world
    v = k / dt
    cores = blas_threads()
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True,
        "scaling": "weak" if args.workload == "2" else "strong",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": _config(world, args.workload),
        "samples_per_s": k * 10 * float(np.mean([ob.get("n_rays", 120) for ob in scene["objects"]])) / dt,
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": kind,
                         "sample": f"{args.steps} full map-update steps of config {args.workload} ({desc}, "
                                   f"numpy/OpenBLAS, {cores} threads)"},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))


def workload_cfg(workload: str):
    from paper_2302_01838_b200 import TrainConfig
    return TrainConfig(rays_per_object=480) if workload == "3" else TrainConfig()


def workload_scene(workload: str, rank: int) -> dict:
    from paper_2302_01838_b200.scenes import config, make_scene
    if workload == "2":   # this rank's own config-2 room
        return make_scene(OBJ_PER_RANK, n_kf=5, seed=rank)
    return config(workload)


def _config(world, workload="2"):
    if workload == "3":
        return {"workload": "config 3: 200 objects x 10 keyframes + background, per-object rays log-uniform in "
                            "[30, 480] (batch width 480, ray_ok=False padding); full map update per step",
                "objects": 200, "hidden_object": 32, "hidden_background": 128, "rays_per_object": "30..480",
                "rays_background": 1200, "points_per_ray": 10, "frame": "1200x680",
                "l2": "flushed (256 MiB write) between timed steps",
                "parallelism": f"object-sharded x{world}" if world > 1 else "single GPU"}
    if workload == "4":
        return {"workload": "config 4: 1000 objects x 5 keyframes + background (config-2 style scene), one map "
                            "placed over the ranks by ObjectSharding.plan (cost-greedy); full map update per step "
                            "+ NCCL all-gather of the per-object losses",
                "objects": 1000, "hidden_object": 32, "hidden_background": 128, "rays_per_object": 120,
                "rays_background": 1200, "points_per_ray": 10, "frame": "1200x680",
                "l2": "flushed (256 MiB write) between timed steps",
                "parallelism": f"object-sharded x{world}" if world > 1 else "single GPU"}
    return {"workload": "config 2: Replica-sized synthetic scene, 50 objects x 5 keyframes + background; full "
                        "map update per step (ray/sample generation + fused MLP fwd/render/L1/bwd + Adam)",
            "objects_per_gpu": OBJ_PER_RANK, "objects": OBJ_PER_RANK * world, "hidden_object": 32,
            "hidden_background": 128, "rays_per_object": 120, "rays_background": 1200, "points_per_ray": 10,
            "frame": "1200x680", "l2": "flushed (256 MiB write) between timed steps",
            "parallelism": f"one config-2 room per GPU x{world}" if world > 1 else "single GPU"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=None)
    ap.add_argument("--workload", default="2", choices=["2", "3", "4"],
                    help="BASELINE config: 2 = 50-object room per GPU (weak), 4 = 1000 objects sharded (strong)")
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    self_launch(args)

    rank, world = dist_setup() if args.impl == "b200" else (int(os.environ.get("RANK", "0")),
                                                            int(os.environ.get("WORLD_SIZE", "1")))
    if args.impl == "reference":
        return run_reference(args, rank, world)

    import numpy as np
    import torch
    from paper_2302_01838_b200 import TrainConfig, _lib
    from paper_2302_01838_b200.mapper import Mapper
    from paper_2302_01838_b200.scenes import make_scene, populate
    from paper_2302_01838_b200.sharding import ObjectSharding

    dev = torch.device("cuda", torch.cuda.current_device())
    lib = _lib.load()
    cfg = workload_cfg(args.workload)
    scene = workload_scene(args.workload, rank)
    if args.workload == "2":
        # weak scaling: each rank maps one config-2 "room" (50 objects + its
        # background); object ids / init keys are globally unique across ranks.
        shard = ObjectSharding(world, [r for r in range(world) for _ in range(OBJ_PER_RANK)], rooms=True)
        mapper = Mapper(scene["intrinsics"], cfg, device=dev, object_id_base=rank * OBJ_PER_RANK,
                        init_index_base=rank * OBJ_PER_RANK, background_init_index=rank)
        populate(mapper, scene)
        k_total = OBJ_PER_RANK * world
    else:
        # strong scaling: one map, each object on exactly one rank (global id
        # and init key kept), the background on the rank the cost plan picks
        shard = ObjectSharding.plan(scene, world, cfg.rays_per_object, cfg.rays_background, cfg.points_per_ray,
                                    cfg.arch_object.hidden, cfg.arch_background.hidden)
        mapper = Mapper(scene["intrinsics"], cfg, device=dev)
        populate(mapper, scene, objects=set(shard.objects_of(rank)),
                 with_background=(rank == shard.background_rank))
        k_total = len(scene["objects"])
    k_local = mapper.obj_params.count
    has_bg = mapper.map.background is not None

    # FP32 FFMA peak (roofline denominator; MEASURED_PEAKS.json has no FP32 entry)
    tf = C.c_float()
    _lib.check(lib.vm_ffma_peak(16384, C.byref(tf), _lib.stream_ptr()), "vm_ffma_peak")
    ffma_peak = float(tf.value)

    for _ in range(args.warmup):
        rep = mapper.train_step()
        shard.gather_losses(rep)
    torch.cuda.synchronize()

    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    lib.vm_profile_enable(1)
    with ClockSampler(dev.index) as clk:
        for i in range(args.steps):
            flush.fill_(float(i))
            ev[i][0].record(stream)
            mapper.enqueue_graph_step(mapper.global_step)
            if world > 1:
                shard.gather_losses_device(mapper._ws.losses[:k_local + has_bg])
            ev[i][1].record(stream)
            mapper.global_step += 1
        torch.cuda.synchronize()
    n_kernels = C.c_long()
    lib.vm_profile_kernels(C.byref(n_kernels))
    lib.vm_profile_enable(0)
    kernels_per_step = mapper.kernels_per_step()
    # dominant-kernel timing: the graph replays above carry no host-visible
    # per-kernel events, so the fused kernel is event-timed on eager launches
    # of the same step (same inputs, L2 flushed before each) right after.
    lib.vm_profile_enable(1)
    n_prof = max(3, min(args.steps, 10))
    for i in range(n_prof):
        flush.fill_(float(i))
        mapper.enqueue_step(mapper.global_step)
        mapper.global_step += 1
    torch.cuda.synchronize()
    n_launch = C.c_int()
    mlp_ms = C.c_double()
    lib.vm_profile_read(C.byref(n_launch), C.byref(mlp_ms))
    # our kernels per graph-replayed step: those the eager steps launched
    # (vm_train_step + vm_sample count their launches) + the step-counter bump
    n_eager = C.c_long()
    lib.vm_profile_kernels(C.byref(n_eager))
    if n_eager.value > 0:
        kernels_per_step = n_eager.value // n_prof + 1
    per_tag = {}
    for tag in (1, 2, 3):  # 1: FFMA kernel KF (objects), 2: tensor-core branch KT (background), 3: reduce + Adam
        n_t, ms_t = C.c_int(), C.c_double()
        lib.vm_profile_read_tag(tag, C.byref(n_t), C.byref(ms_t))
        per_tag[tag] = ms_t.value / n_t.value if n_t.value else None
    lib.vm_profile_enable(0)
    step_ms = sum(a.elapsed_time(b) for a, b in ev)
    t_local = torch.tensor([step_ms], dtype=torch.float64, device=dev)
    if world > 1:
        torch.distributed.all_reduce(t_local, op=torch.distributed.ReduceOp.MAX)
        torch.distributed.barrier()
    total_ms = float(t_local.item())
    ms_per_step = total_ms / args.steps
    value = k_total * args.steps / (total_ms / 1e3)

    # end-to-end through the public API: Mapper.train_step() per step (graph
    # replay + one pinned D2H read of losses/status + StepReport).  Every
    # cfg.steps_per_frame steps -- the cadence at which run_mapping ingests a
    # frame (trainer.py:554-561) -- a frame's map growth is applied through
    # Mapper.add_keyframe: a new keyframe (crop from host memory) for 10% of
    # the objects, rotating, so the crops go host -> device, the sampling
    # tables are rebuilt and re-uploaded and the prefetched batch is redrawn.
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    local = [mapper.instance_for_model(j) for j in range(k_local)]
    n_new = max(1, k_local // 10)
    frame_id = 10 ** 6
    b0 = mapper.arena.uploaded_bytes
    tables = 0
    t0 = time.perf_counter()
    for i in range(args.steps):
        if i % cfg.steps_per_frame == 0 and i > 0 and local:
            frame_id += 1
            for j in range(n_new):
                inst = local[(frame_id * n_new + j) % len(local)]
                kf = inst.keyframes[0]
                mapper.add_keyframe(inst, frame_id, kf.pose, kf.bbox, kf.mask, scene["rgb"], scene["depth"])
        rep = mapper.train_step()
        tables += mapper.last_io_bytes()[0] if (i % cfg.steps_per_frame == 0 and i > 0) else 0
        shard.gather_losses(rep)
    torch.cuda.synchronize()
    e2e_s = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=dev)
    if world > 1:
        torch.distributed.all_reduce(e2e_s, op=torch.distributed.ReduceOp.MAX)
    e2e_value = k_total * args.steps / float(e2e_s.item())
    d2h = mapper.last_io_bytes()[1]
    h2d = -(-(mapper.arena.uploaded_bytes - b0 + tables) // args.steps)  # crops + tables, per step
    # the same public call without map growth: the reference arm's workload
    # (its Mapper.train_step loop, no new keyframes), for the like-for-like ratio
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    t0 = time.perf_counter()
    for i in range(args.steps):
        rep = mapper.train_step()
        shard.gather_losses(rep)
    torch.cuda.synchronize()
    e2e_t = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=dev)
    if world > 1:
        torch.distributed.all_reduce(e2e_t, op=torch.distributed.ReduceOp.MAX)
    e2e_train_only = k_total * args.steps / float(e2e_t.item())

    # rooflines: algorithmic FLOPs per launch / CUDA-event duration of that
    # launch (same step, eager replay with L2 flushed).  KF (objects, FP32
    # FFMA) and KT (background, tcgen05 3xTF32 + its weight-image prep) run
    # concurrently on two streams; the MLP phase is fork .. join.
    rays_obj = sum(int(mapper.instance_for_model(i).n_rays or cfg.rays_per_object) for i in range(k_local))
    flop_obj = rays_obj * cfg.points_per_ray * flop_per_sample(32)
    flop_bg = (cfg.rays_background * cfg.points_per_ray * flop_per_sample(128)) if (cfg.train_background
                                                                                    and has_bg) else 0
    flop_launch = flop_obj + flop_bg
    kernel_ms = mlp_ms.value / max(n_launch.value, 1)
    traffic = traffic_tc = None
    tf_path = ROOT / "profiles" / "traffic.json"
    if tf_path.exists():
        tj = json.loads(tf_path.read_text())
        traffic = tj.get("mlp_kernel_dram_bytes_per_launch")
        traffic_tc = tj.get("tc_train_kernel_dram_bytes_per_launch")
    peaks_path = ROOT / "MEASURED_PEAKS.json"
    bf16 = json.loads(peaks_path.read_text()).get("bf16_tflops") if peaks_path.exists() else None
    tf32_peak = (bf16 if bf16 else 1590.0) / 2.0
    tf32_src = ("dense TF32 = 1/2 of the measured bf16 cuBLAS burst peak in MEASURED_PEAKS.json" if bf16 else
                "dense TF32 = 1/2 of the profiling guide's fallback bf16 peak")
    kernels = []
    if per_tag.get(1):
        a = flop_obj / (per_tag[1] * 1e-3) / 1e12
        kernels.append({"bound": "fp32", "achieved": a, "peak": ffma_peak, "unit": "TFLOP/s", "frac": a / ffma_peak,
                        "traffic": traffic, "kernel": "kf32_train_kernel (KF, FFMA, hidden-32 objects)",
                        "kernel_ms": per_tag[1], "flop_per_launch": flop_obj,
                        "peak_source": "FP32 FFMA throughput measured in this run by vm_ffma_peak "
                                       "(MEASURED_PEAKS.json has no FP32 entry)"})
    if per_tag.get(2) and flop_bg:
        a = flop_bg / (per_tag[2] * 1e-3) / 1e12
        kernels.append({"bound": "tensor", "achieved": a, "peak": tf32_peak, "unit": "TFLOP/s", "frac": a / tf32_peak,
                        "traffic": traffic_tc, "kernel": "tc_train_kernel (KT, tcgen05 3xTF32, hidden-128 background)",
                        "kernel_ms": per_tag[2], "flop_per_launch": flop_bg,
                        "note": "3xTF32 issues 3 MMAs per algorithmic product; tensor-pipe FLOPs = 3x achieved; "
                                "kernel_ms is the branch's event span inside the step, which includes waiting "
                                "for KF32 to free whole SMs",
                        "peak_source": tf32_src})
        try:  # the same background stack alone on an idle GPU (prep + KT + reduce + Adam);
            # VM_BENCH_ALONE=0 skips it (ncu launch lists: per-step kernels only)
            if os.environ.get("VM_BENCH_ALONE", "1") == "0":
                raise RuntimeError("skipped (VM_BENCH_ALONE=0)")
            alone = kt_alone_ms(cfg.rays_background, cfg.points_per_ray)
            kernels[-1]["alone_call_ms"] = alone
            kernels[-1]["alone_frac"] = flop_bg / (alone * 1e-3) / 1e12 / tf32_peak
        except Exception as e:  # measurement aid only: never fail the bench line on it
            kernels[-1]["alone_call_ms"] = None
            kernels[-1]["alone_error"] = repr(e)[:200]
    if not kernels:  # single FFMA launch (e.g. VM_TC=0): the phase is the kernel
        a = flop_launch / (kernel_ms * 1e-3) / 1e12
        kernels.append({"bound": "fp32", "achieved": a, "peak": ffma_peak, "unit": "TFLOP/s", "frac": a / ffma_peak,
                        "traffic": traffic, "kernel": "mlp_kernel (fused KF)", "kernel_ms": kernel_ms,
                        "flop_per_launch": flop_launch, "peak_source": "FP32 FFMA throughput measured in this run"})
    # dominant = largest share of the ncu launch list (profiles/*_summary.md):
    # the FFMA object kernel KF when present (it and KT overlap on two streams)
    dominant = kernels[0]

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        v, n, dt, kind, desc, one = cpu_sample(scene, args.cpu_seconds, cfg, args.workload)
        cores = blas_threads()
        cpu = {"value": v, "unit": UNIT, "cores": cores, "kind": kind,
               "sample": f"{n} full map-update steps of config {args.workload} ({dt*1e3:.0f} ms/step) through "
                         f"{desc} (numpy/OpenBLAS, {cores} threads)",
               "value_1_thread": one}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "weak" if args.workload == "2" else "strong",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic", "config": _config(world, args.workload),
            "samples_per_s": (rays_obj / max(k_local, 1)) * value * cfg.points_per_ray,
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "includes": "Mapper.train_step per step + every steps_per_frame steps a frame's map growth "
                                "(new keyframes for 10% of objects: crops H2D, tables rebuilt, batch redrawn)",
                    "train_only": e2e_train_only},
            "gpu_launches": kernels_per_step * args.steps,
            "roofline": dominant,
            "roofline_kernels": kernels,
            "mlp_phase": {"ms": kernel_ms, "flop": flop_launch,
                          "achieved_tflops": flop_launch / (kernel_ms * 1e-3) / 1e12,
                          "frac_of_fp32_peak": flop_launch / (kernel_ms * 1e-3) / 1e12 / ffma_peak,
                          "note": "the whole fused MLP (KF32 objects || KT background, fork..join): algorithmic "
                                  "FLOPs / phase time against the FP32 FFMA peak, the roofline of the "
                                  "reference's f32 arithmetic (north star: fused-MLP roofline)",
                          "reduce_adam_ms": per_tag.get(3)},
            "clocks": clk.summary(),
            "cpu_baseline": cpu,
        }
        print(json.dumps(line))
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
