"""Small eager map-update run for compute-sanitizer (memcheck / racecheck /
synccheck): config-1 scene, objects (KF32) + background (KT + partial reduce),
sampler (KS) and Adam, plus the generic FFMA kernel (VM_KF32=0 runs), inference,
checkpoints and the layered path."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_2302_01838_b200 import TrainConfig
from paper_2302_01838_b200.mapper import Mapper
from paper_2302_01838_b200.scenes import config, populate

scene = config("1")
cfg = TrainConfig(rays_background=240)
m = Mapper(scene["intrinsics"], cfg, use_graphs=False)
populate(m, scene)
for _ in range(2):
    rep = m.train_step()
torch.cuda.synchronize()
print("ok", rep.step, len(rep.losses))

# graph-replayed steps (init kernel, persistent KF32 + prefetch, KT + PDL
# reduce, loss sums branch, split Adam, vm_step_finish)
mg = Mapper(scene["intrinsics"], cfg, use_graphs=True)
populate(mg, scene)
for _ in range(3):
    rep = mg.train_step()
torch.cuda.synchronize()
print("graph ok", rep.step, len(rep.losses))

# inference (vm_query_grid / vm_eval_rays / vm_view_*) on the trained map
from paper_2302_01838_b200.meshing import query_grid, render_view  # noqa: E402
inst = mg.instance_for_model(0)
query_grid(mg.obj_params, 0, inst.aabb.padded(0.1), inst.pe_scale, 16)
render_view(mg.obj_params, mg.bg_params, mg.map, scene["intrinsics"], scene["background"]["keyframes"][0]["pose"],
            samples_object=8, samples_background=8, samples_refine=4)
torch.cuda.synchronize()
print("infer ok")

# checkpoint pack/unpack (vm_pack_stack)
import tempfile  # noqa: E402
from paper_2302_01838_b200.checkpoint import load_checkpoint, save_checkpoint  # noqa: E402
with tempfile.TemporaryDirectory() as d:
    save_checkpoint(Path(d) / "m.vobj", mg.obj_params, mg.obj_state, mg.bg_params, mg.bg_state, mg.map)
    load_checkpoint(Path(d) / "m.vobj", device=mg.obj_params.arena.device)
torch.cuda.synchronize()
print("ckpt ok")

# layered path (vm_layered.cu): a hidden-256 background behind the fused
# objects in one call, and the layered forward / backward entry points
from paper_2302_01838_b200 import LossWeights, ModelArch, init_stacked  # noqa: E402
from paper_2302_01838_b200.models import backward, forward  # noqa: E402
from paper_2302_01838_b200.trainer import _synthetic_batch, launch_train  # noqa: E402
ao, ab = ModelArch(hidden=32), ModelArch(hidden=200, n_layers=3)
po, so = init_stacked(ao, 2, seed=0)
pb, sb = init_stacked(ab, 1, seed=0, stream=2)
bo, bb = _synthetic_batch(ao, 2, 40, 10, seed=3), _synthetic_batch(ab, 1, 70, 12, seed=4)
for _ in range(2):
    launch_train([(po, so, bo), (pb, sb, bb)], LossWeights())
out, cache = forward(pb, torch.randn(1, 77, ab.input_dim))
backward(pb, cache, torch.ones(1, 77), torch.ones(1, 77, 3))
torch.cuda.synchronize()
print("layered ok")
