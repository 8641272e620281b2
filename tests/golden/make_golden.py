"""Generate golden vectors by running the REAL reference (`vobj`) in the build
container.  /root/reference does not exist on the GPU box, so the outputs are
committed as small .npz fixtures next to this script.

The reference imports scikit-image (meshing) which is not installed; the hot
path never calls it, so a stub module is injected first.

    python tests/golden/make_golden.py          # rewrites tests/golden/*.npz
"""

from __future__ import annotations

import sys
import types
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parents[1]
REF = Path("/root/reference/pkg/src")


def import_reference():
    sk = types.ModuleType("skimage")
    sk.__version__ = "stub"
    meas = types.ModuleType("skimage.measure")
    meas.marching_cubes = lambda *a, **k: (_ for _ in ()).throw(RuntimeError("skimage stub"))
    met = types.ModuleType("skimage.metrics")
    met.structural_similarity = lambda *a, **k: 0.0
    sk.measure, sk.metrics = meas, met
    sys.modules.update({"skimage": sk, "skimage.measure": meas, "skimage.metrics": met})
    sys.path.insert(0, str(REF))
    import vobj  # noqa: F401
    return vobj


def ref_mapper(vobj, scene, rays_obj=120, rays_bg=1200, seed=0, train_bg=True):
    from vobj import trainer as T
    from vobj.geometry import AABB
    from vobj.models import append_model
    from vobj.objects import add_keyframe
    from vobj.rng import PURPOSE_INIT_BACKGROUND, PURPOSE_INIT_OBJECT
    from vobj.render import CameraIntrinsics
    intr = scene["intrinsics"]
    ri = CameraIntrinsics(intr.fx, intr.fy, intr.cx, intr.cy, intr.width, intr.height)
    cfg = T.apply_config_overrides(T.TrainConfig(), {"seed": str(seed), "rays_per_object": str(rays_obj),
                                                     "rays_background": str(rays_bg),
                                                     "train_background": "1" if train_bg else "0"})
    m = T.Mapper(ri, cfg)
    if scene["background"] is not None:
        b = scene["background"]
        idx = append_model(m.bg_params, m.bg_state, cfg.seed, PURPOSE_INIT_BACKGROUND)
        inst = m.map.add_background(AABB(b["aabb"].min, b["aabb"].max), cfg.pe_scale_background, idx)
        for kf in b["keyframes"]:
            add_keyframe(inst, kf["frame_id"], kf["pose"], kf["bbox"], kf["mask"], scene["rgb"], scene["depth"])
    for ob in scene["objects"]:
        idx = append_model(m.obj_params, m.obj_state, cfg.seed, PURPOSE_INIT_OBJECT)
        inst = m.map.add_object(1, AABB(ob["aabb"].min, ob["aabb"].max), cfg.pe_scale_object, idx)
        m.model_to_object.append(inst.object_id)
        for kf in ob["keyframes"]:
            add_keyframe(inst, kf["frame_id"], kf["pose"], kf["bbox"], kf["mask"], scene["rgb"], scene["depth"])
    return m


def flat(params):
    k = params.count
    return np.concatenate([np.concatenate([params.weights[l][:k].reshape(k, -1), params.biases[l][:k]], 1)
                           for l in range(len(params.weights))], 1)


INGEST_STRIDES = dict(keyframe_stride_object=2, keyframe_stride_background=3)
INGEST_RAYS = dict(rays_per_object=48, rays_background=96, steps_per_frame=2)


def ingest_goldens(vobj):
    """Synthetic RGB-D datasets written by the reference's own generator
    (synth.generate: PNGs + poses/intrinsics/classes, committed under
    tests/golden/ds_*), then the reference's ingestion and mapping loop on
    them: per-frame detections / scene bounds, the map after every frame, and
    run_mapping's losses and parameters."""
    import dataclasses
    import shutil
    from vobj import synth
    from vobj.datasets import Dataset
    from vobj.objects import AssociationConfig, extract_detections, scene_bounds
    from vobj.trainer import Mapper, TrainConfig, run_mapping
    specs = {
        "ds_mini": dataclasses.replace(synth.mini_scene(n_frames=8), permute_mask_ids=True),
        "ds_five": dataclasses.replace(synth.five_object_scene(n_frames=6), width=200, height=150, focal=150.0,
                                       depth_noise_std=0.004),
    }
    out = {}
    for name, spec in specs.items():
        root = HERE / name
        if root.exists():
            shutil.rmtree(root)
        ds = synth.generate(spec, root, seed=3)
        shutil.rmtree(root / "gt_mesh")
        acfg = AssociationConfig(**INGEST_STRIDES)
        cfg = TrainConfig(association=acfg)
        m = Mapper(ds.intrinsics, cfg)
        for i in range(len(ds)):
            fr = ds.frame(i)
            dets = extract_detections(fr.rgb, fr.depth, fr.mask, fr.frame_id, ds.intrinsics, fr.pose, ds.classes,
                                      acfg)
            sb = scene_bounds(fr.depth, ds.intrinsics, fr.pose)
            pre = f"{name}_f{i}_"
            out[pre + "scene"] = np.concatenate([sb.min, sb.max]) if sb is not None else np.zeros(0)
            out[pre + "det_bbox"] = np.array([d.bbox for d in dets], np.int64).reshape(-1, 4)
            out[pre + "det_n"] = np.array([d.n_pixels for d in dets], np.int64)
            out[pre + "det_cls"] = np.array([d.semantic_class for d in dets], np.int64)
            out[pre + "det_box"] = np.array([np.concatenate([d.aabb.min, d.aabb.max]) for d in dets]).reshape(-1, 6)
            m.process_frame(fr, ds.classes)
            objs = [m.map.instances[o] for o in m.model_to_object]
            out[pre + "obj_ids"] = np.array([o.object_id for o in objs], np.int64)
            out[pre + "obj_box"] = np.array([np.concatenate([o.aabb.min, o.aabb.max]) for o in objs]).reshape(-1, 6)
            out[pre + "obj_obs"] = np.array([o.obs_count for o in objs], np.int64)
            out[pre + "obj_kf"] = np.array([[k.frame_id, *k.bbox, int(o.object_id)] for o in objs
                                            for k in o.keyframes], np.int64).reshape(-1, 6)
            bg = m.map.background
            out[pre + "bg_box"] = np.concatenate([bg.aabb.min, bg.aabb.max])
            out[pre + "bg_kf"] = np.array([k.frame_id for k in bg.keyframes], np.int64)
        cfg2 = TrainConfig(association=acfg, **INGEST_RAYS)
        mm, reports = run_mapping(ds, cfg2)
        width = max(len(r.losses) for r in reports)
        ids = np.full((len(reports), width), -1, np.int64)
        ls = np.full((len(reports), width, 3), np.nan)
        for j, r in enumerate(reports):
            keys = sorted(r.losses)
            ids[j, :len(keys)] = keys
            ls[j, :len(keys)] = [r.losses[k] for k in keys]
        out[f"{name}_map_ids"], out[f"{name}_map_losses"] = ids, ls
        out[f"{name}_map_obj_params"] = flat(mm.obj_params)
        out[f"{name}_map_bg_params"] = flat(mm.bg_params)
    np.savez_compressed(HERE / "ingest.npz", **out)


def checkpoint_golden(vobj):
    """A VOBJ v1 file written by the reference (checkpoint.py:132-144): two
    trained stacks (hidden 16 / 32, one frozen model) + an object table with
    a keyframe reference (test_checkpoint.py's fixtures)."""
    from vobj.checkpoint import save_checkpoint
    from vobj.geometry import AABB
    from vobj.models import ModelArch, adam_step, backward, forward, init_stacked
    from vobj.objects import Keyframe, ObjectMap

    def trained(k, hidden, seed):
        arch = ModelArch(n_layers=3, hidden=hidden, n_freq=2)
        p, s = init_stacked(arch, k, seed=seed)
        g = np.random.default_rng(seed + 1)
        for _ in range(2):
            x = g.standard_normal((k, 40, arch.input_dim)).astype(np.float32)
            _, cache = forward(p, x)
            gr = backward(p, cache, g.standard_normal((k, 40)).astype(np.float32),
                          g.standard_normal((k, 40, 3)).astype(np.float32))
            adam_step(p, s, gr)
        return p, s

    op, os_ = trained(3, 16, 5)
    bp, bs = trained(1, 32, 9)
    op.frozen[1] = True
    mp = ObjectMap()
    mp.add_background(AABB(np.array([-2.0, -2, -2]), np.array([2.0, 2, 2])), pe_scale=15.0, model_index=0)
    inst = mp.add_object(semantic_class=3, aabb=AABB(np.array([0.1, 0.2, 0.3]), np.array([0.4, 0.5, 0.6])),
                         pe_scale=10.0, model_index=0)
    inst.obs_count = 7
    inst.keyframes.append(Keyframe(frame_id=4, bbox=(1, 2, 10, 12), rgb=np.zeros((10, 9, 3), np.float32),
                                   depth=np.ones((10, 9), np.float32), mask=np.ones((10, 9), bool), pose=np.eye(4)))
    save_checkpoint(HERE / "ckpt_small.bin", op, os_, bp, bs, mp)


def main():
    vobj = import_reference()
    from vobj import models as M
    from vobj import render as Rn
    from vobj import trainer as T
    from vobj.objects import sample_training_pixels
    sys.path.insert(0, str(ROOT))
    from paper_2302_01838_b200.scenes import config, make_scene

    out = {}
    # ---- models: init, forward, backward, adam (models.py) ----------------
    g = np.random.default_rng(123)
    for tag, arch, k in (("h32", M.ModelArch(4, 32, 5), 3), ("h16l3", M.ModelArch(3, 16, 3), 2)):
        p, s = M.init_stacked(arch, k, seed=42)
        out[f"{tag}_init"] = flat(p)
        enc = g.uniform(-1, 1, (k, 57, arch.input_dim)).astype(np.float32)
        fo, cache = M.forward(p, enc)
        go = g.standard_normal((k, 57)).astype(np.float32)
        gc = g.standard_normal((k, 57, 3)).astype(np.float32)
        gr = M.backward(p, cache, go, gc)
        out[f"{tag}_enc"], out[f"{tag}_go"], out[f"{tag}_gc"] = enc, go, gc
        out[f"{tag}_occ"], out[f"{tag}_col"] = fo.occupancy, fo.colour
        out[f"{tag}_dW"] = np.concatenate([np.concatenate([gr.d_weights[l].reshape(k, -1), gr.d_biases[l]], 1)
                                           for l in range(arch.n_layers)], 1)
        mask = np.array([True, False, True][:k])
        M.set_frozen(p, 0, k > 2)
        for _ in range(3):
            M.adam_step(p, s, gr, update_mask=mask)
        out[f"{tag}_adam3"] = flat(p)
        out[f"{tag}_adam3_step"] = s.step[:k].copy()
    # ---- render + losses (render.py) ---------------------------------------
    R, S = 64, 10
    occ = g.uniform(0, 1, (R, S)).astype(np.float32)
    occ[0, 1] = 1.0
    col = g.uniform(0, 1, (R, S, 3)).astype(np.float32)
    t = np.sort(g.uniform(0.1, 8, (R, S)), axis=1).astype(np.float32)
    res = Rn.render_rays(occ, col, t)
    gO, gD, gC = (g.standard_normal(R).astype(np.float32), g.standard_normal(R).astype(np.float32),
                  g.standard_normal((R, 3)).astype(np.float32))
    d_occ, d_col = Rn.render_backward(occ, col, t, res, gO, gD, gC)
    out.update(r_occ=occ, r_col=col, r_t=t, r_O=res.opacity, r_D=res.depth, r_C=res.colour, r_w=res.weights,
               r_T=res.transmittance, r_gO=gO, r_gD=gD, r_gC=gC, r_docc=d_occ, r_dcol=d_col)
    tD = g.uniform(0, 4, R).astype(np.float32)
    tC = g.uniform(0, 1, (R, 3)).astype(np.float32)
    tm, tv, tok = g.random(R) < 0.6, g.random(R) < 0.8, g.random(R) < 0.9
    ld, lc, lo, lt = Rn.compute_losses(res, tD, tC, tm, tv, tok, Rn.LossWeights())
    dO, dD, dC = Rn.loss_output_grads(res, tD, tC, tm, tv, tok, Rn.LossWeights())
    out.update(l_tD=tD, l_tC=tC, l_m=tm, l_v=tv, l_ok=tok, l_ld=ld, l_lc=lc, l_lo=lo, l_lt=lt, l_dO=dO, l_dD=dD,
               l_dC=dC)
    np.savez_compressed(HERE / "ops.npz", **out)

    # ---- sampler + map-update on config 1 (trainer.py / objects.py) ---------
    scene = config("1")
    m = ref_mapper(vobj, scene)
    samp = {}
    for step in (0, 3):
        for k in range(m.obj_params.count):
            inst = m.instance_for_model(k)
            kf, u, v, hit = sample_training_pixels(inst, m.cfg.seed, step, m.cfg.rays_per_object)
            b = m._assemble_batch(inst, m.cfg.rays_per_object, step)
            pre = f"s{step}_o{k}_"
            samp.update({pre + "kf": kf, pre + "u": u, pre + "v": v, pre + "mask": hit, pre + "t": b.t,
                         pre + "ok": b.ray_ok, pre + "tdepth": b.target_depth, pre + "tcol": b.target_colour,
                         pre + "valid": b.valid_depth})
            if step == 0:
                samp[pre + "enc"] = b.encoded
        bg = m.map.background
        b = m._assemble_batch(bg, m.cfg.rays_background, step)
        pre = f"s{step}_bg_"
        samp.update({pre + "t": b.t, pre + "ok": b.ray_ok, pre + "tdepth": b.target_depth, pre + "tmask": b.target_mask})
        if step == 0:
            samp[pre + "enc200"] = b.encoded[:200]
    np.savez_compressed(HERE / "sampler_cfg1.npz", **samp)

    tr = {}
    losses = []
    for step in range(20):
        rep = m.train_step()
        losses.append([rep.losses[oid] for oid in sorted(rep.losses)])
    tr["losses"] = np.array(losses, np.float64)        # [20, 1+K, 3] sorted by object id (0 = bg)
    tr["obj_params"] = flat(m.obj_params)
    tr["bg_params"] = flat(m.bg_params)
    # the reference's own benchmark input (trainer.py:594-606) through train_on_batch
    for tag, arch, k, rays, pts in (("syn32", M.ModelArch(4, 32, 5), 5, 120, 10),
                                    ("syn16", M.ModelArch(3, 16, 3), 3, 24, 6)):
        p, s = M.init_stacked(arch, k, seed=11)
        batch = T._synthetic_batch(arch, k, rays, pts, seed=7)
        ls = [T.train_on_batch(p, s, batch, Rn.LossWeights()) for _ in range(20)]
        tr[f"{tag}_losses"] = np.array(ls)
        tr[f"{tag}_params"] = flat(p)
    np.savez_compressed(HERE / "train_cfg1.npz", **tr)

    # ---- forward-only inference on the trained config-1 map (meshing.py) ----
    from vobj.meshing import query_grid, render_view
    from vobj.render import CameraIntrinsics
    inf = {}
    o0 = m.instance_for_model(0)
    inf["grid_obj0"] = query_grid(m.obj_params, 0, o0.aabb.padded(0.10), o0.pe_scale, (9, 10, 11)).values
    bgi = m.map.background
    inf["grid_bg"] = query_grid(m.bg_params, bgi.model_index, bgi.aabb.padded(0.10), bgi.pe_scale, 8).values
    intr = scene["intrinsics"]
    ri = CameraIntrinsics(intr.fx, intr.fy, intr.cx, intr.cy, intr.width, intr.height)
    pose = scene["background"]["keyframes"][0]["pose"]
    for tag, thr in (("v", 0.5), ("v0", 0.0)):
        view = render_view(m.obj_params, m.bg_params, m.map, ri, pose, samples_object=16, samples_background=16,
                           samples_refine=8, threshold=thr)
        inf[tag + "_rgb"], inf[tag + "_depth"], inf[tag + "_inst"] = view.rgb, view.depth, view.instance
    np.savez_compressed(HERE / "infer_cfg1.npz", **inf)
    ingest_goldens(vobj)
    checkpoint_golden(vobj)
    import numpy
    (HERE / "PROVENANCE.txt").write_text(
        "Generated by tests/golden/make_golden.py from the reference at /root/reference/pkg/src\n"
        f"numpy {numpy.__version__}; scipy {__import__('scipy').__version__}\n")
    for f in ("ops.npz", "sampler_cfg1.npz", "train_cfg1.npz", "infer_cfg1.npz", "ingest.npz",
              "ckpt_small.bin"):
        print(f, (HERE / f).stat().st_size)


if __name__ == "__main__":
    main()
