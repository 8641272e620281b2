"""Synthetic scenes for the BASELINE.json configurations (host numpy data).

There is no dataset access, so the workloads are synthetic RGB-D keyframes
with the reference's shapes (SURVEY 8d / appendix "Config-2 generator"):
one shared random frame (rgb U(0,1), depth U(0.5,4) m), five look-at poses
on a 3 m orbit, a full-frame background with mask U<0.7 per keyframe, and per
object a random box (centre U(-1.5,1.5)^3, half-extent U(0.1,0.3)^3) with
keyframe crops of 60-140 px and mask U<0.6.  A scene is a plain dict so the
same data can populate this package's Mapper and the CPU oracle.
"""

from __future__ import annotations

import numpy as np

from .geometry import AABB, look_at
from .render import CameraIntrinsics


def make_scene(n_objects: int, n_kf: int = 5, width: int = 1200, height: int = 680, focal: float = 600.0,
               crop=(60, 140), n_kf_bg: int = 5, seed: int = 0, with_background: bool = True) -> dict:
    rng = np.random.default_rng(seed)
    intr = CameraIntrinsics(fx=focal, fy=focal, cx=width / 2 - 0.5, cy=height / 2 - 0.5, width=width,
                            height=height)
    rgb = rng.random((height, width, 3), dtype=np.float32)
    depth = (0.5 + 3.5 * rng.random((height, width))).astype(np.float32)
    angles = np.linspace(0.0, 2 * np.pi, max(n_kf, n_kf_bg), endpoint=False)
    poses = [look_at((3 * np.cos(a), 3 * np.sin(a), 1.5), (0.0, 0.0, 0.0)) for a in angles]
    scene = dict(intrinsics=intr, rgb=rgb, depth=depth, background=None, objects=[])
    if with_background:
        kfs = [dict(frame_id=j, pose=poses[j], bbox=(0, 0, width, height),
                    mask=rng.random((height, width)) < 0.7) for j in range(n_kf_bg)]
        scene["background"] = dict(aabb=AABB((-3.0, -3.0, -1.0), (3.0, 3.0, 3.0)), keyframes=kfs)
    for _ in range(n_objects):
        c = rng.uniform(-1.5, 1.5, 3)
        h = rng.uniform(0.1, 0.3, 3)
        kfs = []
        for j in range(n_kf):
            cw, ch = (int(x) for x in rng.integers(crop[0], crop[1], 2))
            cw, ch = min(cw, width), min(ch, height)
            u0 = int(rng.integers(0, width - cw + 1))
            v0 = int(rng.integers(0, height - ch + 1))
            kfs.append(dict(frame_id=j, pose=poses[j], bbox=(u0, v0, u0 + cw, v0 + ch),
                            mask=rng.random((ch, cw)) < 0.6))
        scene["objects"].append(dict(aabb=AABB(c - h, c + h), keyframes=kfs))
    return scene


def config(name: str) -> dict:
    """BASELINE.json configs by number ("1".."5"); sizes per SURVEY 8d."""
    if name == "1":   # oracle case: 3 objects + bg, 20 steps on CPU
        return make_scene(3, n_kf=2, width=160, height=120, focal=100.0, crop=(20, 60), n_kf_bg=2, seed=1)
    if name in ("2", "5"):
        return make_scene(50, n_kf=5, seed=0)
    if name == "3":   # load-imbalance stress: per-object rays log-uniform in [30, 480]
        sc = make_scene(200, n_kf=10, seed=3)
        g = np.random.default_rng(33)
        for ob, r in zip(sc["objects"], np.exp(g.uniform(np.log(30), np.log(480), len(sc["objects"])))):
            ob["n_rays"] = int(round(r))
        return sc
    if name == "4":
        return make_scene(1000, n_kf=5, seed=4)
    raise KeyError(f"unknown config {name!r}")


def populate(mapper, scene: dict, objects=None, with_background: bool = True) -> None:
    """Register the scene's background/objects/keyframes in a Mapper.

    ``objects`` optionally restricts to a subset of object indices (a rank's
    share under multi-GPU object sharding): object i then keeps its global id
    i + 1 and global init index i, exactly as in the unsharded map.
    """
    if scene["background"] is not None and with_background:
        bg = mapper.add_background(scene["background"]["aabb"])
        for kf in scene["background"]["keyframes"]:
            mapper.add_keyframe(bg, kf["frame_id"], kf["pose"], kf["bbox"], kf["mask"], scene["rgb"],
                                scene["depth"])
    for i, ob in enumerate(scene["objects"]):
        if objects is not None and i not in objects:
            continue
        if objects is None:
            inst = mapper.add_object(1, ob["aabb"], n_rays=ob.get("n_rays"))
        else:
            inst = mapper.add_object(1, ob["aabb"], object_id=i + 1, init_index=i, n_rays=ob.get("n_rays"))
        for kf in ob["keyframes"]:
            mapper.add_keyframe(inst, kf["frame_id"], kf["pose"], kf["bbox"], kf["mask"], scene["rgb"],
                                scene["depth"])
