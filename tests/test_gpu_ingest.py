"""Per-frame ingestion and the mapping loop on the GPU vs the reference's own
outputs (tests/golden/ingest.npz) on datasets its generator wrote:

* vm_decode_frame == Dataset.frame's conversions, bit for bit;
* device extract_detections / scene_bounds: 2D boxes and pixel counts exact,
  3D boxes within 1e-12 (the device backprojects without BLAS's FMA order);
* Mapper.process_frame: object ids, boxes, observation counts and keyframes
  after every frame equal to the reference's;
* run_mapping (ingest + 2 train steps per frame): every step's losses within
  rtol 1e-4 and the final parameters within 1e-4 relative L2 per model.
"""

from pathlib import Path

import numpy as np
import pytest
import torch

from paper_2302_01838_b200 import TrainConfig
from paper_2302_01838_b200.datasets import Dataset, DeviceFrame
from paper_2302_01838_b200.ingest import FrameIngestor, extract_detections_device
from paper_2302_01838_b200.mapper import Mapper, run_mapping
from paper_2302_01838_b200.objects import AssociationConfig

from .helpers import flat_params, rel_l2

pytestmark = pytest.mark.gpu
G = Path(__file__).resolve().parent / "golden"
STRIDES = dict(keyframe_stride_object=2, keyframe_stride_background=3)
NAMES = ["ds_mini", "ds_five"]


@pytest.fixture(scope="module")
def gold():
    return np.load(G / "ingest.npz")


def _close(a, b):
    np.testing.assert_allclose(np.asarray(a, np.float64), b, rtol=1e-12, atol=1e-12)


def test_device_decode_matches_dataset_frame(cuda):
    ds = Dataset(G / "ds_five")
    for i in (0, 3):
        fr = ds.frame(i)
        df = DeviceFrame(i, *ds.frame_raw(i), fr.pose, ds.depth_scale, "cuda")
        np.testing.assert_array_equal(df.rgb.cpu().numpy(), fr.rgb)
        np.testing.assert_array_equal(df.depth.cpu().numpy(), fr.depth)
        np.testing.assert_array_equal(df.mask.cpu().numpy(), fr.mask)


@pytest.mark.parametrize("name", NAMES)
def test_device_detections_match_reference(cuda, gold, name):
    ds = Dataset(G / name)
    acfg = AssociationConfig(**STRIDES)
    ing = FrameIngestor("cuda")
    for i in range(len(ds)):
        fr = ds.frame(i)
        pre = f"{name}_f{i}_"
        dets, sb = extract_detections_device(ing, fr, ds.intrinsics, ds.classes, acfg)
        _close(np.concatenate([sb.min, sb.max]), gold[pre + "scene"])
        np.testing.assert_array_equal(np.array([d.bbox for d in dets]).reshape(-1, 4), gold[pre + "det_bbox"])
        np.testing.assert_array_equal([d.n_pixels for d in dets], gold[pre + "det_n"])
        np.testing.assert_array_equal([d.semantic_class for d in dets], gold[pre + "det_cls"])
        _close(np.array([np.concatenate([d.aabb.min, d.aabb.max]) for d in dets]).reshape(-1, 6),
               gold[pre + "det_box"])


@pytest.mark.parametrize("name", NAMES)
def test_process_frame_matches_reference(cuda, gold, name):
    ds = Dataset(G / name)
    m = Mapper(ds.intrinsics, TrainConfig(association=AssociationConfig(**STRIDES)))
    for i in range(len(ds)):
        m.process_frame(ds.frame(i), ds.classes)
        pre = f"{name}_f{i}_"
        objs = [m.map.instances[o] for o in m.model_to_object]
        np.testing.assert_array_equal([o.object_id for o in objs], gold[pre + "obj_ids"])
        _close(np.array([np.concatenate([o.aabb.min, o.aabb.max]) for o in objs]).reshape(-1, 6),
               gold[pre + "obj_box"])
        np.testing.assert_array_equal([o.obs_count for o in objs], gold[pre + "obj_obs"])
        kf = np.array([[k.frame_id, *k.bbox, o.object_id] for o in objs for k in o.keyframes]).reshape(-1, 6)
        np.testing.assert_array_equal(kf, gold[pre + "obj_kf"])
        bg = m.map.background
        _close(np.concatenate([bg.aabb.min, bg.aabb.max]), gold[pre + "bg_box"])
        np.testing.assert_array_equal([k.frame_id for k in bg.keyframes], gold[pre + "bg_kf"])
    assert m.frames_seen == len(ds) and m.last_frame_id == len(ds) - 1


@pytest.mark.parametrize("name", NAMES)
def test_run_mapping_matches_reference(cuda, gold, name):
    ds = Dataset(G / name)
    cfg = TrainConfig(association=AssociationConfig(**STRIDES), rays_per_object=48, rays_background=96,
                      steps_per_frame=2)
    m, reports = run_mapping(ds, cfg)
    ids, losses = gold[f"{name}_map_ids"], gold[f"{name}_map_losses"]
    assert len(reports) == ids.shape[0]
    for j, r in enumerate(reports):
        keys = [int(k) for k in ids[j] if k >= 0]
        assert sorted(r.losses) == keys
        got = np.array([r.losses[k] for k in keys])
        np.testing.assert_allclose(got, losses[j, :len(keys)], rtol=1e-4, atol=1e-5, err_msg=f"step {j}")
    for part, params in (("obj", m.obj_params), ("bg", m.bg_params)):
        ref = gold[f"{name}_map_{part}_params"].astype(np.float64)
        e = rel_l2(flat_params(params), ref)
        print(name, part, "rel L2 after run_mapping", e.max())
        assert e.max() <= 1e-4
