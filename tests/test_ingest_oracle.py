"""Per-frame ingestion oracle (oracle.vobj_oracle IngestMap / extract_detections
/ scene_bounds / associate) and the drop-in Dataset reader, pinned to the
reference's own outputs on datasets its synthetic generator wrote
(tests/golden/ds_*, ingest.npz).  CPU only."""

from pathlib import Path

import numpy as np
import pytest

from oracle import vobj_oracle as O
from paper_2302_01838_b200.datasets import Dataset
from paper_2302_01838_b200.objects import AssociationConfig

G = Path(__file__).resolve().parent / "golden"
STRIDES = dict(keyframe_stride_object=2, keyframe_stride_background=3)


@pytest.fixture(scope="module")
def gold():
    return np.load(G / "ingest.npz")


def _close(a, b):
    np.testing.assert_allclose(np.asarray(a, np.float64), b, rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("name", ["ds_mini", "ds_five"])
def test_ingestion_oracle_matches_reference(gold, name):
    ds = Dataset(G / name)
    acfg = AssociationConfig(**STRIDES)
    im = O.IngestMap(ds.intrinsics, stride_object=acfg.keyframe_stride_object,
                     stride_background=acfg.keyframe_stride_background, margin=acfg.bbox_margin_px,
                     min_pixels=acfg.min_pixels, trim=acfg.outlier_trim, iou_threshold=acfg.iou_threshold)
    for i in range(len(ds)):
        fr = ds.frame(i)
        pre = f"{name}_f{i}_"
        dets, sb = im.process_frame(fr.frame_id, fr.rgb, fr.depth, fr.mask, fr.pose, ds.classes)
        _close(np.concatenate([sb.min, sb.max]), gold[pre + "scene"])
        np.testing.assert_array_equal(np.array([d["bbox"] for d in dets]).reshape(-1, 4), gold[pre + "det_bbox"])
        np.testing.assert_array_equal([d["n_pixels"] for d in dets], gold[pre + "det_n"])
        np.testing.assert_array_equal([d["cls"] for d in dets], gold[pre + "det_cls"])
        _close(np.array([np.concatenate([d["aabb"].min, d["aabb"].max]) for d in dets]).reshape(-1, 6),
               gold[pre + "det_box"])
        np.testing.assert_array_equal([o.object_id for o in im.objects], gold[pre + "obj_ids"])
        _close(np.array([np.concatenate([o.aabb.min, o.aabb.max]) for o in im.objects]).reshape(-1, 6),
               gold[pre + "obj_box"])
        np.testing.assert_array_equal([o.obs for o in im.objects], gold[pre + "obj_obs"])
        kf = np.array([[f, *b, o.object_id] for o in im.objects for f, b in o.kfs]).reshape(-1, 6)
        np.testing.assert_array_equal(kf, gold[pre + "obj_kf"])
        _close(np.concatenate([im.background.aabb.min, im.background.aabb.max]), gold[pre + "bg_box"])
        np.testing.assert_array_equal([f for f, _ in im.background.kfs], gold[pre + "bg_kf"])


def test_dataset_reader_matches_reference_conversions():
    """datasets.py:155-175: f32 RGB / 255 (BGR flipped), depth / depth_scale."""
    import cv2
    ds = Dataset(G / "ds_five")
    fr = ds.frame(2)
    bgr = cv2.imread(str(G / "ds_five" / "rgb" / "000002.png"), cv2.IMREAD_COLOR)
    d16 = cv2.imread(str(G / "ds_five" / "depth" / "000002.png"), cv2.IMREAD_UNCHANGED)
    np.testing.assert_array_equal(fr.rgb, bgr[:, :, ::-1].astype(np.float32) / 255.0)
    np.testing.assert_array_equal(fr.depth, d16.astype(np.float32) / ds.depth_scale)
    assert fr.mask.dtype == np.int32 and len(ds) == 6 and ds.classes
    with pytest.raises(IndexError):
        ds.frame(6)
