"""VOBJ v1 checkpoints from / into the device arena (checkpoint.py:1-169):

* a file written by the reference (tests/golden/ckpt_small.bin: hidden-16 and
  hidden-32 stacks, a frozen model, keyframe references) loads into device
  stacks and saves back byte-identical (test_checkpoint.py:100-107's
  byte-stability contract, across implementations);
* a GPU-trained map (config 1, 3 steps) round-trips bit-exactly (parameters,
  Adam moments, steps, frozen flags, object table) and the file is stable.
"""

from pathlib import Path

import numpy as np
import pytest
import torch

from paper_2302_01838_b200 import TrainConfig
from paper_2302_01838_b200.checkpoint import load_checkpoint, save_checkpoint
from paper_2302_01838_b200.mapper import Mapper
from paper_2302_01838_b200.objects import Keyframe
from paper_2302_01838_b200.scenes import config, populate

pytestmark = pytest.mark.gpu
G = Path(__file__).resolve().parent / "golden"


def _reattach(mp, refs):
    """Keyframes come back as (frame_id, bbox) references (checkpoint.py:
    150-154); re-attach them (pixels would be re-hydrated from the dataset)."""
    for oid, rr in zip(sorted(mp.instances), refs):
        for fid, bbox in rr:
            h, w = bbox[3] - bbox[1], bbox[2] - bbox[0]
            mp.instances[oid].keyframes.append(Keyframe(frame_id=fid, pose=np.eye(4), bbox=bbox,
                                                        mask=np.ones((h, w), bool), rgb=np.zeros((h, w, 3), np.float32),
                                                        depth=np.ones((h, w), np.float32)))


def test_reference_file_round_trips_byte_identical(cuda, tmp_path):
    op, os_, bp, bs, mp, refs = load_checkpoint(G / "ckpt_small.bin")
    assert op.count == 3 and op.arch.hidden == 16 and bp.count == 1 and bp.arch.hidden == 32
    assert op.frozen[:3].tolist() == [False, True, False]
    assert [r for r in refs if r] == [[(4, (1, 2, 10, 12))]]
    assert mp.instances[1].obs_count == 7 and mp.instances[0].is_background
    _reattach(mp, refs)
    out = tmp_path / "again.bin"
    save_checkpoint(out, op, os_, bp, bs, mp)
    assert out.read_bytes() == (G / "ckpt_small.bin").read_bytes()


def test_trained_map_round_trip(cuda, tmp_path):
    scene = config("1")
    m = Mapper(scene["intrinsics"], TrainConfig())
    populate(m, scene)
    for _ in range(3):
        m.train_step()
    m.obj_params.frozen[2] = True
    p1 = tmp_path / "a.bin"
    save_checkpoint(p1, m.obj_params, m.obj_state, m.bg_params, m.bg_state, m.map)
    op, os_, bp, bs, mp, refs = load_checkpoint(p1)
    for a, b in ((m.obj_params, op), (m.bg_params, bp)):
        k = a.count
        for l in range(a.arch.n_layers):
            assert torch.equal(a.weights[l][:k], b.weights[l][:k])
            assert torch.equal(a.biases[l][:k], b.biases[l][:k])
        assert np.array_equal(a.frozen[:k], b.frozen[:k])
    for a, b in ((m.obj_state, os_), (m.bg_state, bs)):
        k = int((a.step > 0).sum()) or 1
        for l in range(a.arch.n_layers):
            assert torch.equal(a.m_weights[l][:k], b.m_weights[l][:k])
            assert torch.equal(a.v_biases[l][:k], b.v_biases[l][:k])
        assert torch.equal(a.step[:k], b.step[:k])
    assert sorted(mp.instances) == sorted(m.map.instances)
    assert [len(r) for r in refs] == [len(m.map.instances[i].keyframes) for i in sorted(m.map.instances)]
    _reattach(mp, refs)
    p2 = tmp_path / "b.bin"
    save_checkpoint(p2, op, os_, bp, bs, mp)
    assert p1.read_bytes() == p2.read_bytes()


def test_bad_files_rejected(cuda, tmp_path):
    bad = tmp_path / "x.bin"
    bad.write_bytes(b"NOPE" + bytes(8))
    with pytest.raises(ValueError, match="magic"):
        load_checkpoint(bad)
    raw = (G / "ckpt_small.bin").read_bytes()
    bad.write_bytes(raw[:-3])
    with pytest.raises(ValueError, match="truncated"):
        load_checkpoint(bad)
    bad.write_bytes(raw + b"\0")
    with pytest.raises(ValueError, match="trailing"):
        load_checkpoint(bad)
