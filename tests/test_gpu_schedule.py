"""The step's launch schedule never changes its bits: the persistent work
queue, programmatic dependent launch, the capture order of the sampler, KT
launched first and the serial (unforked) order all give parameters, Adam
state and losses identical to the default schedule, bit for bit (every
reduction has a fixed order that does not depend on which CTA or stream ran
it)."""

import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]

SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
from paper_2302_01838_b200 import TrainConfig
from paper_2302_01838_b200.mapper import Mapper
from paper_2302_01838_b200.scenes import config, populate
scene = config("1")
m = Mapper(scene["intrinsics"], TrainConfig())
populate(m, scene)
losses = []
for _ in range(3):
    rep = m.train_step()
    losses.append([rep.losses[k] for k in sorted(rep.losses)])
torch.cuda.synchronize()
np.savez(sys.argv[2], obj=m.obj_params.arena.cpu().numpy(), bg=m.bg_params.arena.cpu().numpy(),
         om=m.obj_state.m_arena.cpu().numpy(), bv=m.bg_state.v_arena.cpu().numpy(), losses=np.array(losses))
"""

VARIANTS = [{}, {"VM_KF_PERSIST": "0"}, {"VM_PDL": "0"}, {"VM_SAMPLE_FIRST": "1"}, {"VM_KT_FIRST": "2"},
            {"VM_NO_FORK": "1"}]


def test_schedule_variants_are_bit_identical(cuda, tmp_path):
    outs = []
    for i, v in enumerate(VARIANTS):
        out = tmp_path / f"v{i}.npz"
        env = dict(os.environ, **v)
        r = subprocess.run([sys.executable, "-c", SCRIPT, str(ROOT), str(out)], env=env, capture_output=True,
                           text=True, timeout=600)
        assert r.returncode == 0, f"{v}: {r.stderr[-2000:]}"
        outs.append(np.load(out))
    ref = outs[0]
    for v, o in zip(VARIANTS[1:], outs[1:]):
        for key in ("obj", "bg", "om", "bv", "losses"):
            np.testing.assert_array_equal(o[key], ref[key], err_msg=f"{v} {key}")
