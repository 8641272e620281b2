"""The C-ABI library loads and exports every entry point include/vmap_b200.h
declares; host-only helpers (layout) agree with the Python mirror.  CPU only:
no compute call touches the GPU here."""

import ctypes as C
import re
from pathlib import Path

import pytest

from paper_2302_01838_b200 import _lib

HDR = Path(__file__).resolve().parents[1] / "include" / "vmap_b200.h"


def declared():
    txt = re.sub(r"/\*.*?\*/", "", HDR.read_text(), flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\**\s+\**(vm_\w+)\s*\(", txt, flags=re.M)))


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    names = declared()
    assert len(names) >= 15
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(_lib.EXPORTED)
    assert lib.vm_version().startswith(b"vmap_b200")


@pytest.mark.parametrize("n_layers,hidden,d,block,n", [(4, 32, 33, 3428, 3332), (4, 128, 33, 38276, 37892),
                                                       (3, 16, 21, 24 * 32 + 32 + 32 * 32 + 32 + 4 * 32 + 4, 3 * 0 + 16 * 21 + 16 + 16 * 16 + 16 + 4 * 16 + 4)])
def test_layout(n_layers, hidden, d, block, n):
    L = _lib.layout(n_layers, hidden, d)
    assert L.block == block and L.n_params == n
    assert all(L.w_off[l] % 4 == 0 and L.b_off[l] % 4 == 0 for l in range(n_layers))


def test_layout_rejects_bad_arch():
    with pytest.raises(ValueError):
        _lib.layout(1, 32, 33)
    with pytest.raises(NotImplementedError):
        _lib.layout(4, 1 << 17, 33)
    with pytest.raises(ValueError):
        _lib.layout(9, 32, 33)  # > VM_MAX_LAYERS


def test_layout_wide_models():
    """Widths above 128 (layered path): hidden rows padded to a multiple of 32."""
    L = _lib.layout(4, 200, 63)
    assert L.hidden_pad == 224
    assert list(L.fi_pad[:4]) == [64, 224, 224, 224] and list(L.fo_pad[:4]) == [224, 224, 224, 4]
    assert L.n_params == 200 * 63 + 200 + 2 * (200 * 200 + 200) + 4 * 200 + 4


def _plan_bytes(archs, rays, points):
    """vm_train_workspace_bytes for stacks of the given (n_layers, hidden,
    n_freq) architectures -- host-only planning, no device pointer is read."""
    lib = _lib.load()
    n = len(archs)
    vs = (_lib.VmStack * n)()
    vb = (_lib.VmBatch * n)()
    for i, (nl, h, f) in enumerate(archs):
        d = 3 + 6 * f
        vs[i].arch = _lib.VmArch(nl, h, d, 0)
        vs[i].count = vs[i].capacity = 2
        vb[i].n_models, vb[i].n_rays, vb[i].n_points, vb[i].input_dim = 2, rays, points, d
        vb[i].encoded = 16  # non-null: the layered path takes the encoded input
    return lib.vm_train_workspace_bytes(vs, vb, n)


def test_train_planning_routes_wide_models_to_the_layered_path():
    """The fused plan for the config-2 stacks; the layered plan (all layer
    activations kept for the backward: (L-1) x K x R*S x hidden_pad floats
    and more) for widths / sample counts the fused kernels lack; the hybrid
    (fused objects + layered background) in between."""
    fused = _plan_bytes([(4, 32, 5), (4, 128, 5)], 120, 10)
    assert fused > 0
    acts = 3 * 2 * 120 * 10 * 256 * 4
    wide = _plan_bytes([(4, 256, 5)], 120, 10)
    assert wide > acts
    assert _plan_bytes([(4, 64, 5)], 30, 40) > 3 * 2 * 30 * 40 * 64 * 4  # 40 samples per ray
    hybrid = _plan_bytes([(4, 32, 5), (4, 256, 5)], 120, 10)
    assert hybrid >= _plan_bytes([(4, 32, 5)], 120, 10) + wide
    assert _plan_bytes([(4, 32, 5)], 120, 65) == 0  # > 64 samples per ray: rejected
