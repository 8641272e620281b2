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
