"""Test configuration.

`-m gpu` tests need a CUDA device and the in-tree libvmap_b200.so; everything
else runs on CPU (oracle vs golden vectors, host logic, C-ABI exports, gloo
multi-process paths).  The oracle under oracle/ is test infrastructure only.
"""

import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200) and the built CUDA library")


@pytest.fixture(scope="session")
def cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2302_01838_b200 import _lib
    _lib.load()  # fail loudly if the extension is missing
    return torch.device("cuda")
