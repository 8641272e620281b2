"""Deterministic RNG keys (drop-in for vobj/rng.py:15-34).

Host-side model initialisation draws from these numpy streams exactly like
the reference.  The training-step streams (PURPOSE_PIXELS, PURPOSE_SAMPLES)
are regenerated bit-exactly on the device by the CUDA sampler
(csrc/vm_sample.cu: SeedSequence -> PCG64 jump-ahead -> Lemire / ziggurat).
"""

from __future__ import annotations

import numpy as np

PURPOSE_INIT_OBJECT = 1
PURPOSE_INIT_BACKGROUND = 2
PURPOSE_PIXELS = 3
PURPOSE_SAMPLES = 4
PURPOSE_BENCH = 5
PURPOSE_EVAL = 6
PURPOSE_SYNTH = 7


def keyed_rng(seed: int, purpose: int, *extra: int) -> np.random.Generator:
    parts = (seed, purpose, *extra)
    for p in parts:
        if p < 0:
            raise ValueError(f"rng key parts must be non-negative, got {parts}")
    return np.random.default_rng(np.random.SeedSequence(parts))
