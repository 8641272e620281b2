"""The pure-Python restatement of numpy's streams (the device RNG's spec)
against numpy itself (bit-exact).  CPU only."""

import numpy as np
import pytest

from oracle import numpy_rng as R

KEYS = [(0, 3, 7, 11), (0, 4, 1, 0), (5, 4, 123456789, 2 ** 40), (2 ** 33 + 5, 3, 0, 0), (0, 4, 0, 0)]


@pytest.mark.parametrize("key", KEYS)
def test_seed_sequence_and_pcg64(key):
    s, inc = R.pcg64_seed(key)
    st = np.random.PCG64(np.random.SeedSequence(key)).state["state"]
    assert (st["state"], st["inc"]) == (s, inc)
    raw = np.random.PCG64(np.random.SeedSequence(key)).random_raw(64)
    stream = R.Stream(key)
    assert [stream.next64() for _ in range(64)] == [int(x) for x in raw]
    assert R.Stream(key).word_at(41) == int(raw[41])


def test_survey_test_vectors():
    s, inc = R.pcg64_seed((0, 3, 7, 11))
    assert s == 0x78ACDFE786B248FD7E0B75F609C46263 and inc == 0x359D0F16090E1C9E5F25959D22673F97
    st = R.Stream((0, 3, 7, 11))
    assert st.next64() == 0x7687802B01B6B79B and st.next64() == 0x123F8D9E12A70537


@pytest.mark.parametrize("n", [1, 2, 5, 7, 10])
def test_integers_then_random_layout(n):
    key = (0, 3, 9, n)
    g = np.random.default_rng(np.random.SeedSequence(key))
    a, b = g.integers(0, n, size=61), g.random((61, 2))
    st = R.Stream(key)
    assert list(a) == R.integers(st, n, 61)
    assert np.array_equal(b.ravel(), np.array([st.next_double() for _ in range(122)]))


@pytest.mark.parametrize("key", KEYS[:3])
def test_ziggurat_normals(key):
    tabs = R.load_ziggurat_tables()
    g = np.random.default_rng(np.random.SeedSequence(key))
    z = g.standard_normal(6000)
    st = R.Stream(key)
    assert np.array_equal(z, np.array([R.standard_normal(st, tabs) for _ in range(6000)]))
    assert st.pos > 6000  # slow-path draws consume extra words
