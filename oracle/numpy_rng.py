"""Pure-Python restatement of the numpy random streams the hot path consumes.

TEST INFRASTRUCTURE ONLY (see oracle/vobj_oracle.py header).

The reference draws every random number through
`np.random.default_rng(np.random.SeedSequence((seed, purpose, obj, step)))`
(`/root/reference/pkg/src/vobj/rng.py:24-34`).  That algorithm lives in the
third-party dependency numpy (installed here: numpy 2.3.5; pyproject lower
bound `numpy>=1.24`, `/root/reference/pkg/pyproject.toml:10-16`).  This file
restates numpy's published algorithms from scratch so the CUDA sampler has a
readable spec; `tests/test_numpy_rng.py` pins every function against numpy
itself (bit-exact):

* SeedSequence entropy pool + generate_state (numpy/random/bit_generator.pyx)
* PCG64 (XSL-RR 128/64) seeding, stepping, jump-ahead
* Generator.integers(0, n) for int64 with n <= 2**32: 32-bit Lemire over the
  low then high half of each 64-bit output (objects.py:336)
* Generator.random(): (next64 >> 11) * 2**-53 (objects.py:337, render.py:184)
* Generator.standard_normal(): 256-layer ziggurat (render.py:185), tables
  extracted from numpy's libnpyrandom.a by oracle/gen_ziggurat_tables.py
"""

from __future__ import annotations

import math

M32 = 0xFFFFFFFF
M64 = (1 << 64) - 1
M128 = (1 << 128) - 1
PCG_MULT = (2549297995355413924 << 64) + 4865540595714422341

# SeedSequence hash constants (numpy/random/bit_generator.pyx)
INIT_A, MULT_A = 0x43B0D7E5, 0x931E8875
INIT_B, MULT_B = 0x8B51F9DD, 0x58F38DED
MIX_L, MIX_R = 0xCA01F9DD, 0x4973F715
POOL = 4


def _entropy_words(parts) -> list[int]:
    words = []
    for p in parts:
        if p < 0:
            raise ValueError("negative entropy")
        if p == 0:
            words.append(0)
        while p:
            words.append(p & M32)
            p >>= 32
    return words


def seed_state(parts, n_words: int = 8) -> list[int]:
    """SeedSequence(parts).generate_state(n_words, uint32)."""
    hc = INIT_A

    def hashmix(v):
        nonlocal hc
        v = (v ^ hc) & M32
        hc = (hc * MULT_A) & M32
        v = (v * hc) & M32
        return (v ^ (v >> 16)) & M32

    def mix(x, y):
        r = (MIX_L * x - MIX_R * y) & M32
        return (r ^ (r >> 16)) & M32

    ent = _entropy_words(parts)
    pool = [hashmix(ent[i] if i < len(ent) else 0) for i in range(POOL)]
    for s in range(POOL):
        for d in range(POOL):
            if s != d:
                pool[d] = mix(pool[d], hashmix(pool[s]))
    for e in ent[POOL:]:
        for d in range(POOL):
            pool[d] = mix(pool[d], hashmix(e))
    hb = INIT_B
    out = []
    for i in range(n_words):
        v = pool[i % POOL] ^ hb
        hb = (hb * MULT_B) & M32
        v = (v * hb) & M32
        out.append((v ^ (v >> 16)) & M32)
    return out


def pcg64_seed(parts) -> tuple[int, int]:
    """(state, inc) of PCG64(SeedSequence(parts))."""
    w = seed_state(parts, 8)
    u64 = [w[2 * i] | (w[2 * i + 1] << 32) for i in range(4)]
    initstate = (u64[0] << 64) | u64[1]
    initseq = (u64[2] << 64) | u64[3]
    inc = ((initseq << 1) | 1) & M128
    s = (0 * PCG_MULT + inc) & M128
    s = (s + initstate) & M128
    s = (s * PCG_MULT + inc) & M128
    return s, inc


def pcg64_output(state: int) -> int:
    """XSL-RR of a 128-bit state."""
    hi, lo = state >> 64, state & M64
    x = hi ^ lo
    rot = hi >> 58
    return ((x >> rot) | (x << ((64 - rot) & 63))) & M64


def pcg64_advance(state: int, inc: int, delta: int) -> int:
    """State after `delta` LCG steps (Brown's O(log n) jump)."""
    acc_mult, acc_plus = 1, 0
    cur_mult, cur_plus = PCG_MULT, inc
    while delta:
        if delta & 1:
            acc_mult = (acc_mult * cur_mult) & M128
            acc_plus = (acc_plus * cur_mult + cur_plus) & M128
        cur_plus = ((cur_mult + 1) * cur_plus) & M128
        cur_mult = (cur_mult * cur_mult) & M128
        delta >>= 1
    return (acc_mult * state + acc_plus) & M128


class Stream:
    """Word-addressable PCG64 stream: word(i) is the i-th next_uint64()."""

    def __init__(self, parts):
        self.state0, self.inc = pcg64_seed(parts)
        self.state = self.state0
        self.pos = 0

    def word_at(self, i: int) -> int:
        return pcg64_output(pcg64_advance(self.state0, self.inc, i + 1))

    def next64(self) -> int:
        self.state = (self.state * PCG_MULT + self.inc) & M128
        self.pos += 1
        return pcg64_output(self.state)

    def next_double(self) -> float:
        return (self.next64() >> 11) * (1.0 / 9007199254740992.0)


def lemire32(x32: int, n: int) -> tuple[int, bool]:
    """One bounded draw in [0, n) from a 32-bit word; (value, needs_redraw)."""
    m = x32 * n
    left = m & M32
    if left < n:
        thr = (M32 - (n - 1)) % n
        if left < thr:
            return 0, True
    return m >> 32, False


def integers(st: Stream, n: int, size: int) -> list[int]:
    """Generator.integers(0, n, size) for n <= 2**32 (low half first)."""
    if n == 1:
        return [0] * size
    out, buf, have = [], 0, False
    while len(out) < size:
        if have:
            x, have = buf, False
        else:
            w = st.next64()
            x, buf, have = w & M32, w >> 32, True
        v, redraw = lemire32(x, n)
        if not redraw:
            out.append(v)
    return out


def load_ziggurat_tables():
    from pathlib import Path
    import re
    src = (Path(__file__).resolve().parents[1] / "paper_2302_01838_b200" / "csrc"
           / "ziggurat_tables.h").read_text()

    def grab(name, conv):
        body = re.search(name + r"\[256\] = \{(.*?)\};", src, re.S).group(1)
        return [conv(tok) for tok in re.findall(r"0x[0-9a-fA-F]+", body)]

    import struct
    ki = grab("vm_zig_ki", lambda s: int(s, 16))
    as_f64 = lambda s: struct.unpack("<d", struct.pack("<Q", int(s, 16)))[0]
    return ki, grab("vm_zig_wi", as_f64), grab("vm_zig_fi", as_f64)


ZIG_R = 3.6541528853610087963519472518
ZIG_INV_R = 0.27366123732975827203338247596


def standard_normal(st: Stream, tables) -> float:
    """numpy random_standard_normal (ziggurat, 256 layers, 52-bit mantissa)."""
    ki, wi, fi = tables
    while True:
        r = st.next64()
        idx = r & 0xFF
        r >>= 8
        sign = r & 1
        rabs = (r >> 1) & 0x000FFFFFFFFFFFFF
        x = rabs * wi[idx]
        if sign:
            x = -x
        if rabs < ki[idx]:
            return x
        if idx == 0:
            while True:
                xx = -ZIG_INV_R * math.log1p(-st.next_double())
                yy = -math.log1p(-st.next_double())
                if yy + yy > xx * xx:
                    return -(ZIG_R + xx) if (rabs >> 8) & 1 else ZIG_R + xx
        elif (fi[idx - 1] - fi[idx]) * st.next_double() + fi[idx] < math.exp(-0.5 * x * x):
            return x
