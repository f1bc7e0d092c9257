"""CPU restatement of the reference's synthetic teacher (TEST INFRASTRUCTURE).

Only tests/ import this module; the product path is
paper_2511_10676_b200.synthgen over the K11 kernels in csrc/synthgen.cu.

What it restates:
  * pkg/src/moepredict/synthgen.py:44-47  `_rng`: sample i draws from
    numpy.random.Generator(Philox(key=(seed << 64) + i)).
  * pkg/src/moepredict/synthgen.py:162-189 `generate_dataset`: per-sample
    standard normals (activation, then noise from the same stream), teacher
    transform, noise, layer_norm (core.py:57-68), gate softmax
    (core.py:117-127, :19-24), float32 cast + top-k labels (make_dataset,
    synthgen.py:148-159).
  * Third-party arithmetic the reference calls (not in /root/reference):
    numpy 2.3.5 `Philox` = Random123 Philox4x64-10 (counter incremented
    before each 4-word block, key = (low 64, high 64) of the 128-bit key),
    and `Generator.standard_normal` = numpy's 256-layer ziggurat
    (random_standard_normal: 8 index bits, 1 sign bit, 52 mantissa bits per
    64-bit draw; tail from -log1p(-U) pairs; wedge test against
    exp(-x^2/2)). The ziggurat tables are read out of the installed numpy by
    driving its Philox state (`extract_tables`), not copied from its source.
  * numpy's add.reduce along a contiguous axis = 0 + pairwise_sum (8
    accumulators per block of <= 128, halving split rounded to a multiple of
    8) — `pairwise_sum`, checked against np.sum / mean / var in
    tests/test_oracle_golden.py.

Pinned by tests/test_oracle_golden.py against numpy itself (raw Philox words,
standard normals) and against tests/golden/synthgen_golden.npz written by the
real reference (tests/golden/make_golden.py).
"""

from __future__ import annotations

import math

import numpy as np

MASK64 = (1 << 64) - 1
PHILOX_M = (0xD2E7470EE14C6C93, 0xCA5A826395121157)
PHILOX_W = (0x9E3779B97F4A7C15, 0xBB67AE8584CAA73B)
ZIG_R = 3.6541528853610088
ZIG_INV_R = 0.27366123732975828
TEACHER_KEY_OFFSET = 1 << 62   # synthgen.py:41


def philox4x64(ctr, key):
    """Philox4x64-10 block (Random123), python ints."""
    c0, c1, c2, c3 = ctr
    k0, k1 = key
    for _ in range(10):
        p0 = PHILOX_M[0] * c0
        p1 = PHILOX_M[1] * c2
        c0, c1, c2, c3 = ((p1 >> 64) ^ c1 ^ k0), p1 & MASK64, ((p0 >> 64) ^ c3 ^ k1), p0 & MASK64
        k0 = (k0 + PHILOX_W[0]) & MASK64
        k1 = (k1 + PHILOX_W[1]) & MASK64
    return c0, c1, c2, c3


class PhiloxStream:
    """numpy.random.Philox(key=key) raw 64-bit stream (counter from 0)."""

    def __init__(self, key: int):
        self.key = (key & MASK64, (key >> 64) & MASK64)
        self.ctr = 0
        self.buf = ()
        self.pos = 4

    def next64(self) -> int:
        if self.pos < 4:
            v = self.buf[self.pos]
            self.pos += 1
            return v
        self.ctr += 1
        c = self.ctr
        self.buf = philox4x64((c & MASK64, (c >> 64) & MASK64, 0, 0), self.key)
        self.pos = 1
        return self.buf[0]

    def next_double(self) -> float:
        return (self.next64() >> 11) * (1.0 / 9007199254740992.0)


def stream_key(seed: int, index: int) -> int:
    """synthgen.py:44-47."""
    return ((int(seed) & MASK64) << 64) + int(index)


_TABLES = None


def extract_tables():
    """(ki uint64[256], wi f64[256], fi f64[256]) of numpy's double ziggurat.

    wi[i] is the value returned for (index i, rabs 1); ki[i] is the smallest
    52-bit rabs for which index i leaves the fast path — both read off numpy
    by loading chosen words into the Philox buffer. fi[i] = exp(-x_i^2 / 2)
    with x_i = wi[i] * 2^52 (fi[0] = 1): only compared against uniform draws
    in the wedge test, so an ulp there changes a sample with probability
    ~1e-16."""
    global _TABLES
    if _TABLES is not None:
        return _TABLES
    bg = np.random.Philox(key=1)
    g = np.random.Generator(bg)
    st0 = bg.state

    def call(words):
        bg.state = {"bit_generator": "Philox", "state": dict(st0["state"]),
                    "buffer": np.array(words, dtype=np.uint64), "buffer_pos": 0,
                    "has_uint32": 0, "uinteger": 0}
        return float(g.standard_normal())

    def word(idx, rabs):
        return (rabs << 9) | idx

    m52 = (1 << 52) - 1
    u_max, u_zero, u_tail = ((1 << 53) - 1) << 11, 0, int(0.95 * (1 << 53)) << 11
    mark = word(200, 12345)
    mark_v = call([mark, 0, 0, 0])
    wi = np.zeros(256)
    wi[0] = call([word(0, 1), u_tail, u_max, 0])
    for i in range(1, 256):
        wi[i] = call([word(i, 1), u_zero, mark, 0])   # fast path, or wedge accepted at U = 0

    def slow(i, rabs):
        if i == 0:  # tail returns R + xx > 4 for U = 0.95; the fast path stays below R
            return abs(call([word(0, rabs), u_tail, u_max, 0])) > 4.0
        return call([word(i, rabs), u_max, mark, 0]) == mark_v  # wedge rejects at U ~ 1

    ki = np.zeros(256, dtype=np.uint64)
    for i in range(256):
        if slow(i, 0):
            continue
        if not slow(i, m52):
            ki[i] = m52 + 1
            continue
        lo, hi = 0, m52
        while hi - lo > 1:
            mid = (lo + hi) // 2
            if slow(i, mid):
                hi = mid
            else:
                lo = mid
        ki[i] = hi
    x = wi * 4503599627370496.0
    fi = np.exp(-0.5 * x * x)
    fi[0] = 1.0
    _TABLES = (ki, wi, fi)
    return _TABLES


def standard_normal(stream: PhiloxStream) -> float:
    """numpy random_standard_normal (distributions.c), one draw."""
    ki, wi, fi = extract_tables()
    while True:
        r = stream.next64()
        idx = r & 0xFF
        r >>= 8
        sign = r & 1
        rabs = (r >> 1) & 0x000FFFFFFFFFFFFF
        x = rabs * float(wi[idx])
        if sign:
            x = -x
        if rabs < int(ki[idx]):
            return x
        if idx == 0:
            while True:
                xx = -ZIG_INV_R * math.log1p(-stream.next_double())
                yy = -math.log1p(-stream.next_double())
                if yy + yy > xx * xx:
                    return -(ZIG_R + xx) if ((rabs >> 8) & 1) else ZIG_R + xx
        else:
            if (float(fi[idx - 1]) - float(fi[idx])) * stream.next_double() + float(fi[idx]) < math.exp(-0.5 * x * x):
                return x


def sample_normals(seed: int, index: int, d: int, noise: bool):
    """Sample `index`'s activation (and noise) rows: synthgen.py:170-174."""
    s = PhiloxStream(stream_key(seed, index))
    x = np.array([standard_normal(s) for _ in range(d)])
    nz = np.array([standard_normal(s) for _ in range(d)]) if noise else None
    return x, nz


def pairwise_sum(a) -> float:
    """numpy pairwise_sum for float64 (loops_utils.h), + the 0 initial value."""
    def pw(lo, n):
        if n < 8:
            r = 0.0
            for i in range(n):
                r += a[lo + i]
            return r
        if n <= 128:
            r = [a[lo + j] for j in range(8)]
            i = 8
            while i < n - (n % 8):
                for j in range(8):
                    r[j] += a[lo + i + j]
                i += 8
            res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]))
            while i < n:
                res += a[lo + i]
                i += 1
            return res
        n2 = n // 2
        n2 -= n2 % 8
        return pw(lo, n2) + pw(lo + n2, n - n2)
    a = [float(v) for v in a]
    return 0.0 + pw(0, len(a))


def layer_norm(x, eps=1e-5):
    """core.py:57-68 (numpy mean / var / sqrt / divide)."""
    x = np.asarray(x, dtype=np.float64)
    mean = x.mean(axis=-1, keepdims=True)
    var = x.var(axis=-1, keepdims=True)
    return (x - mean) / np.sqrt(var + eps)


def softmax(z):
    """core.py:19-24."""
    z = np.asarray(z, dtype=np.float64)
    z = z - z.max(axis=-1, keepdims=True)
    e = np.exp(z)
    return e / e.sum(axis=-1, keepdims=True)


def top_k_batch(scores, k):
    """core.py:42-48."""
    order = np.argsort(-np.asarray(scores, dtype=np.float64), axis=1, kind="stable")
    return np.sort(order[:, :k], axis=1)


def generate_dataset(gate, k, n, seed=0, transform="identity", mix=None, w_in=None, w_out=None,
                     post_norm=True, noise_sigma=0.0, first_index=0):
    """synthgen.py:162-189 + make_dataset :148-159. Teacher matrices are passed
    in (random_mix_matrix / _nonlinear_maps draw them from one numpy stream,
    synthgen.py:79-90). Returns (x f32, scores f32, topk int64, x f64)."""
    d = gate.shape[1]
    rows = [sample_normals(seed, first_index + i, d, noise_sigma > 0) for i in range(n)]
    x = np.stack([r[0] for r in rows])
    if transform == "identity":
        post = x.copy()
    elif transform == "linear":
        post = x @ mix.T
    else:
        post = np.tanh(x @ w_in.T) @ w_out.T
    if noise_sigma > 0:
        post += noise_sigma * np.stack([r[1] for r in rows])
    if post_norm:
        post = layer_norm(post)
    scores = softmax(post @ np.asarray(gate, dtype=np.float64).T)
    s32 = scores.astype(np.float32)
    return x.astype(np.float32), s32, top_k_batch(s32, k), x
