"""Fast synthetic inputs directly in the ds SoA format (numpy), for benchmark
sizes where the scalar builders (genmat.synth_matrix) would need millions of
Python objects.  Same distribution as the reference's random_uniform family
(genmat.py:242-246: x = 2U - 1, U uniform with a full p-bit mantissa): sign
uniform, |x| = U with exponent e <= 0 taken with probability 2^(e-1), mantissa
bits uniform with the MSB set.  The bits differ from gmpy2's generator -- the
benchmark only needs the shape and distribution, not the reference's exact
draws (parity tests use the reference builders)."""

from __future__ import annotations

import numpy as np

from .soa import CLS_NEG, CLS_POS, CLS_PZERO, SoA


def random_uniform_soa(n: int, p: int, seed: int, kind: str = "real", pinned: bool = False) -> SoA:
    L = (p + 31) // 32
    ncomp = 2 if kind == "complex" else 1
    count = n * n
    rng = np.random.default_rng(seed)
    s = SoA(ncomp, L, count, pinned=pinned)
    zb = 32 * L - p
    for c in range(ncomp):
        limbs = s.limbs[c]
        for l in range(L):
            limbs[l] = rng.integers(0, 2 ** 32, size=count, dtype=np.uint32)
        if zb:
            limbs[zb // 32] &= np.uint32((0xFFFFFFFF << (zb % 32)) & 0xFFFFFFFF)
            for l in range(zb // 32):
                limbs[l] = 0
        limbs[L - 1] |= np.uint32(0x80000000)
        # exponent: U in [2^(e-1), 2^e) with probability 2^(e-1), e <= 0
        s.exp[c] = -rng.geometric(0.5, size=count).astype(np.int32) + 1
        s.cls[c] = np.where(rng.integers(0, 2, size=count) == 1, CLS_NEG, CLS_POS).astype(np.uint8)
    return s


# ---------------------------------------------------------------- ds-splitmix
# Host twin of the device builder (csrc/ds_gen.cu, ds_generate): the same
# counter-based draw of genmat's random_uniform family, bit for bit.
_G = np.uint64(0x9E3779B97F4A7C15)


def _mix64(x):
    x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return x ^ (x >> np.uint64(31))


def counter_uniform_soa(n: int, p: int, seed: int, rows=None, pinned: bool = False, cols=None) -> SoA:
    """x = 2U - 1 (genmat.py:242-246) for the elements of `rows` x `cols` (default: all n
    rows and columns, row-major, count len(rows)*len(cols)), drawn from the counter-based ds-splitmix generator
    that ds_generate runs on the device: element (row, col) is a pure function of
    (seed, row, col, p).  K = the left-aligned p-bit integer U 2^p with 32-bit limbs
    R_{2q} | R_{2q+1} << 32 = mix64(key + (idx * npairs + q + 1) * G), idx = row*n + col,
    key = mix64(seed ^ 0x243F6A8885A308D3); x = (K - 2^(32L-1)) 2^(1-32L) exactly."""
    L = (p + 31) // 32
    zb = 32 * L - p
    rows = np.arange(n) if rows is None else np.asarray(rows)
    cols = np.arange(n) if cols is None else np.asarray(cols)
    idx = (rows[:, None].astype(np.uint64) * np.uint64(n) + cols.astype(np.uint64)[None, :]).reshape(-1)
    cnt = idx.size
    with np.errstate(over="ignore"):
        key = _mix64(np.uint64(seed & (2 ** 64 - 1)) ^ np.uint64(0x243F6A8885A308D3))
        npairs = np.uint64((L + 1) // 2)
        R = np.empty((L, cnt), dtype=np.uint32)
        for q in range((L + 1) // 2):
            v = _mix64(key + (idx * npairs + np.uint64(q + 1)) * _G)
            R[2 * q] = (v & np.uint64(0xFFFFFFFF)).astype(np.uint32)
            if 2 * q + 1 < L:
                R[2 * q + 1] = (v >> np.uint64(32)).astype(np.uint32)
    if zb:
        R[0] &= np.uint32((0xFFFFFFFF << zb) & 0xFFFFFFFF)
    pos = (R[L - 1] >> np.uint32(31)).astype(bool)
    # M = K - 2^(32L-1) (pos) or 2^(32L-1) - K: exact multi-limb arithmetic through Python ints is
    # too slow at size; the two's complement is ~K + 1 with the +1 stopping at the first nonzero limb
    nz = R != 0
    f = np.where(nz.any(axis=0), nz.argmax(axis=0), L)
    lidx = np.arange(L)[:, None]
    neg_m = np.where(lidx < f[None, :], np.uint32(0), np.where(lidx == f[None, :], (np.uint32(0) - R), ~R))
    M = np.where(pos[None, :], R, neg_m).astype(np.uint32)
    M[L - 1] &= np.uint32(0x7FFFFFFF)
    s = SoA(1, L, cnt, pinned=pinned)
    exp = np.zeros(cnt, dtype=np.int64)
    cls = np.where(pos, CLS_POS, CLS_NEG).astype(np.uint8)
    # normalise: left shift by clz(M) (almost always < 32 bits: the top limb is nonzero)
    top = np.full(cnt, -1, dtype=np.int64)
    for l in range(L - 1, -1, -1):
        sel = (top < 0) & (M[l] != 0)
        top[sel] = l
    zero = top < 0
    mt = M[np.maximum(top, 0), np.arange(cnt)]
    _, e2 = np.frexp(mt.astype(np.float64))  # bit length of the top nonzero limb (exact)
    clz = np.where(zero, 0, 32 - e2).astype(np.int64)
    lz = 32 * (L - 1 - np.maximum(top, 0)) + clz
    lq, lr = lz // 32, lz % 32
    out = s.limbs[0]
    # common case (top limb of M nonzero, lz < 32): one funnel shift per limb plane
    lr64 = lr.astype(np.uint64)
    sh_lo = (np.uint64(32) - lr64)
    prev = np.zeros(cnt, dtype=np.uint64)
    for l in range(L):
        hi = M[l].astype(np.uint64)
        out[l] = (((hi << lr64) | (prev >> sh_lo)) & np.uint64(0xFFFFFFFF)).astype(np.uint32)
        prev = hi
    # rare: M's top limb is zero (lz >= 32): shift exactly with Python integers
    for e in np.nonzero((lq > 0) & ~zero)[0]:
        Mi = int.from_bytes(np.ascontiguousarray(M[:, e]).tobytes(), "little") << int(lz[e])
        out[:, e] = np.frombuffer(Mi.to_bytes(4 * L, "little"), dtype=np.uint32)
    exp[:] = 1 - lz
    # K = 0 (not pos, no nonzero limb): x = -1;  M = 0 (pos, K = 2^(32L-1)): x = +0
    m1 = (~pos) & (f == L)
    out[:, m1] = 0
    out[L - 1, m1] = np.uint32(0x80000000)
    exp[m1] = 1
    z = zero & ~m1
    out[:, z] = 0
    exp[z] = 0
    cls[z] = CLS_PZERO
    s.exp[0] = exp.astype(np.int32)
    s.cls[0] = cls
    return s
