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

from .soa import CLS_NEG, CLS_POS, SoA


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
