"""Scalar conformance: the device RN mul/sub/add/div (real and complex) against
libmpfr/libmpc via the oracle, on random and adversarial operands (exponent
gaps, exact cancellation, ties, signed zeros, binade crossings, odd p)."""
import pytest

import oracle
from _util import first_mismatch
from paper_1308_1536_b200 import mp
from paper_1308_1536_b200.engine import scalar_op
from paper_1308_1536_b200.soa import SoA

pytestmark = pytest.mark.gpu


def corpus(p, seed, count, kind):
    rs = mp.random_state(seed)
    A, B = [], []
    with mp.context(precision=p):
        for i in range(count):
            a = 2 * mp.mpfr_random(rs) - 1
            b = 2 * mp.mpfr_random(rs) - 1
            mode = i % 12
            if mode == 1:
                b = a  # exact cancellation
            elif mode == 2:
                b = mp.mul_2exp(b, -(p + (i % 5) - 2))  # gap around p+2
            elif mode == 3:
                b = mp.mul_2exp(b, (i % 9) * 37)  # large gaps
            elif mode == 4:
                a = mp.mpfr(0) if i % 2 else -mp.mpfr(0)
            elif mode == 5:
                b = mp.mpfr(0) if i % 3 else -mp.mpfr(0)
            elif mode == 6:
                a = mp.mpfr(1)
                b = mp.mul_2exp(mp.mpfr(1), -p)  # tie region below a power of two
            elif mode == 7:
                a = mp.mpfr(int(a * 1000))
                b = mp.mpfr(int(b * 1000) or 3)
            elif mode == 8:
                b = a + mp.mul_2exp(mp.mpfr(1), -p + 3) if a != 0 else b  # near-cancellation
            elif mode == 9:
                a = mp.mul_2exp(mp.mpfr(1), 1) - mp.mul_2exp(mp.mpfr(1), -p + 1)  # all-ones mantissa
            if kind == "complex":
                c = 2 * mp.mpfr_random(rs) - 1
                d = 2 * mp.mpfr_random(rs) - 1
                if mode == 10:
                    c = mp.mpfr(0)
                if mode == 11:
                    d = -mp.mpfr(0)
                if mode == 4:
                    c = -mp.mpfr(0)
                a, b = mp.mpc(a, c), mp.mpc(b, d)
            A.append(a)
            B.append(b)
    return SoA.from_scalars(A, p, kind), SoA.from_scalars(B, p, kind)


@pytest.mark.parametrize("kind", ["real", "complex"])
@pytest.mark.parametrize("op", ["mul", "sub", "add", "div"])
@pytest.mark.parametrize("p", [64, 65, 127, 256, 333, 1000, 4096])
def test_scalar_op_conformance(kind, op, p):
    count = 240 if kind == "real" else 120
    a, b = corpus(p, 7 * p + len(op), count, kind)
    if op == "div":  # no division by zero
        for c in range(b.ncomp):
            pass
        zero = (b.cls >= 2).all(axis=0)
        b.cls[0, zero] = 0
        b.limbs[0, -1, zero] = 0x80000000
        b.exp[0, zero] = 1
    ref = oracle.scalar_op(op, kind, p, a, b)
    got = scalar_op(op, kind, p, a, b)
    assert not first_mismatch(ref, got, p, limit=5)
