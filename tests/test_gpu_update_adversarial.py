"""Adversarial single-step checks of the fused real update (ds_update.cu)
against the oracle: with a_00 = 1 the first step uses z_j = a_j0 exactly, so
a_jk can be crafted relative to RN(z_j * b_k) -- exact cancellation, +-1 ulp
residues, exponent gaps around p+2, exact (integer / power-of-two) products
that force the full-product fallback, all-ones mantissas, signed zeros."""
import os

import pytest

import oracle
from _util import first_mismatch, results_digest
from paper_1308_1536_b200 import mp
from paper_1308_1536_b200.engine import DeviceElimination, HostResults
from paper_1308_1536_b200.soa import SoA

pytestmark = pytest.mark.gpu


def crafted(n, p, seed):
    rs = mp.random_state(seed)
    with mp.context(precision=p):
        def rnd():
            return 2 * mp.mpfr_random(rs) - 1
        one = mp.mpfr(1)
        ulp = lambda x: mp.mul_2exp(mp.mpfr(1), int(x.as_mantissa_exp()[1]) + p - p) if x != 0 else mp.mpfr(0)  # noqa
        b = [one] + [rnd() for _ in range(n - 1)]
        z = [one] + [rnd() for _ in range(n - 1)]
        for k in range(1, n):
            m = k % 9
            if m == 1:
                b[k] = mp.mpfr(k)  # small integer
            elif m == 2:
                b[k] = mp.mul_2exp(one, k - n)  # power of two
            elif m == 3:
                b[k] = mp.mul_2exp(one, 1) - mp.mul_2exp(one, 1 - p)  # all-ones mantissa
            elif m == 4:
                b[k] = mp.mpfr(0) if k % 2 else -mp.mpfr(0)
        for j in range(1, n):
            m = j % 7
            if m == 1:
                z[j] = mp.mpfr(j * 3 - 7)
            elif m == 2:
                z[j] = mp.mul_2exp(one, -j)
            elif m == 3:
                z[j] = mp.mul_2exp(one, 1) - mp.mul_2exp(one, 1 - p)
            elif m == 4:
                z[j] = -mp.mpfr(0) if j % 2 else mp.mpfr(0)
        rows = [b]
        for j in range(1, n):
            row = [z[j]]
            for k in range(1, n):
                t = z[j] * b[k]
                mode = (3 * j + 5 * k) % 13
                if mode == 0:
                    a = t  # exact cancellation
                elif mode == 1 and t != 0:
                    m_, e_ = t.as_mantissa_exp()
                    a = t + mp.mul_2exp(one, int(e_))  # one ulp above
                elif mode == 2 and t != 0:
                    m_, e_ = t.as_mantissa_exp()
                    a = t - mp.mul_2exp(one, int(e_) + (j % 3))
                elif mode == 3 and t != 0:
                    a = mp.mul_2exp(rnd(), int(t.as_mantissa_exp()[1]) + p + (k % 5) - 3)  # gap ~ p+2
                elif mode == 4 and t != 0:
                    a = mp.mul_2exp(rnd(), int(t.as_mantissa_exp()[1]) + 2 * p - (k % 5) + 1)
                elif mode == 5:
                    a = mp.mpfr(0) if k % 2 else -mp.mpfr(0)
                elif mode == 6:
                    a = -t * 3  # addition path with carry
                elif mode == 7:
                    a = t / 2 + mp.mul_2exp(rnd(), -3 * p)
                elif mode == 8:
                    a = mp.mpfr(int(rnd() * 64))
                else:
                    a = rnd()
                row.append(a)
            rows.append(row)
    vals = [x for r in rows for x in r]
    return SoA.from_scalars(vals, p, "real")


@pytest.mark.parametrize("p", [64, 65, 96, 120, 121, 127, 128, 130, 200, 256, 300, 511, 1024, 2047, 4096, 5000])
@pytest.mark.parametrize("steps", [1, 3])
def test_fused_update_adversarial(p, steps):
    n = 40
    A = crafted(n, p, p + 17 * steps)
    ref = oracle.OracleRank(n, p, "real")
    ref.load(A)
    res_o = HostResults.alloc(n, 1, ref.L, True)
    ref.run(True, True, 0, steps, res_o)
    fin_o = A.copy()
    ref.fetch(fin_o)
    # below the engine crossover (768 bits) run the tensor-core engine too (DS_TC_MIN_BITS)
    for env in ([None, "256"] if 256 <= p < 768 else [None]):
        old = os.environ.get("DS_TC_MIN_BITS")
        if env:
            os.environ["DS_TC_MIN_BITS"] = env
        try:
            with DeviceElimination(n, p, "real") as eng:
                eng.load(A)
                res_d = HostResults.alloc(n, 1, eng.L, True)
                eng.run(True, True, 0, steps, res_d)
                fin_d = A.copy()
                eng.fetch(fin_d)
                if env:
                    assert eng.counters()["tc_engine"]
        finally:
            if env:
                if old is None:
                    os.environ.pop("DS_TC_MIN_BITS", None)
                else:
                    os.environ["DS_TC_MIN_BITS"] = old
        mism = first_mismatch(fin_o, fin_d, p)
        assert not mism, mism
        assert results_digest(res_o, fin_o, n, p, steps) == results_digest(res_d, fin_d, n, p, steps)
