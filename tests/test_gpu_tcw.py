"""Wide-precision tensor-core update (ds_tc.cu k_prod_tcw + k_tcw_finish):
the short products on the tensor cores with the pivot-row digits streamed per
K chunk, stored as limbs, then rounded and subtracted per element.  It is the
engine above 8192 bits; DS_TC_WIDE=1 forces it at any precision so it can be
checked against the oracle and the other engines at sizes the oracle finishes
quickly."""
import numpy as np
import pytest

import oracle
from _util import first_mismatch, results_digest
from test_gpu_tc import _device_run
from test_gpu_update_adversarial import crafted
from paper_1308_1536_b200.engine import HostResults
from paper_1308_1536_b200.synth import random_uniform_soa

pytestmark = pytest.mark.gpu
WIDE = {"DS_TC_WIDE": "1", "DS_TC_MIN_BITS": "256"}


def _oracle(A, n, p, steps, minors=True):
    ref = oracle.OracleRank(n, p, "real")
    ref.load(A)
    res = HostResults.alloc(n, 1, ref.L, minors)
    ref.run(minors, True, 0, steps, res)
    fin = A.copy()
    ref.fetch(fin)
    return res, fin


@pytest.mark.parametrize("n,p,steps", [(150, 1024, 4), (133, 257, 3), (140, 2000, 3), (131, 4095, 2),
                                          (261, 512, 3)])
def test_wide_forced_matches_oracle(n, p, steps):
    A = random_uniform_soa(n, p, seed=11 * n + p)
    res_o, fin_o = _oracle(A, n, p, steps)
    res_d, fin_d = _device_run(A, n, p, steps, True, env=WIDE)
    mism = first_mismatch(fin_o, fin_d, p)
    assert not mism, mism
    assert results_digest(res_o, fin_o, n, p, steps) == results_digest(res_d, fin_d, n, p, steps)


@pytest.mark.parametrize("p", [256, 300, 1024, 2047, 4096])
@pytest.mark.parametrize("steps", [1, 3])
def test_wide_forced_adversarial(p, steps):
    """Exact cancellation, +-1 ulp, exponent gaps, exact (integer / power-of-two)
    products -- the tie / all-ones cases of the short-product decision."""
    n = 40
    A = crafted(n, p, p + 17 * steps)
    res_o, fin_o = _oracle(A, n, p, steps)
    res_d, fin_d = _device_run(A, n, p, steps, True, env=WIDE)
    mism = first_mismatch(fin_o, fin_d, p)
    assert not mism, mism
    assert results_digest(res_o, fin_o, n, p, steps) == results_digest(res_d, fin_d, n, p, steps)


@pytest.mark.parametrize("minors", [True, False])
def test_wide_forced_matches_tc(minors):
    """Several row chunks (small product buffer), many column tiles, vs the regular TC engine."""
    n, p, steps = 600, 4096, 12
    A = random_uniform_soa(n, p, seed=5 + n)
    res_t, fin_t = _device_run(A, n, p, steps, minors)
    res_w, fin_w = _device_run(A, n, p, steps, minors, env=dict(WIDE, DS_TCW_BUDGET_MB="64"))
    assert np.array_equal(fin_t.cls, fin_w.cls)
    assert np.array_equal(fin_t.exp, fin_w.exp)
    assert np.array_equal(fin_t.limbs, fin_w.limbs)
    assert results_digest(res_t, fin_t, n, p, steps) == results_digest(res_w, fin_w, n, p, steps)


@pytest.mark.parametrize("n,p,steps", [(136, 16384, 2), (40, 16000, 2), (40, 32768, 2), (24, 33220, 3)])
def test_wide_native_matches_oracle(n, p, steps):
    """16384 bits and up: the wide engine is the default (A no longer fits in TMEM);
    33220 bits = 10,000 decimal digits, the paper's headline precision."""
    A = random_uniform_soa(n, p, seed=n + 3 * p)
    res_o, fin_o = _oracle(A, n, p, steps)
    res_d, fin_d = _device_run(A, n, p, steps, True)
    mism = first_mismatch(fin_o, fin_d, p)
    assert not mism, mism
    assert results_digest(res_o, fin_o, n, p, steps) == results_digest(res_d, fin_d, n, p, steps)


def test_wide_16k_matches_dfma():
    n, p, steps = 300, 16384, 6
    A = random_uniform_soa(n, p, seed=1234)
    res_w, fin_w = _device_run(A, n, p, steps, True)
    res_f, fin_f = _device_run(A, n, p, steps, True, env={"DS_DISABLE_TC": "1"})
    assert np.array_equal(fin_f.limbs, fin_w.limbs)
    assert np.array_equal(fin_f.exp, fin_w.exp)
    assert np.array_equal(fin_f.cls, fin_w.cls)
    assert results_digest(res_f, fin_f, n, p, steps) == results_digest(res_w, fin_w, n, p, steps)


# ---------------------------------------------------------------- complex
# Complex elements (mpc) on the wide engine: the four component products
# z_c1 * b_c2 on the tensor cores, Re / Im = the exact two-product sums rounded
# once (mpc_mul), then the per-component subtraction (mpc_sub).
from test_gpu_parity import _random_matrix, device_eliminate  # noqa: E402
from paper_1308_1536_b200 import mp  # noqa: E402
from paper_1308_1536_b200.soa import SoA  # noqa: E402


@pytest.mark.parametrize("n,p,special", [(24, 256, True), (30, 1024, False), (20, 2000, True), (14, 4096, True),
                                          (12, 300, False), (10, 8192, True), (8, 16384, False)])
def test_wide_complex_full_elimination_matches_oracle(n, p, special):
    A = _random_matrix(n, p, 77 * n + p, "complex", special)
    rc_o, done_o, res_o, fin_o = oracle.eliminate_soa(A, n, p, "complex")
    rc_d, done_d, res_d, fin_d = device_eliminate(A, n, p, "complex")
    assert done_o == done_d
    assert not first_mismatch(fin_o, fin_d, p)
    assert results_digest(res_o, fin_o, n, p, done_o) == results_digest(res_d, fin_d, n, p, done_d)


def test_wide_complex_real_valued_and_imaginary():
    """Zero imaginary (or real) parts: zero component products, exact zero sums and signed zeros."""
    n, p = 16, 512
    rs = mp.random_state(5)
    with mp.context(precision=p):
        vals = []
        for i in range(n * n):
            x = 2 * mp.mpfr_random(rs) - 1
            m = i % 3
            vals.append(mp.mpc(x, 0) if m == 0 else (mp.mpc(0, x) if m == 1 else mp.mpc(x, -x)))
    A = SoA.from_scalars(vals, p, "complex")
    from paper_1308_1536_b200.engine import DeviceElimination
    rc_o, done_o, res_o, fin_o = oracle.eliminate_soa(A, n, p, "complex")
    rc_d, done_d, res_d, fin_d = device_eliminate(A, n, p, "complex")
    assert done_o == done_d
    assert not first_mismatch(fin_o, fin_d, p)
    assert results_digest(res_o, fin_o, n, p, done_o) == results_digest(res_d, fin_d, n, p, done_d)


@pytest.mark.parametrize("budget_mb", [None, "16"])
def test_wide_complex_matches_general_engine(budget_mb):
    """Many column tiles and rows (and, with a small product buffer, several row
    chunks): bit-identical to the exact thread-level engine."""
    import os
    from paper_1308_1536_b200.engine import DeviceElimination
    n, p, steps = 260, 1024, 5
    A = random_uniform_soa(n, p, seed=31, kind="complex")

    def run(env):
        old = os.environ.get("DS_DISABLE_TC")
        oldb = os.environ.get("DS_TCW_BUDGET_MB")
        if env:
            os.environ["DS_DISABLE_TC"] = "1"
        elif budget_mb:
            os.environ["DS_TCW_BUDGET_MB"] = budget_mb
        try:
            with DeviceElimination(n, p, "complex") as eng:
                eng.load(A)
                res = HostResults.alloc(n, 2, eng.L, True)
                eng.run(True, True, 0, steps, res)
                fin = A.copy()
                eng.fetch(fin)
                return res, fin, eng.counters()
        finally:
            if old is None:
                os.environ.pop("DS_DISABLE_TC", None)
            else:
                os.environ["DS_DISABLE_TC"] = old
            if oldb is None:
                os.environ.pop("DS_TCW_BUDGET_MB", None)
            else:
                os.environ["DS_TCW_BUDGET_MB"] = oldb
    res_t, fin_t, cnt = run(False)
    assert cnt["tc_engine"]
    res_g, fin_g, _ = run(True)
    assert np.array_equal(fin_t.cls, fin_g.cls)
    assert np.array_equal(fin_t.exp, fin_g.exp)
    assert np.array_equal(fin_t.limbs, fin_g.limbs)
    assert results_digest(res_t, fin_t, n, p, steps) == results_digest(res_g, fin_g, n, p, steps)


@pytest.mark.parametrize("n,p,bad", [(12, 256, 2), (20, 1024, 5), (10, 4096, 3)])
def test_complex_zero_pivot_after_first_step(n, p, bad):
    """A complex matrix whose leading (bad+1)-minor is exactly singular (row `bad` duplicates row 0,
    so it is eliminated to exact zeros by step 0): the device stops at step `bad` with every earlier minors row
    emitted -- the side-stream emission of size bad+1 must not be cancelled by the later zero
    pivot (the reference emits it before raising, elim.py:209-226)."""
    import random
    from paper_1308_1536_b200 import mp
    from paper_1308_1536_b200.soa import SoA
    rnd = random.Random(n * p + bad)
    with mp.context(precision=p):
        rows = [[mp.mpc(rnd.randint(-9, 9), rnd.randint(-9, 9)) for _ in range(n)] for _ in range(n)]
        rows[bad] = list(rows[0])
        vals = [x for r in rows for x in r]
    A = SoA.from_scalars(vals, p, "complex")
    from paper_1308_1536_b200.engine import DeviceElimination
    rc_o, done_o, res_o, fin_o = oracle.eliminate_soa(A, n, p, "complex")
    assert done_o == bad
    with DeviceElimination(n, p, "complex") as eng:
        eng.load(A)
        res_d = HostResults.alloc(n, 2, eng.L, True)
        rc, done_d = eng.run(True, True, 0, n, res_d)
        fin_d = A.copy()
        eng.fetch(fin_d)
    assert done_d == bad
    assert results_digest(res_o, fin_o, n, p, done_o) == results_digest(res_d, fin_d, n, p, done_d)
    assert res_d.row_flags[bad] & 1  # size bad+1 emitted


@pytest.mark.parametrize("p", [1024, 4096])
def test_complex_warp_and_thread_engines_agree(p):
    """The warp-cooperative complex kernels (ds_cwarp.cuh) and the thread-level ones (DS_CX_THREAD=1)
    give the same bits on an exponent-spread complex matrix (wide exact sums, perturbations)."""
    import os
    n = 40
    A = _random_matrix(n, p, 5 * n + p, "complex", True)
    rc_w, done_w, res_w, fin_w = device_eliminate(A, n, p, "complex")
    os.environ["DS_CX_THREAD"] = "1"
    try:
        rc_t, done_t, res_t, fin_t = device_eliminate(A, n, p, "complex")
    finally:
        os.environ.pop("DS_CX_THREAD", None)
    assert done_w == done_t
    assert results_digest(res_w, fin_w, n, p, done_w) == results_digest(res_t, fin_t, n, p, done_t)
