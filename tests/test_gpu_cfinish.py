"""Warp-cooperative complex finish (csrc/ds_cfinish.cuh, k_cfw_finish) against the
thread-per-element finish it replaces (k_tcw_finish_c, DS_CX_FINISH_THREAD=1) and
against the oracle: bit-identical states, traces and minors on complex matrices
whose shapes exercise every branch -- cancelling component products, zero real or
imaginary parts, exponent gaps wide enough to take the lane-0 path (perturbation
terms, alignments past the registers), and the precisions of each K instance
(words per lane 2, 3, 5, 9)."""
import os

import pytest

import oracle
from _util import first_mismatch, results_digest
from test_gpu_parity import device_eliminate
from paper_1308_1536_b200 import mp
from paper_1308_1536_b200.soa import SoA
from paper_1308_1536_b200.synth import random_uniform_soa

pytestmark = pytest.mark.gpu


def _matrix(n, p, seed, spread_bits, zeros):
    rs = mp.random_state(seed)
    with mp.context(precision=p):
        vals = []
        for i in range(n * n):
            x = 2 * mp.mpfr_random(rs) - 1
            y = 2 * mp.mpfr_random(rs) - 1
            if spread_bits and i % 5 == 2:
                x = mp.mul_2exp(x, (i % 3 - 1) * spread_bits)
            if spread_bits and i % 7 == 4:
                y = mp.mul_2exp(y, -(i % 4) * spread_bits // 2)
            if zeros and i % 9 == 1:
                y = mp.mpfr(0)
            if zeros and i % 13 == 6:
                x = mp.mpfr(0)
            if i % 17 == 8:
                y = x  # |re| == |im|: cancelling products
            vals.append(mp.mpc(x, y))
    return SoA.from_scalars(vals, p, "complex")


@pytest.fixture(autouse=True)
def _force_warp(monkeypatch):
    # the warp finish also where the thread kernel is the faster default (K = 2, p <~ 1400)
    monkeypatch.setenv("DS_CX_FINISH_WARP", "1")


def _thread_finish(A, n, p):
    os.environ["DS_CX_FINISH_THREAD"] = "1"
    try:
        return device_eliminate(A, n, p, "complex")
    finally:
        os.environ.pop("DS_CX_FINISH_THREAD", None)


@pytest.mark.parametrize("n,p,spread,zeros", [
    (48, 256, 0, True), (40, 256, 700, False), (36, 1024, 90, True), (30, 1024, 2400, True),
    (32, 2000, 300, False), (24, 4096, 0, True), (24, 4096, 900, True), (20, 4096, 9000, False),
    (12, 8192, 200, True),
])
def test_warp_finish_matches_thread_finish(n, p, spread, zeros):
    A = _matrix(n, p, 1000 * n + p + spread, spread, zeros)
    rc_w, done_w, res_w, fin_w = device_eliminate(A, n, p, "complex")
    rc_t, done_t, res_t, fin_t = _thread_finish(A, n, p)
    assert done_w == done_t
    assert not first_mismatch(fin_t, fin_w, p)
    assert results_digest(res_w, fin_w, n, p, done_w) == results_digest(res_t, fin_t, n, p, done_t)


@pytest.mark.parametrize("n,p,spread", [(20, 1024, 2400), (14, 4096, 900), (10, 2000, 0)])
def test_warp_finish_matches_oracle(n, p, spread):
    A = _matrix(n, p, 7 * n + p, spread, True)
    rc_o, done_o, res_o, fin_o = oracle.eliminate_soa(A, n, p, "complex")
    rc_d, done_d, res_d, fin_d = device_eliminate(A, n, p, "complex")
    assert done_o == done_d
    assert not first_mismatch(fin_o, fin_d, p)
    assert results_digest(res_o, fin_o, n, p, done_o) == results_digest(res_d, fin_d, n, p, done_d)


def test_warp_finish_many_blocks_and_row_chunks():
    """Several product row chunks (small product budget) and element groups that
    straddle rows (ncols not a multiple of 8): same bits as the thread finish."""
    n, p = 203, 1024
    A = random_uniform_soa(n, p, seed=17, kind="complex")
    os.environ["DS_TCW_BUDGET_MB"] = "8"
    try:
        r_w = device_eliminate(A, n, p, "complex")
        r_t = _thread_finish(A, n, p)
    finally:
        os.environ.pop("DS_TCW_BUDGET_MB", None)
    assert r_w[1] == r_t[1] == n
    assert not first_mismatch(r_t[3], r_w[3], p)
    assert results_digest(r_w[2], r_w[3], n, p, n) == results_digest(r_t[2], r_t[3], n, p, n)


@pytest.mark.parametrize("n,p", [(30, 1024), (16, 4096), (12, 333)])
def test_warp_finish_exact_products(n, p):
    """Rows of small Gaussian integers (like the power matrix's first row of ones):
    their short products omit nothing, and the warp finish rounds those sums directly
    (k_lowdig) instead of sending them to the exact engine -- same bits as the thread
    finish and the oracle."""
    rs = mp.random_state(n + p)
    with mp.context(precision=p):
        vals = []
        for i in range(n * n):
            r, c = divmod(i, n)
            if r % 3 == 0 or c % 4 == 1:
                vals.append(mp.mpc(mp.mpfr(int(7 * mp.mpfr_random(rs)) - 3), mp.mpfr(int(5 * mp.mpfr_random(rs)) - 2)))
            else:
                vals.append(mp.mpc(2 * mp.mpfr_random(rs) - 1, 2 * mp.mpfr_random(rs) - 1))
        vals[0] = mp.mpc(1, 0)
    A = SoA.from_scalars(vals, p, "complex")
    rc_o, done_o, res_o, fin_o = oracle.eliminate_soa(A, n, p, "complex")
    rc_w, done_w, res_w, fin_w = device_eliminate(A, n, p, "complex")
    rc_t, done_t, res_t, fin_t = _thread_finish(A, n, p)
    assert done_o == done_w == done_t
    want = results_digest(res_o, fin_o, n, p, done_o)
    assert not first_mismatch(fin_o, fin_w, p)
    assert results_digest(res_w, fin_w, n, p, done_w) == want
    assert results_digest(res_t, fin_t, n, p, done_t) == want
