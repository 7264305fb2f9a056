"""Tensor-core update (ds_tc.cu, tcgen05 kind::i8) against the oracle and
against the DFMA update engine (ds_update.cu, selected with DS_DISABLE_TC):
several 128-row tiles, many columns per CTA (TMEM double-buffer reuse), the
column range with and without collected minors, ragged tails."""
import os

import numpy as np
import pytest

import oracle
from _util import first_mismatch, results_digest
from paper_1308_1536_b200.engine import DeviceElimination, HostResults
from paper_1308_1536_b200.synth import random_uniform_soa

pytestmark = pytest.mark.gpu


def _device_run(A, n, p, steps, minors, env=None):
    old = {}
    for k, v in (env or {}).items():
        old[k] = os.environ.get(k)
        os.environ[k] = v
    try:
        with DeviceElimination(n, p, "real") as eng:
            eng.load(A)
            res = HostResults.alloc(n, 1, eng.L, minors)
            eng.run(minors, True, 0, steps, res)
            fin = A.copy()
            eng.fetch(fin)
            return res, fin
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


@pytest.mark.parametrize("n,p,steps", [(150, 4096, 3), (152, 4096, 3), (261, 1024, 5), (300, 2048, 4),
                                          (140, 2000, 4), (130, 333, 6)])
def test_tc_matches_oracle(n, p, steps):
    A = random_uniform_soa(n, p, seed=n + p)
    ref = oracle.OracleRank(n, p, "real")
    ref.load(A)
    res_o = HostResults.alloc(n, 1, ref.L, True)
    ref.run(True, True, 0, steps, res_o)
    fin_o = A.copy()
    ref.fetch(fin_o)
    res_d, fin_d = _device_run(A, n, p, steps, True)
    mism = first_mismatch(fin_o, fin_d, p)
    assert not mism, mism
    assert results_digest(res_o, fin_o, n, p, steps) == results_digest(res_d, fin_d, n, p, steps)


@pytest.mark.parametrize("minors", [True, False])
@pytest.mark.parametrize("n,p,steps", [(600, 4096, 40), (1000, 1024, 200)])
def test_tc_matches_dfma_engine(n, p, steps, minors):
    A = random_uniform_soa(n, p, seed=7 * n + p)
    res_t, fin_t = _device_run(A, n, p, steps, minors)
    res_f, fin_f = _device_run(A, n, p, steps, minors, env={"DS_DISABLE_TC": "1"})
    assert np.array_equal(fin_t.cls, fin_f.cls)
    assert np.array_equal(fin_t.exp, fin_f.exp)
    assert np.array_equal(fin_t.limbs, fin_f.limbs)
    assert results_digest(res_f, fin_f, n, p, steps) == results_digest(res_t, fin_t, n, p, steps)


@pytest.mark.parametrize("n,p,steps", [(140, 256, 5), (133, 257, 4), (136, 4064, 3), (131, 4095, 3)])
def test_tc_precision_edges(n, p, steps):
    """Smallest TC precision, non-multiple-of-32 precisions (low mask zb > 0), largest sizes."""
    A = random_uniform_soa(n, p, seed=3 * n + p)
    ref = oracle.OracleRank(n, p, "real")
    ref.load(A)
    res_o = HostResults.alloc(n, 1, ref.L, True)
    ref.run(True, True, 0, steps, res_o)
    fin_o = A.copy()
    ref.fetch(fin_o)
    res_d, fin_d = _device_run(A, n, p, steps, True, env={"DS_TC_MIN_BITS": "256"})  # TC engine below its default
    assert not first_mismatch(fin_o, fin_d, p)
    assert results_digest(res_o, fin_o, n, p, steps) == results_digest(res_d, fin_d, n, p, steps)


@pytest.mark.parametrize("minors,series", [(False, True), (True, False)])
def test_tc_lookahead_modes_vs_dfma(minors, series):
    """Whole eliminations (lookahead active) in the no-minors / no-series modes against the DFMA engine."""
    n, p = 300, 1024
    A = random_uniform_soa(n, p, seed=11)
    outs = []
    for env in (None, {"DS_DISABLE_TC": "1"}):
        old = {}
        for k, v in (env or {}).items():
            old[k] = os.environ.get(k)
            os.environ[k] = v
        try:
            with DeviceElimination(n, p, "real") as eng:
                eng.load(A)
                res = HostResults.alloc(n, 1, eng.L, minors)
                eng.run(minors, series, 0, n, res)
                fin = A.copy()
                eng.fetch(fin)
                outs.append((res, fin))
        finally:
            for k, v in old.items():
                if v is None:
                    os.environ.pop(k, None)
                else:
                    os.environ[k] = v
    (rt, ft), (rf, ff) = outs
    assert np.array_equal(ft.limbs, ff.limbs) and np.array_equal(ft.exp, ff.exp) and np.array_equal(ft.cls, ff.cls)
    assert results_digest(rt, ft, n, p, n) == results_digest(rf, ff, n, p, n)


@pytest.mark.parametrize("n,p,steps", [(136, 8192, 2), (130, 6000, 2)])
def test_tc_one_group_wide_precision(n, p, steps):
    """Precisions where one epilogue group per CTA is used (two groups' windows do not fit)."""
    A = random_uniform_soa(n, p, seed=5 * n + p)
    ref = oracle.OracleRank(n, p, "real")
    ref.load(A)
    res_o = HostResults.alloc(n, 1, ref.L, True)
    ref.run(True, True, 0, steps, res_o)
    fin_o = A.copy()
    ref.fetch(fin_o)
    res_d, fin_d = _device_run(A, n, p, steps, True, env={"DS_TC_MIN_BITS": "256"})  # TC engine below its default
    assert not first_mismatch(fin_o, fin_d, p)
    assert results_digest(res_o, fin_o, n, p, steps) == results_digest(res_d, fin_d, n, p, steps)


def test_dfma_wide_precision_16k():
    """p = 16384 on the DFMA engine (16-column CTAs) against the oracle."""
    n, p, steps = 40, 16384, 2
    A = random_uniform_soa(n, p, seed=99)
    ref = oracle.OracleRank(n, p, "real")
    ref.load(A)
    res_o = HostResults.alloc(n, 1, ref.L, True)
    ref.run(True, True, 0, steps, res_o)
    fin_o = A.copy()
    ref.fetch(fin_o)
    res_d, fin_d = _device_run(A, n, p, steps, True, env={"DS_DISABLE_TC": "1"})
    assert not first_mismatch(fin_o, fin_d, p)
    assert results_digest(res_o, fin_o, n, p, steps) == results_digest(res_d, fin_d, n, p, steps)


def test_progressive_minors_d2h_matches_full_fetch():
    """ds_run with pinned result buffers streams finalised minors rows to the host during the run
    (triangle, batches of 64 steps); the outputs must equal a pageable-buffer run's full fetch."""
    n, p = 300, 1024
    A = random_uniform_soa(n, p, seed=21)
    outs = []
    for pinned in (True, False):
        with DeviceElimination(n, p, "real") as eng:
            eng.load(A)
            res = HostResults.alloc(n, 1, eng.L, True, pinned=pinned)
            eng.run(True, True, 0, n, res)
            fin = A.copy()
            eng.fetch(fin)
            outs.append((res, fin))
    (rp, fp), (rq, fq) = outs
    assert results_digest(rp, fp, n, p, n) == results_digest(rq, fq, n, p, n)


def test_device_resume_from_checkpoint(tmp_path):
    """Checkpoint mid-run (native MPMAT writer), load it, resume on the device: the
    final state and the minors equal an uninterrupted device run."""
    from paper_1308_1536_b200.checkpoint import Checkpoint
    from paper_1308_1536_b200.soa import SoA
    n, p, stop = 260, 1024, 97
    A = random_uniform_soa(n, p, seed=31)
    with DeviceElimination(n, p, "real") as eng:
        eng.load(A)
        res = HostResults.alloc(n, 1, eng.L, True)
        eng.run(True, True, 0, stop, res)
        cur = A.copy()
        eng.fetch(cur)
        Checkpoint(tmp_path).write_soa(cur, n, p, "real", stop, [res.pivots.get(i, p) for i in range(stop)])
    soa, _, _, _, trace = Checkpoint(tmp_path).load_soa()
    with DeviceElimination(n, p, "real") as eng:
        eng.load(soa)
        eng.set_det(SoA.from_scalars([trace.det_series[-1]], p, "real"))
        res_r = HostResults.alloc(n, 1, eng.L, True)
        eng.run(True, True, stop, n, res_r)
        fin_r = soa.copy()
        eng.fetch(fin_r)
    res_f, fin_f = _device_run(A, n, p, n, True)
    assert np.array_equal(fin_r.limbs, fin_f.limbs) and np.array_equal(fin_r.cls, fin_f.cls)
    assert np.array_equal(fin_r.exp, fin_f.exp)
    for m in range(stop + 2, n + 1):  # minors emitted after the resume point: m valid entries in row m-1
        sl = slice((m - 1) * n, (m - 1) * n + m)
        for a, b in ((res_r.signed, res_f.signed), (res_r.normalized, res_f.normalized)):
            assert np.array_equal(a.limbs[:, :, sl], b.limbs[:, :, sl]) and np.array_equal(a.exp[:, sl], b.exp[:, sl])
            assert np.array_equal(a.cls[:, sl], b.cls[:, sl])
    assert np.array_equal(res_r.dets.limbs[:, :, stop:], res_f.dets.limbs[:, :, stop:])


def test_lookahead_tile_fallbacks_applied_before_next_multipliers():
    """Column 1 (the lookahead tile at step 0) full of undecidable short products:
    z_j = 1 + 2^(1-p), b_1 = 1.5 makes z_j b_1 an exact tie at p bits, which the
    tensor-core kernel hands to the exact fallback.  Step 1's multipliers (run on the
    lookahead stream) read column 1, so those fallbacks must land first."""
    from paper_1308_1536_b200 import mp
    from paper_1308_1536_b200.soa import SoA
    n, p, steps = 300, 1024, 3
    rs = mp.random_state(12)
    with mp.context(precision=p):
        one = mp.mpfr(1)
        zt = one + mp.mul_2exp(one, 1 - p)
        vals = []
        for j in range(n):
            for k in range(n):
                if j == 0 and k == 0:
                    v = one
                elif j == 0 and k == 1:
                    v = mp.mpfr(1.5)
                elif k == 0 and j % 3 != 2:
                    v = zt
                else:
                    v = 2 * mp.mpfr_random(rs) - 1
                vals.append(v)
    A = SoA.from_scalars(vals, p, "real")
    ref = oracle.OracleRank(n, p, "real")
    ref.load(A)
    res_o = HostResults.alloc(n, 1, ref.L, True)
    ref.run(True, True, 0, steps, res_o)
    fin_o = A.copy()
    ref.fetch(fin_o)
    with DeviceElimination(n, p, "real") as eng:
        eng.load(A)
        res_d = HostResults.alloc(n, 1, eng.L, True)
        eng.run(True, True, 0, steps, res_d)
        fin_d = A.copy()
        eng.fetch(fin_d)
        cnt = eng.counters()
    assert cnt["tc_fallback_elements"] > 0  # the construction does reach the fallback
    mism = first_mismatch(fin_o, fin_d, p)
    assert not mism, mism
    assert results_digest(res_o, fin_o, n, p, steps) == results_digest(res_d, fin_d, n, p, steps)
