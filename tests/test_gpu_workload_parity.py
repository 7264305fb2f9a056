"""Bit parity of the BENCHMARKED workloads (BASELINE.json configs 2, 3 and 5)
against the oracle, at their full sizes.

The oracle cannot eliminate N=2000 @4096 in test time, so each full-size
device run is checked three ways (tests/parity_check.py):
  * the complete matrix state after its first 8 pivot steps (every element)
    vs OracleRank(n, p).run(0, 8);
  * the prefix property -- det_series / pivots / every minors row of size <= m
    and the final leading m x m block vs an oracle run on A[1..m,1..m];
  * Laplace residuals (elim.py:232-248) of the largest sizes on the original
    entries.
Both the leading-steps state and the full results come from ONE device
context: steps [0, 8) are run, the matrix is fetched, and the same context
continues with steps [8, n) (the resume path of ds_run).
"""
import os

import numpy as np
import pytest

import parity_check as pc
from paper_1308_1536_b200.engine import DeviceElimination, HostResults
from paper_1308_1536_b200.synth import random_uniform_soa

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run_split(A, n, p, kind="real", head=8, head_minors=True):
    """Device run of steps [0, head), fetch, then [head, n) in the same context."""
    with DeviceElimination(n, p, kind) as eng:
        eng.load(A)
        res_h = HostResults.alloc(n, eng.ncomp, eng.L, head_minors)
        rc, done = eng.run(True, True, 0, head, res_h)
        assert done == head
        fin_h = A.copy()
        eng.fetch(fin_h)
        res = HostResults.alloc(n, eng.ncomp, eng.L, True)
        rc, done = eng.run(True, True, head, n, res)
        assert done == n
        eng.results(n, res)  # the whole trace and every minors row
        fin = A.copy()
        eng.fetch(fin)
        counters = eng.counters()
    return res_h, fin_h, res, fin, counters


def _check(A, n, p, m, laplace_sizes, laplace_max_log2, kind="real", head=8, head_minors=True):
    res_h, fin_h, res, fin, counters = _run_split(A, n, p, kind, head, head_minors)
    lead = pc.leading_steps(A, n, p, kind, head, fin_h, res_h)
    assert lead["ok"], lead
    pre = pc.prefix(A, n, p, kind, m, res, fin)
    assert pre["ok"], pre
    assert all(res.row_flags[1:] & 1), "every minors row 2..n emitted"
    if laplace_sizes:
        lap = pc.laplace(A, n, p, res, laplace_sizes)
        assert lap["worst_log2"] < laplace_max_log2, lap
    return counters


def test_config3_random_n2000_p4096():
    """Config 3' (N=2000 @4096, random real): the shape the bench times."""
    n, p = 2000, 4096
    A = random_uniform_soa(n, p, seed=2000)
    _check(A, n, p, m=384, laplace_sizes=[n, n - 1, 1000], laplace_max_log2=-p / 2)


def test_config2_random_n1000_p1024():
    """Config 2 (N=1000 @1024, random real)."""
    n, p = 1000, 1024
    A = random_uniform_soa(n, p, seed=70)
    _check(A, n, p, m=500, laplace_sizes=[n, 999, 500], laplace_max_log2=-p / 2)


def test_config3_beta_n2000_p4096():
    """The bench workload itself: the Artless beta matrix N=2000 @4096 (genmat.beta_matrix, bit-identical
    host builder, cached column Gammas)."""
    from paper_1308_1536_b200 import hostgen
    from paper_1308_1536_b200.soa import SoA
    n, p = 2000, 4096
    z = np.load(os.path.join(ROOT, "data", f"beta_gammas_p{p}_N{n}.npz"))
    gammas = SoA(2, int(z["L"]), int(z["count"]), np.ascontiguousarray(z["limbs"]), np.ascontiguousarray(z["exp"]),
                 np.ascontiguousarray(z["cls"]))
    bb = hostgen.BetaBuilder(os.path.join(ROOT, "data", "zeta_zeros_4096.txt"), n, p, gammas=gammas)
    bb.fill(n)
    A = bb.out
    # beta matrices are ill-conditioned by design (the paper's reason for 10,000 digits): the
    # Laplace residual of the largest sizes is recorded, not bounded, here -- parity is the gate
    _check(A, n, p, m=384, laplace_sizes=[], laplace_max_log2=0)


def test_config5_precision_prefix_n2000_p33220():
    """Config 5's precision (33,220 bits = 10,000 digits) at N=2000: wide tensor-core engine."""
    n, p = 2000, 33220
    A = random_uniform_soa(n, p, seed=33220)
    counters = _check(A, n, p, m=96, laplace_sizes=[n], laplace_max_log2=-p / 2, head=1,
                      head_minors=False)
    assert counters["tc_engine"]
