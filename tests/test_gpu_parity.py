"""GPU parity: the sm_100a path (through the C ABI) against the golden vectors
of the unmodified reference and against the CPU oracle, bit for bit."""
import numpy as np
import pytest

import oracle
from _util import build_input, first_mismatch, golden_names, load_golden, results_digest
from paper_1308_1536_b200 import mp
from paper_1308_1536_b200.engine import DeviceElimination, HostResults
from paper_1308_1536_b200.soa import SoA

pytestmark = pytest.mark.gpu


def device_eliminate(A: SoA, n, p, kind, collect_minors=True, series=True):
    with DeviceElimination(n, p, kind) as eng:
        eng.load(A)
        res = HostResults.alloc(n, eng.ncomp, eng.L, collect_minors)
        rc, done = eng.run(collect_minors, series, 0, n, res)
        final = A.copy()
        eng.fetch(final)
        launches = eng.launches()
    assert launches > 0
    return rc, done, res, final


@pytest.mark.parametrize("name", golden_names())
def test_device_matches_reference_goldens(name):
    meta, arrays = load_golden(name)
    A = build_input(meta, arrays)
    n, p, kind = meta["n"], meta["prec"], meta["kind"]
    rc, done, res, final = device_eliminate(A, n, p, kind, meta["collect_minors"], meta["series"])
    if meta["zero_pivot_step"] is not None:
        assert done + 1 == meta["zero_pivot_step"]
    else:
        assert done == n
    assert results_digest(res, final, n, p, done) == meta["digest"]


def _random_matrix(n, p, seed, kind="real", special=False):
    rs = mp.random_state(seed)
    with mp.context(precision=p):
        vals = []
        for i in range(n * n):
            x = 2 * mp.mpfr_random(rs) - 1
            if special and i % 7 == 3:
                x = mp.mpfr(int(x * 8))  # small integers and zeros
            if special and i % 11 == 5:
                x = mp.mul_2exp(x, (i % 5 - 2) * 40)  # exponent spread
            vals.append(x if kind == "real" else mp.mpc(x, 1 - x * x))
    return SoA.from_scalars(vals, p, kind)


@pytest.mark.parametrize("n,p,kind,special", [
    (17, 64, "real", False), (17, 65, "real", True), (21, 96, "real", False), (19, 127, "real", True),
    (23, 128, "real", False), (18, 129, "real", True), (25, 255, "real", False), (24, 333, "real", True),
    (33, 1024, "real", False), (16, 2048, "real", True), (12, 4100, "real", False), (40, 512, "real", True),
    (9, 192, "complex", False), (8, 320, "complex", True), (7, 1024, "complex", False),
])
def test_device_matches_oracle_random(n, p, kind, special):
    A = _random_matrix(n, p, n * 1000 + p, kind, special)
    rc_o, done_o, res_o, fin_o = oracle.eliminate_soa(A, n, p, kind)
    rc_d, done_d, res_d, fin_d = device_eliminate(A, n, p, kind)
    assert done_o == done_d
    assert not first_mismatch(fin_o, fin_d, p)
    assert not first_mismatch(res_o.dets, res_d.dets, p)
    assert results_digest(res_o, fin_o, n, p, done_o) == results_digest(res_d, fin_d, n, p, done_d)


def test_nominors_and_series_false_large():
    n, p = 48, 768
    A = _random_matrix(n, p, 5)
    for cm, se in ((False, True), (True, False)):
        o = oracle.eliminate_soa(A, n, p, "real", cm, se)
        d = device_eliminate(A, n, p, "real", cm, se)
        assert results_digest(o[2], o[3], n, p, o[1]) == results_digest(d[2], d[3], n, p, d[1])
