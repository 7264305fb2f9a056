"""Edge shapes on the device through the drop-in API, against the CPU oracle:
1x1 and 2x2 matrices, more ranks than rows (ranks owning no row), panels
larger than the matrix, zero matrices (exact zero pivot at step 0), and
precisions at the engine boundaries."""
import pytest

import oracle
from _util import results_digest
from paper_1308_1536_b200 import MatrixBuffer, Precision, ZeroPivot, eliminate, mp, par_eliminate
from paper_1308_1536_b200.engine import HostResults
from paper_1308_1536_b200.paged import paged_eliminate
from paper_1308_1536_b200.scalars import canonical_bits
from paper_1308_1536_b200.soa import SoA

pytestmark = pytest.mark.gpu


def _matrix(n, p, kind, seed, zero=False):
    rs = mp.random_state(seed)
    with mp.context(precision=p):
        vals = []
        for _ in range(n * n):
            x = mp.mpfr(0) if zero else 2 * mp.mpfr_random(rs) - 1
            vals.append(x if kind == "real" else mp.mpc(x, x / 3))
    return SoA.from_scalars(vals, p, kind)


def _oracle_digest(A, n, p, kind):
    rc, done, res, fin = oracle.eliminate_soa(A, n, p, kind)
    return done, results_digest(res, fin, n, p, done)


def _digest_objs(trace, minors, Abuf, n, p, kind):
    """results_digest of the drop-in's objects, via SoA (same canonical forms)."""
    res = HostResults.alloc(n, 2 if kind == "complex" else 1, (p + 31) // 32, minors is not None)
    for i, (pv, dv) in enumerate(zip(trace.pivots, trace.det_series)):
        res.pivots.set(i, pv, p)
        res.dets.set(i, dv, p)
    if minors is not None:
        for m in minors.sizes():
            r = minors.rows[m]
            res.row_flags[m - 1] = 1 | (2 if r.normalized is not None else 0)
            for k in range(m):
                res.signed.set((m - 1) * n + k, r.signed[k], p)
                if r.normalized is not None:
                    res.normalized.set((m - 1) * n + k, r.normalized[k], p)
    fin = Abuf.to_soa()
    return results_digest(res, fin, n, p, len(trace.pivots))


def _run(fn):
    try:
        trace, minors = fn()[:2]
    except ZeroPivot as exc:
        trace, minors = exc.trace, exc.series
    return trace, minors


@pytest.mark.parametrize("n,p,kind", [(1, 64, "real"), (2, 256, "real"), (1, 256, "complex"), (2, 1024, "complex"),
                                      (3, 767, "real"), (3, 768, "real"), (5, 8193, "real")])
@pytest.mark.parametrize("how", ["eliminate", "local3", "paged"])
def test_small_shapes(n, p, kind, how):
    A = _matrix(n, p, kind, 7 * n + p)
    done, want = _oracle_digest(A, n, p, kind)
    buf = MatrixBuffer.from_soa(n, kind, Precision(p), A)
    if how == "eliminate":
        trace, minors = _run(lambda: eliminate(buf))
    elif how == "local3":  # three ranks, some owning no row
        trace, minors = _run(lambda: par_eliminate(buf, 3, transport="local"))
    else:
        trace, minors = _run(lambda: paged_eliminate(buf, 4))
    assert len(trace.pivots) == done
    assert _digest_objs(trace, minors, buf, n, p, kind) == want


@pytest.mark.parametrize("kind", ["real", "complex"])
def test_zero_matrix_raises_at_step_one(kind):
    n, p = 4, 256
    A = _matrix(n, p, kind, 1, zero=True)
    buf = MatrixBuffer.from_soa(n, kind, Precision(p), A)
    with pytest.raises(ZeroPivot) as ei:
        eliminate(buf)
    assert ei.value.step == 1 and ei.value.trace.step == 0 and not ei.value.trace.pivots
    assert all(canonical_bits(x) == canonical_bits(y) for rx, ry in zip(buf.rows, MatrixBuffer.from_soa(
        n, kind, Precision(p), A).rows) for x, y in zip(rx, ry))
