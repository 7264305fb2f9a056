"""pivot_mode="partial" (elim.py:184-208): det-only row swaps on the device.

Golden vectors come from the unmodified reference
(tests/golden/partial/make_partial_goldens.py); the GPU tests run the drop-in
elim.eliminate and compare pivots, signed det series and the final buffer bit
for bit.  The CPU tests pin the goldens' inputs and the argument checks."""
import glob
import json
import os

import numpy as np
import pytest

from _util import GOLDEN, generate
from golden.digest import digest_parts
from paper_1308_1536_b200 import mp
from paper_1308_1536_b200.elim import eliminate
from paper_1308_1536_b200.errors import ZeroPivot
from paper_1308_1536_b200.matrix import MatrixBuffer
from paper_1308_1536_b200.scalars import Precision, canonical_bits
from paper_1308_1536_b200.soa import SoA

PARTIAL = os.path.join(GOLDEN, "partial")


def partial_names():
    return sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(PARTIAL, "*.npz")))


def load_partial(name):
    z = np.load(os.path.join(PARTIAL, f"{name}.npz"))
    meta = json.loads(str(z["meta"]))
    if "in_limbs" in z.files:
        s = SoA(z["in_limbs"].shape[0], z["in_limbs"].shape[1], z["in_limbs"].shape[2],
                np.ascontiguousarray(z["in_limbs"]), np.ascontiguousarray(z["in_exp"]),
                np.ascontiguousarray(z["in_cls"]))
        A = MatrixBuffer.from_soa(meta["n"], meta["kind"], Precision(meta["prec"]), s)
    else:
        A = generate(meta["gen"])
    return meta, A


def trace_digest(trace, A):
    return digest_parts([canonical_bits(x) for x in trace.pivots], [canonical_bits(x) for x in trace.det_series],
                        [], [canonical_bits(x) for row in A.rows for x in row])


def test_partial_goldens_present():
    assert len(partial_names()) >= 10


@pytest.mark.parametrize("name", partial_names())
def test_partial_golden_inputs(name):
    meta, A = load_partial(name)
    assert A.fingerprint() == meta["fingerprint"]


def test_partial_argument_checks():
    A = MatrixBuffer.from_rows([[1, 2], [3, 4]], Precision(256))
    with pytest.raises(ValueError):
        eliminate(A, collect_minors=True, pivot_mode="partial")
    with pytest.raises(ValueError):
        eliminate(A, collect_minors=False, pivot_mode="partial", start_step=1)
    with pytest.raises(ValueError):
        eliminate(A, collect_minors=False, pivot_mode="full")
    with Precision(256).context():
        C = MatrixBuffer(2, "complex", Precision(256), [[mp.mpc(1, 1), mp.mpc(2, 0)], [mp.mpc(0, 1), mp.mpc(1, 0)]])
    with pytest.raises(NotImplementedError):
        eliminate(C, collect_minors=False, pivot_mode="partial")


@pytest.mark.gpu
@pytest.mark.parametrize("name", partial_names())
def test_partial_device_matches_reference(name):
    meta, A = load_partial(name)
    zp = None
    try:
        trace, minors = eliminate(A, collect_minors=False, pivot_mode="partial")
        assert minors is None
    except ZeroPivot as exc:
        zp = exc.step
        trace = exc.trace
    assert zp == meta["zero_pivot_step"]
    assert trace.step == meta["steps"]
    assert trace_digest(trace, A) == meta["digest"]


@pytest.mark.gpu
def test_partial_step_hook_signs_match_full_run():
    """step_hook path (one ds_run per step) gives the same signed det series."""
    meta, A = load_partial("pp_int7_s1")
    seen = []
    trace, _ = eliminate(A, collect_minors=False, pivot_mode="partial",
                         step_hook=lambda k, buf, tr: seen.append(canonical_bits(tr.det_series[-1])) and False)
    assert trace_digest(trace, A) == meta["digest"]
    assert seen == [canonical_bits(x) for x in trace.det_series]


@pytest.mark.gpu
def test_partial_wide_column_scan():
    """n > 1024 (several rows per scanning thread): a column-diagonally-dominant
    matrix needs no swaps; with rows 0 and n-1 exchanged, step 0 swaps them back
    (the maximum sits in the last row, scanned by a thread's second stride), so
    pivots and the final buffer equal the unpivoted run on the dominant matrix
    and every det carries the flipped sign (elim.py:204-216)."""
    n, p = 1100, 256
    rs = mp.random_state(5)
    with mp.context(precision=p):
        rows = [[(2 * mp.mpfr_random(rs) - 1) for _ in range(n)] for _ in range(n)]
        for i in range(n):
            rows[i][i] = mp.mpfr(2 * n) + rows[i][i]
    D = MatrixBuffer(n, "real", Precision(p), [list(r) for r in rows])
    B = MatrixBuffer(n, "real", Precision(p), [list(r) for r in rows])
    B.rows[0], B.rows[n - 1] = B.rows[n - 1], B.rows[0]
    tD, _ = eliminate(D, collect_minors=False)
    tB, _ = eliminate(B, collect_minors=False, pivot_mode="partial")
    assert [canonical_bits(x) for x in tB.pivots] == [canonical_bits(x) for x in tD.pivots]
    with Precision(p).context():
        flipped = [canonical_bits(-x) for x in tD.det_series]
    assert [canonical_bits(x) for x in tB.det_series] == flipped
    assert [canonical_bits(x) for r in B.rows for x in r] == [canonical_bits(x) for r in D.rows for x in r]


def test_swap_signs_keep_full_precision():
    """The sign applied to the fetched det chain is an exact negation at p bits
    (not a rounding to the ambient default precision)."""
    from paper_1308_1536_b200.elim import EliminationTrace, _apply_swap_signs
    P = Precision(512)
    with P.context():
        third = mp.mpfr(1) / 3
        dets = [third, third * 7, third * 11]
    tr = EliminationTrace(n=3, prec=P)
    tr.det_series = list(dets)
    _apply_swap_signs(tr, [True, False, True], 0)
    with P.context():
        want = [-dets[0], -dets[1], dets[2]]
    assert [canonical_bits(x) for x in tr.det_series] == [canonical_bits(x) for x in want]
    assert tr.det_series[0].precision == 512
