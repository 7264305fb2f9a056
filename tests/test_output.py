"""Output path: dets.txt / minors_<m>.txt as the reference CLI
writes them (cli.py:218-232).  The native writer (csrc/hostio.c) and the Python
writer (output.py) are compared byte for byte with files the UNMODIFIED
reference wrote for the same inputs (tests/golden/make_output_goldens.py).
The results come from the CPU oracle, which is bit-identical to the
reference (tests/test_oracle_golden.py)."""
import filecmp
import os
import random

import pytest

import oracle
from paper_1308_1536_b200 import genmat, mp
from paper_1308_1536_b200.elim import EliminationTrace, MinorSeries, minor_rows_from_results
from paper_1308_1536_b200.engine import HostResults
from paper_1308_1536_b200.matrix import MatrixBuffer
from paper_1308_1536_b200.output import write_dets, write_minors, write_results
from paper_1308_1536_b200.scalars import Precision, canonical_bits

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "output")
P256 = Precision(256)


def _complex8():
    prec = Precision(192)
    rnd = random.Random(9)
    with prec.context():
        rows = [[mp.mpc(mp.mpfr(rnd.uniform(-1, 1)), mp.mpfr(rnd.uniform(-1, 1))) for _ in range(8)] for _ in range(8)]
    return MatrixBuffer(8, "complex", prec, rows)


CASES = {
    "identity3": (lambda: MatrixBuffer.from_rows([[1, 0, 0], [0, 1, 0], [0, 0, 1]], P256), None, True),
    "zero_pivot3": (lambda: MatrixBuffer.from_rows([[1, 2, 3], [2, 4, 5], [1, 1, 1]], P256), None, True),
    "uniform13_s5_p192": (lambda: genmat.synth_matrix("random_uniform", 13, 5, Precision(192)), None, True),
    "uniform13_s5_p192_d25": (lambda: genmat.synth_matrix("random_uniform", 13, 5, Precision(192)), 25, True),
    "hilbert12_p100": (lambda: genmat.synth_matrix("hilbert", 12, 0, Precision(100)), None, True),
    "series_false_u6": (lambda: genmat.synth_matrix("random_uniform", 6, 8, P256), None, False),
    "complex8_r9_p192": (_complex8, None, True),
}


def _run(A, series):
    n, p = A.n, A.prec.bits
    ref = oracle.OracleRank(n, p, A.kind)
    ref.load(A.to_soa())
    res = HostResults.alloc(n, 2 if A.kind == "complex" else 1, ref.L, True)
    rc, done = ref.run(True, series, 0, n, res)
    return res, done


def _same_tree(a, b):
    fa, fb = sorted(os.listdir(a)), sorted(os.listdir(b))
    assert fa == fb, (fa, fb)
    mism = [f for f in fa if not filecmp.cmp(os.path.join(a, f), os.path.join(b, f), shallow=False)]
    assert not mism, mism


@pytest.mark.parametrize("name", sorted(CASES))
def test_native_writer_matches_reference_files(name, tmp_path):
    build, digits, series = CASES[name]
    A = build()
    res, done = _run(A, series)
    write_results(res, A.n, A.prec.bits, A.kind, tmp_path, done, digits=digits)
    _same_tree(os.path.join(GOLD, name), tmp_path)


@pytest.mark.parametrize("name", sorted(CASES))
def test_python_writer_matches_reference_files(name, tmp_path):
    build, digits, series = CASES[name]
    A = build()
    res, done = _run(A, series)
    p = A.prec.bits
    dig = digits or A.prec.decimal_digits
    trace = EliminationTrace(n=A.n, prec=A.prec)
    trace.det_series = [res.dets.get(i, p) for i in range(done)]
    minors = MinorSeries(A.prec)
    for row in minor_rows_from_results(res, A.n, p):
        minors.rows[row.n] = row
    write_dets(trace, os.path.join(tmp_path, "dets.txt"), dig)
    write_minors(minors, tmp_path, dig)
    _same_tree(os.path.join(GOLD, name), tmp_path)


# ---------------------------------------------------------------- checkpoints
from paper_1308_1536_b200.checkpoint import Checkpoint, load_mpmat  # noqa: E402
from paper_1308_1536_b200.soa import SoA  # noqa: E402

CKPT = {"uniform13_s5_p192_step4": (lambda: genmat.synth_matrix("random_uniform", 13, 5, Precision(192)), 4),
        "complex8_r9_p192_step3": (_complex8, 3)}


def _oracle_state(A, steps):
    n, p = A.n, A.prec.bits
    ref = oracle.OracleRank(n, p, A.kind)
    ref.load(A.to_soa())
    res = HostResults.alloc(n, 2 if A.kind == "complex" else 1, ref.L, True)
    ref.run(True, True, 0, steps, res)
    cur = A.to_soa()
    ref.fetch(cur)
    pivots = [res.pivots.get(i, p) for i in range(steps)]
    return cur, pivots


@pytest.mark.parametrize("name", sorted(CKPT))
def test_checkpoint_write_matches_reference(name, tmp_path):
    build, steps = CKPT[name]
    A = build()
    cur, pivots = _oracle_state(A, steps)
    Checkpoint(tmp_path).write_soa(cur, A.n, A.prec.bits, A.kind, steps, pivots)
    _same_tree(os.path.join(GOLD, "ckpt_" + name), tmp_path)


@pytest.mark.parametrize("name", sorted(CKPT))
def test_checkpoint_load_and_resume(name):
    """Loading the reference's checkpoint gives its exact state; resuming from it
    ends bit-identical to the uninterrupted run."""
    build, steps = CKPT[name]
    A = build()
    n, p = A.n, A.prec.bits
    cur, pivots = _oracle_state(A, steps)
    soa, n2, bits, kind, trace = Checkpoint(os.path.join(GOLD, "ckpt_" + name)).load_soa()
    assert (n2, bits, kind, trace.step) == (n, p, A.kind, steps)
    assert [soa.canonical(i, p) for i in range(n * n)] == [cur.canonical(i, p) for i in range(n * n)]
    assert [canonical_bits(a) for a in trace.pivots] == [canonical_bits(b) for b in pivots]
    # resume: load the state, seed the det chain, run the remaining steps
    nc = 2 if A.kind == "complex" else 1
    ref = oracle.OracleRank(n, p, A.kind)
    ref.load(soa)
    ref.set_det(SoA.from_scalars([trace.det_series[-1]], p, A.kind))
    res_r = HostResults.alloc(n, nc, ref.L, True)
    ref.run(True, True, steps, n, res_r)
    fin_r = soa.copy()
    ref.fetch(fin_r)
    full = oracle.OracleRank(n, p, A.kind)
    full.load(A.to_soa())
    res_f = HostResults.alloc(n, nc, full.L, True)
    full.run(True, True, 0, n, res_f)
    fin_f = A.to_soa()
    full.fetch(fin_f)
    assert [fin_r.canonical(i, p) for i in range(n * n)] == [fin_f.canonical(i, p) for i in range(n * n)]
    for m in range(steps + 2, n + 1):  # minors emitted after the resume point
        base = (m - 1) * n
        assert [res_r.signed.canonical(base + k, p) for k in range(m)] == \
            [res_f.signed.canonical(base + k, p) for k in range(m)]
    for i in range(steps, n):
        assert res_r.dets.canonical(i, p) == res_f.dets.canonical(i, p)


def test_mpmat_roundtrip_random(tmp_path):
    """save_mpmat -> load_mpmat is the identity on the bits (format_scalar's default digits)."""
    from paper_1308_1536_b200.checkpoint import save_mpmat
    from paper_1308_1536_b200.synth import random_uniform_soa
    for n, p in ((17, 333), (9, 4096)):
        S = random_uniform_soa(n, p, seed=n + p)
        path = os.path.join(tmp_path, f"m{n}.mpmat")
        save_mpmat(S, n, p, "real", path)
        T, n2, p2, kind = load_mpmat(path)
        assert (n2, p2, kind) == (n, p, "real")
        assert [T.canonical(i, p) for i in range(n * n)] == [S.canonical(i, p) for i in range(n * n)]


def test_minors_stream_binary_round_trip(tmp_path):
    """DSMR v1 records written by output.MinorsStream (the consumer of the device's minors
    stream) read back bit for bit; rows without the emitted flag are skipped."""
    import numpy as np
    from paper_1308_1536_b200.output import MinorsStream, read_minors_binary
    from paper_1308_1536_b200.synth import random_uniform_soa
    n, p = 6, 100
    s, t = random_uniform_soa(n, p, 3), random_uniform_soa(n, p, 4)
    path = tmp_path / "x.dsmr"
    st = MinorsStream(n, p, path=str(path), keep_upto=n)
    st(1, 1, 3, s, t, np.array([3, 1, 3], dtype=np.uint8))
    st(4, 1, 2, s, t, np.array([0, 3], dtype=np.uint8))
    st.close()
    rows = list(read_minors_binary(str(path)))
    assert [(m, fl) for m, fl, _, _ in rows] == [(2, 3), (3, 1), (4, 3), (6, 3)]
    for m, fl, sg, nm in rows:
        r = m - 2 if m <= 4 else m - 5
        sl = slice(r * n, r * n + m)
        assert np.array_equal(sg.limbs, s.limbs[:, :, sl]) and np.array_equal(sg.exp, s.exp[:, sl])
        assert (nm is None) == (not fl & 2)
        if nm is not None:
            assert np.array_equal(nm.limbs, t.limbs[:, :, sl])
    assert st.sizes == [2, 3, 4, 6] and st.digest.startswith("sum64:")


def test_write_results_applies_partial_pivot_swap_signs(tmp_path):
    """write_results(..., swaps=) writes the signed det_series of a pivot_mode="partial" run: the
    device keeps the unsigned pivot product and every row swap flips the sign of all later
    determinants (elim.py:207, 216) -- an exact sign flip of the class byte."""
    from paper_1308_1536_b200 import mp
    from paper_1308_1536_b200.engine import HostResults
    from paper_1308_1536_b200.output import write_results
    from paper_1308_1536_b200.scalars import format_scalar
    n, p = 4, 128
    res = HostResults.alloc(n, 1, (p + 31) // 32, False)
    with mp.context(precision=p):
        vals = [mp.mpfr(3), mp.mpfr(-5), mp.mpfr(7), mp.mpfr(0)]
    for i, v in enumerate(vals):
        res.dets.set(i, v, p)
    write_results(res, n, p, "real", tmp_path, n, digits=10, minors=False, swaps=[False, True, False, True])
    got = (tmp_path / "dets.txt").read_text().splitlines()
    with mp.context(precision=p):
        want = [vals[0], -vals[1], -vals[2], vals[3]]  # sign flips from step 1 on, back at step 3
    assert got == [f"{i + 1} {format_scalar(w, 10)}" for i, w in enumerate(want)]
