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
from paper_1308_1536_b200.scalars import Precision

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
