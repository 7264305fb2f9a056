"""Record the reference CLI's result files as golden text (test infrastructure).

Run in this container only (the reference is absent on the GPU box):

    MPMATH_NOGMPY=1 PYTHONPATH=oracle/gmpy2_shim:/root/reference/pkg/src \\
        python tests/golden/make_output_goldens.py

For a few cases of make_goldens.py (same inputs), the UNMODIFIED reference
runs eliminate() and writes dets.txt / minors_<m>.txt with its own
cli._write_dets / cli._write_minors (cli.py:218-232) at the CLI's default
digits (Precision.decimal_digits, cli.py:326) and, for one case, digits=25;
and, for two cases, a mid-run checkpoint directory with its own
cli._Checkpointer.write (matrix.mpmat + state.txt, cli.py:110-120).
tests/test_output.py compares the product's writers byte for byte.
"""

import os
import shutil
import sys

HERE = os.path.dirname(os.path.abspath(__file__))

import gmpy2  # noqa: E402,F401  (the shim)
from detseries.cli import _write_dets, _write_minors  # noqa: E402
from detseries.elim import eliminate  # noqa: E402
from detseries.errors import ZeroPivot  # noqa: E402
from detseries.genmat import synth_matrix  # noqa: E402
from detseries.matrix import MatrixBuffer  # noqa: E402
from detseries.scalars import Precision  # noqa: E402
from gmpy2 import mpc  # noqa: E402

OUT = os.path.join(HERE, "output")
P256 = Precision(256)


def record(name, A, digits=None, series=True):
    d = os.path.join(OUT, name)
    shutil.rmtree(d, ignore_errors=True)
    os.makedirs(d)
    dig = digits or A.prec.decimal_digits
    try:
        trace, minors = eliminate(A, collect_minors=True, series=series)
    except ZeroPivot as exc:  # the CLI writes the partial results (cli.py:345-351)
        trace, minors = exc.trace, exc.series
    _write_dets(trace, os.path.join(d, "dets.txt"), dig)
    _write_minors(minors, d, dig)
    print(name, sorted(os.listdir(d))[:4], "...")


def main():
    record("identity3", MatrixBuffer.from_rows([[1, 0, 0], [0, 1, 0], [0, 0, 1]], P256))
    record("zero_pivot3", MatrixBuffer.from_rows([[1, 2, 3], [2, 4, 5], [1, 1, 1]], P256))
    record("uniform13_s5_p192", synth_matrix("random_uniform", 13, 5, Precision(192)))
    record("uniform13_s5_p192_d25", synth_matrix("random_uniform", 13, 5, Precision(192)), digits=25)
    record("hilbert12_p100", synth_matrix("hilbert", 12, 0, Precision(100)))
    record("series_false_u6", synth_matrix("random_uniform", 6, 8, P256), series=False)
    prec = Precision(192)
    rows = []
    import random
    rnd = random.Random(9)
    with prec.context():
        for _ in range(8):
            rows.append([mpc(gmpy2.mpfr(rnd.uniform(-1, 1)), gmpy2.mpfr(rnd.uniform(-1, 1))) for _ in range(8)])
    record("complex8_r9_p192", MatrixBuffer(8, "complex", prec, rows))


def record_checkpoint(name, A, stop_after):
    """The reference's _Checkpointer.write (cli.py:110-120) after `stop_after` steps."""
    from detseries.cli import _Checkpointer
    d = os.path.join(OUT, "ckpt_" + name)
    shutil.rmtree(d, ignore_errors=True)
    ck = _Checkpointer(d, every=0)

    def hook(completed, buf, trace):
        if completed == stop_after:
            ck.write(buf, trace)
            return True
        return False

    eliminate(A, collect_minors=True, series=True, step_hook=lambda c, B, t: hook(c, B, t))
    print("ckpt", name, sorted(os.listdir(d)))


def main_ckpt():
    record_checkpoint("uniform13_s5_p192_step4", synth_matrix("random_uniform", 13, 5, Precision(192)), 4)
    prec = Precision(192)
    import random
    rnd = random.Random(9)
    with prec.context():
        rows = [[mpc(gmpy2.mpfr(rnd.uniform(-1, 1)), gmpy2.mpfr(rnd.uniform(-1, 1))) for _ in range(8)]
                for _ in range(8)]
    record_checkpoint("complex8_r9_p192_step3", MatrixBuffer(8, "complex", prec, rows), 3)


if __name__ == "__main__":
    main()
    main_ckpt()
