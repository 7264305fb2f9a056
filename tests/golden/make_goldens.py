"""Record golden vectors from the UNMODIFIED reference (test infrastructure).

Run in this container only (the reference is absent on the GPU box):

    MPMATH_NOGMPY=1 PYTHONPATH=oracle/gmpy2_shim:/root/reference/pkg/src \
        python tests/golden/make_goldens.py

The reference package imports gmpy2; oracle/gmpy2_shim supplies the gmpy2 API
over the system MPFR/MPC that gmpy2 itself wraps.  For every case we store the
input matrix in the ds SoA format (or, for large generated inputs, the
generator call plus the reference's MatrixBuffer.fingerprint()), the exact
outputs of the reference's eliminate() (elim.py:158-229) as SoA arrays, and a
digest (tests/golden/digest.py) of trace, minors and final buffer.
"""

import json
import os
import random
import sys
from fractions import Fraction

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

import gmpy2  # noqa: E402  (the shim)
from detseries.elim import eliminate  # noqa: E402
from detseries.errors import ZeroPivot  # noqa: E402
from detseries.genmat import SpougeGamma, beta_matrix, load_zeros, power_matrix, synth_matrix  # noqa: E402
from detseries.matrix import MatrixBuffer  # noqa: E402
from detseries.parexec import par_eliminate  # noqa: E402
from detseries.scalars import Precision, canonical_bits  # noqa: E402
from gmpy2 import mpc  # noqa: E402
from digest import digest_parts  # noqa: E402

ZEROS = "/root/reference/pkg/data/zeta_zeros.txt"


def limbs_of(x, prec):
    """(L little-endian u32 limbs, exp, cls) of a shim mpfr at `prec`."""
    L = (prec + 31) // 32
    if x == 0:
        return [0] * L, 0, (3 if gmpy2.is_signed(x) else 2)
    m, e = x.as_mantissa_exp()
    m, e = int(m), int(e)
    neg = m < 0
    mag = abs(m)
    p = x.precision
    assert p == prec, (p, prec)
    M = mag << (32 * L - p)  # left-aligned in 32L bits
    assert M.bit_length() == 32 * L
    limbs = [(M >> (32 * k)) & 0xFFFFFFFF for k in range(L)]
    return limbs, e + p, (1 if neg else 0)


def soa_of(values, prec, kind):
    ncomp = 2 if kind == "complex" else 1
    L = (prec + 31) // 32
    n = len(values)
    limbs = np.zeros((ncomp, L, n), dtype=np.uint32)
    exp = np.zeros((ncomp, n), dtype=np.int32)
    cls = np.full((ncomp, n), 2, dtype=np.uint8)
    for i, x in enumerate(values):
        parts = (x,) if ncomp == 1 else (x.real, x.imag)
        for c, v in enumerate(parts):
            lb, e, k = limbs_of(v, prec)
            limbs[c, :, i] = lb
            exp[c, i] = e
            cls[c, i] = k
    return limbs, exp, cls


def run_case(name, A, collect_minors=True, series=True, store_input=True, gen=None, par_workers=None):
    n, prec, kind = A.n, A.prec.bits, A.kind
    original = A.copy()
    fp = A.fingerprint()
    flat_in = [x for row in A.rows for x in row]
    zp = None
    try:
        if par_workers:
            trace, minors, _ = par_eliminate(A, par_workers, transport="local", collect_minors=collect_minors,
                                             series=series)
        else:
            trace, minors = eliminate(A, collect_minors=collect_minors, series=series)
    except ZeroPivot as exc:
        zp = exc.step
        trace, minors = exc.trace, exc.series
    rows = []
    if minors is not None:
        for m in minors.sizes():
            r = minors.rows[m]
            rows.append((m, [canonical_bits(x) for x in r.signed],
                         None if r.normalized is None else [canonical_bits(x) for x in r.normalized]))
    dig = digest_parts([canonical_bits(x) for x in trace.pivots], [canonical_bits(x) for x in trace.det_series],
                       rows, [canonical_bits(x) for row in A.rows for x in row])
    meta = dict(name=name, n=n, prec=prec, kind=kind, collect_minors=collect_minors, series=series,
                zero_pivot_step=zp, steps=trace.step, fingerprint=fp, digest=dig, gen=gen,
                emitted=[m for m, _, _ in rows])
    arrays = {}
    if store_input:
        arrays["in_limbs"], arrays["in_exp"], arrays["in_cls"] = soa_of(flat_in, prec, kind)
        # full outputs for small cases
        arrays["piv_limbs"], arrays["piv_exp"], arrays["piv_cls"] = soa_of(trace.pivots, prec, kind)
        arrays["det_limbs"], arrays["det_exp"], arrays["det_cls"] = soa_of(trace.det_series, prec, kind)
        arrays["out_limbs"], arrays["out_exp"], arrays["out_cls"] = soa_of(
            [x for row in A.rows for x in row], prec, kind)
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), meta=json.dumps(meta), **arrays)
    print(f"{name}: n={n} p={prec} {kind} steps={trace.step} zp={zp} digest={dig[:16]}", flush=True)
    del original


def main():
    P256 = Precision(256)
    run_case("worked_2x2", MatrixBuffer.from_rows([[1, 2], [3, 4]], P256))
    run_case("worked_3x3", MatrixBuffer.from_rows([[2, 1, 1], [1, 3, 2], [1, 0, 0]], P256))
    run_case("identity3", MatrixBuffer.from_rows([[1, 0, 0], [0, 1, 0], [0, 0, 1]], P256))
    run_case("zero_pivot3", MatrixBuffer.from_rows([[1, 2, 3], [2, 4, 5], [1, 1, 1]], P256))
    for seed in range(5):  # test_elim.py:53-72
        rng = random.Random(seed)
        entries = [[rng.randint(-5, 5) for _ in range(7)] for _ in range(7)]
        run_case(f"int7_s{seed}", MatrixBuffer.from_rows(entries, Precision(512)))
    for seed in range(3):  # criterion 1 style rationals (test_acceptance.py:58-78)
        rng = random.Random(100 + seed)
        n = rng.randint(3, 8)
        entries = [[Fraction(rng.randint(-9, 9), rng.randint(1, 5)) for _ in range(n)] for _ in range(n)]
        with Precision(512).context():
            rows = [[gmpy2.mpfr(gmpy2.mpq(x.numerator, x.denominator)) for x in r] for r in entries]
        run_case(f"rational_s{seed}", MatrixBuffer(n, "real", Precision(512), rows))
    run_case("uniform13_s5_p192", synth_matrix("random_uniform", 13, 5, Precision(192)),
             gen=["random_uniform", 13, 5, 192])
    run_case("uniform12_s17_p256", synth_matrix("random_uniform", 12, 17, P256), gen=["random_uniform", 12, 17, 256])
    run_case("uniform30_s4_p256", synth_matrix("random_uniform", 30, 4, P256), gen=["random_uniform", 30, 4, 256])
    run_case("uniform20_s3_p64", synth_matrix("random_uniform", 20, 3, Precision(64)),
             gen=["random_uniform", 20, 3, 64])
    run_case("hilbert12_p100", synth_matrix("hilbert", 12, 0, Precision(100)), gen=["hilbert", 12, 0, 100])
    run_case("illcond10_p333", synth_matrix("random_illcond", 10, 2, Precision(333)),
             gen=["random_illcond", 10, 2, 333])
    run_case("series_false_u6", synth_matrix("random_uniform", 6, 8, P256), series=False,
             gen=["random_uniform", 6, 8, 256])
    run_case("nominors_u9_p320", synth_matrix("random_uniform", 9, 11, Precision(320)), collect_minors=False,
             gen=["random_uniform", 9, 11, 320])
    run_case("uniform24_s2_p4096", synth_matrix("random_uniform", 24, 2, Precision(4096)),
             gen=["random_uniform", 24, 2, 4096])
    # complex 8x8 of test_parexec.py:147-157
    prec = Precision(192)
    rs = gmpy2.random_state(9)
    with prec.context():
        rows = [[mpc(2 * gmpy2.mpfr_random(rs) - 1, 2 * gmpy2.mpfr_random(rs) - 1) for _ in range(8)]
                for _ in range(8)]
    run_case("complex8_s9_p192", MatrixBuffer(8, "complex", prec, rows), par_workers=3)
    # complex with exact integer parts (zero-sign and exact-cancellation paths)
    rng = random.Random(77)
    with P256.context():
        rows = [[mpc(rng.randint(-3, 3), rng.randint(-3, 3)) for _ in range(6)] for _ in range(6)]
        rows[0][0] = mpc(2, 0)
    run_case("complex_int6", MatrixBuffer(6, "complex", P256, rows))
    # config 1a: beta matrix N=64 @256 (Artless Eq. 9)
    zeros = load_zeros(ZEROS, Precision(256), 64)
    run_case("beta64_p256", beta_matrix(zeros, 64, SpougeGamma(), Precision(256)), gen=["beta", 64, 256])
    # config 1b: power matrix M=32 (N=65) @256, t=25 (test_acceptance.py:264-268)
    zeros = load_zeros(ZEROS, Precision(2048), 32)
    with Precision(2048).context():
        t = gmpy2.mpfr(25)
    run_case("power32_p256", power_matrix(zeros, 32, t, Precision(256)), gen=["power", 32, 25, 256])
    # criterion 5 input: uniform N=128 seed 7 @1024 -- digest + fingerprint only
    run_case("uniform128_s7_p1024", synth_matrix("random_uniform", 128, 7, Precision(1024)), store_input=False,
             gen=["random_uniform", 128, 7, 1024])


if __name__ == "__main__":
    main()
