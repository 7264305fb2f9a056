"""Record pivot_mode="partial" golden vectors from the UNMODIFIED reference
(test infrastructure; run in this container only):

    MPMATH_NOGMPY=1 PYTHONPATH=oracle/gmpy2_shim:/root/reference/pkg/src \
        python tests/golden/partial/make_partial_goldens.py

Each case runs the reference's eliminate(A, collect_minors=False,
pivot_mode="partial") (elim.py:158-229, row swaps at 204-208) and stores the
input (SoA, or the builder call), the outcome (steps, ZeroPivot step) and the
digest of pivots, signed det series and the final buffer.  Kept apart from
tests/golden/*.npz, whose cases run without pivoting.
"""

import json
import os
import random
import sys

import numpy as np

sys.set_int_max_str_digits(0)  # fingerprints / digests of >4300-digit mantissas (p >= 16384)

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))

import gmpy2  # noqa: E402  (the shim)
from detseries.elim import eliminate  # noqa: E402
from detseries.errors import ZeroPivot  # noqa: E402
from detseries.genmat import synth_matrix  # noqa: E402
from detseries.matrix import MatrixBuffer  # noqa: E402
from detseries.scalars import Precision, canonical_bits  # noqa: E402
from digest import digest_parts  # noqa: E402
from make_goldens import soa_of  # noqa: E402


def run_case(name, A, gen=None):
    n, prec = A.n, A.prec.bits
    flat_in = [x for row in A.rows for x in row]
    fp = A.fingerprint()
    zp = None
    try:
        trace, _ = eliminate(A, collect_minors=False, pivot_mode="partial")
    except ZeroPivot as exc:
        zp = exc.step
        trace = exc.trace
    dig = digest_parts([canonical_bits(x) for x in trace.pivots], [canonical_bits(x) for x in trace.det_series],
                       [], [canonical_bits(x) for row in A.rows for x in row])
    meta = dict(name=name, n=n, prec=prec, kind=A.kind, collect_minors=False, series=True, pivot_mode="partial",
                zero_pivot_step=zp, steps=trace.step, fingerprint=fp, digest=dig, gen=gen,
                negative_dets=sum(1 for x in trace.det_series if x < 0))
    arrays = {}
    if gen is None:
        arrays["in_limbs"], arrays["in_exp"], arrays["in_cls"] = soa_of(flat_in, prec, A.kind)
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), meta=json.dumps(meta), **arrays)
    print(f"{name}: n={n} p={prec} steps={trace.step} zp={zp} digest={dig[:16]}", flush=True)


def main():
    P256 = Precision(256)
    # integer matrices: exact dets; many equal magnitudes (+k and -k) test the first-maximum rule
    for seed in range(4):
        rng = random.Random(seed)
        entries = [[rng.randint(-5, 5) for _ in range(7)] for _ in range(7)]
        run_case(f"pp_int7_s{seed}", MatrixBuffer.from_rows(entries, Precision(512)))
    rng = random.Random(41)
    entries = [[rng.choice([-2, -1, 1, 2]) for _ in range(12)] for _ in range(12)]
    run_case("pp_ties12_p320", MatrixBuffer.from_rows(entries, Precision(320)))
    # zero leading pivot that the unpivoted elimination rejects (ZeroPivot(2) without pivoting)
    run_case("pp_zero_pivot3", MatrixBuffer.from_rows([[1, 2, 3], [2, 4, 5], [1, 1, 1]], P256))
    # singular: a zero column below the diagonal at step 2 -> ZeroPivot even with pivoting
    run_case("pp_singular4", MatrixBuffer.from_rows([[2, 1, 1, 3], [4, 2, 5, 1], [6, 3, 2, 2], [1, 0.5, 7, 1]],
                                                    P256))
    run_case("pp_uniform20_s3_p64", synth_matrix("random_uniform", 20, 3, Precision(64)),
             gen=["random_uniform", 20, 3, 64])
    run_case("pp_hilbert12_p100", synth_matrix("hilbert", 12, 0, Precision(100)), gen=["hilbert", 12, 0, 100])
    run_case("pp_uniform30_s4_p256", synth_matrix("random_uniform", 30, 4, P256), gen=["random_uniform", 30, 4, 256])
    run_case("pp_illcond24_p333", synth_matrix("random_illcond", 24, 2, Precision(333)),
             gen=["random_illcond", 24, 2, 333])
    run_case("pp_uniform48_s6_p1024", synth_matrix("random_uniform", 48, 6, Precision(1024)),
             gen=["random_uniform", 48, 6, 1024])
    run_case("pp_uniform24_s2_p4096", synth_matrix("random_uniform", 24, 2, Precision(4096)),
             gen=["random_uniform", 24, 2, 4096])
    run_case("pp_uniform16_s1_p8192", synth_matrix("random_uniform", 16, 1, Precision(8192)),
             gen=["random_uniform", 16, 1, 8192])
    run_case("pp_uniform10_s2_p16384", synth_matrix("random_uniform", 10, 2, Precision(16384)),
             gen=["random_uniform", 10, 2, 16384])
    run_case("pp_uniform140_s9_p256", synth_matrix("random_uniform", 140, 9, P256),
             gen=["random_uniform", 140, 9, 256])


if __name__ == "__main__":
    main()
