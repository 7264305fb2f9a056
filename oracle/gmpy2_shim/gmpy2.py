"""gmpy2-API shim over the system MPFR 4.2.1 / MPC 1.3.1 / GMP 6.3.0 (ctypes).

TEST INFRASTRUCTURE ONLY.  gmpy2 is not installed in this image and cannot
be installed offline.  The reference package
(/root/reference/pkg/src/detseries) imports gmpy2 for every scalar; putting
this directory on sys.path lets the UNMODIFIED reference run in this
container so that tests/golden/make_goldens.py can record its outputs and
pin the C oracle (oracle/ds_oracle.c) against them.

It covers exactly the surface the reference uses (grep of src/, tests/,
scripts/): mpfr, mpc, mpz, mpq, context(precision=), random_state,
mpfr_random, const_pi, exp, log, log2, log10, sqrt, sin, cos, factorial,
gamma, is_finite, is_signed, mul_2exp, div_2exp and arithmetic/comparison
with int, float and Fraction.  Every arithmetic result is the correctly
rounded (RNDN) MPFR/MPC result at the active context precision, which is
what gmpy2 computes; integer and float operands are converted exactly
first.

The implementation is the product's host scalar module
(paper_1308_1536_b200/mp.py, a superset of this surface); this file only
re-exports it under the name the reference imports, so there is one copy of
the MPFR/MPC bindings.

Known deviation risk (documented in DESIGN.md): gmpy2.mpfr_random is
restated as mpfr_urandom(RNDN) over gmp_randinit_default + gmp_randseed,
which is believed (not verified, no real gmpy2 here) to be gmpy2's
implementation.  Parity never depends on it: both sides of every parity test
consume the same recorded inputs.
"""

import os as _os
import sys as _sys

_ROOT = _os.path.dirname(_os.path.dirname(_os.path.dirname(_os.path.abspath(__file__))))
if _ROOT not in _sys.path:
    _sys.path.insert(0, _ROOT)

from paper_1308_1536_b200.mp import *  # noqa: E402,F401,F403

