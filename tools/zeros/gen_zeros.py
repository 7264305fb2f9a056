"""Parallel zeta-zero generation (input data prep; follows the reference's
scripts/make_zeros.py:37-45: mp.prec = bits + 64, nstr with bits*0.30103+5
digits).  Worker k writes raw decimal strings for its slice; merge_zeros.py
rounds them at `bits` and writes the reference's zeros-file format.

usage: python gen_zeros.py START END BITS OUTFILE
"""
import os
import sys
import time

os.environ.setdefault("MPMATH_NOGMPY", "1")
import mpmath  # noqa: E402

start, end, bits, out = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), sys.argv[4]
mpmath.mp.prec = bits + 64
digits = int(bits * 0.30103) + 5
t0 = time.time()
with open(out, "a") as f:
    for k in range(start, end + 1):
        z = mpmath.zetazero(k)
        f.write(f"{k} {mpmath.nstr(z.imag, digits, strip_zeros=False)}\n")
        f.flush()
        print(f"{k} {time.time() - t0:.0f}s", flush=True)
