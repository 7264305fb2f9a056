"""Like gen_zeros.py but for an explicit list of indices (rebalancing)."""
import os
import sys
import time

os.environ.setdefault("MPMATH_NOGMPY", "1")
import mpmath  # noqa: E402

bits, out = int(sys.argv[1]), sys.argv[2]
ks = [int(x) for x in sys.argv[3:]]
mpmath.mp.prec = bits + 64
digits = int(bits * 0.30103) + 5
t0 = time.time()
with open(out, "a") as f:
    for k in ks:
        z = mpmath.zetazero(k)
        f.write(f"{k} {mpmath.nstr(z.imag, digits, strip_zeros=False)}\n")
        f.flush()
        print(f"{k} {time.time() - t0:.0f}s", flush=True)
