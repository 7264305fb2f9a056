"""Precompute Gamma(1/4 - i gamma_j/2) at p+64 bits for the first N zeros
(the column-only, expensive part of genmat.beta_entry, genmat.py:171) with the
C builder, into data/beta_gammas_p{p}_N{N}.npz.  tests/test_hostgen.py
recomputes sample columns and checks them bit for bit.

usage: python tools/make_beta_gamma_cache.py N P [THREADS]
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1308_1536_b200 import hostgen  # noqa: E402

N, P = int(sys.argv[1]), int(sys.argv[2])
threads = int(sys.argv[3]) if len(sys.argv) > 3 else 0
t0 = time.time()
g = hostgen.beta_gammas_soa(os.path.join(ROOT, "data", "zeta_zeros_4096.txt"), N, P, nthreads=threads)
out = os.path.join(ROOT, "data", f"beta_gammas_p{P}_N{N}.npz")
np.savez_compressed(out, L=g.L, count=g.count, limbs=g.limbs, exp=g.exp, cls=g.cls, prec=P + 64,
                    zeros="data/zeta_zeros_4096.txt")
print(f"wrote {out} in {time.time() - t0:.0f}s")
