"""Where the end-to-end time goes: H2D load, run (resident outputs), run with
results into pinned host buffers (progressive minors D2H), final fetch.

usage: python tools/e2e_probe.py N P"""
import os
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_1308_1536_b200.engine import DeviceElimination, HostResults  # noqa: E402
from paper_1308_1536_b200.synth import random_uniform_soa  # noqa: E402

n, p = int(sys.argv[1]), int(sys.argv[2])
A = random_uniform_soa(n, p, 1, pinned=True)
L = (p + 31) // 32
res = HostResults.alloc(n, 1, L, True, pinned=True)


def t(fn):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    fn()
    torch.cuda.synchronize()
    return time.perf_counter() - t0


with DeviceElimination(n, p, "real") as eng:
    eng.load(A)
    eng.run(True, True, 0, n, None)  # warm
    tl = t(lambda: eng.load(A))
    tr = t(lambda: eng.run(True, True, 0, n, None))
    eng.load(A)
    tres = t(lambda: eng.run(True, True, 0, n, res))
    os.environ["DS_NO_PROGRESSIVE_D2H"] = "1"
    eng.load(A)
    tfull = t(lambda: eng.run(True, True, 0, n, res))
    tf = t(lambda: eng.results(n, res))
print(f"n={n} p={p}: load {tl:.3f}s  run {tr:.3f}s  run+results(progressive) {tres:.3f}s  "
      f"run+results(full fetch) {tfull:.3f}s  fetch alone {tf:.3f}s  "
      f"(H2D {A.nbytes / tl / 1e9:.1f} GB/s)")
