"""Precision sweep probe (BASELINE config 4: N=1000, p = 256 ... 32768).

usage: python tools/sweep_probe.py N STEPS p1 p2 ...
Runs the first STEPS elimination steps (all minors) of a random-uniform N x N
matrix at each precision, reports the device time and the extrapolated time of
the full elimination (work per step ~ (n-1-i) * n element updates)."""
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_1308_1536_b200.engine import DeviceElimination  # noqa: E402
from paper_1308_1536_b200.synth import random_uniform_soa  # noqa: E402

n, steps = int(sys.argv[1]), int(sys.argv[2])
for p in map(int, sys.argv[3:]):
    A = random_uniform_soa(n, p, 1)
    L = (p + 31) // 32
    with DeviceElimination(n, p, "real") as eng:
        eng.load(A)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        eng.run(True, True, 0, steps, None)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        done_w = sum((n - 1 - i) * (n - 1) for i in range(steps))
        all_w = sum((n - 1 - i) * (n - 1) for i in range(n))
        est = dt * all_w / done_w
        work = n * (n - 1) ** 2 / 2 * L * L
        print(f"p={p} L={L} steps={steps} t={dt:.3f}s -> full N={n} est {est:.2f}s "
              f"({work / est:.3e} limb-MAC/s) {eng.counters()}", flush=True)
