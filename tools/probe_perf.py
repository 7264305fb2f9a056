"""Quick timing probe of full eliminations on one GPU (not the bench)."""
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_1308_1536_b200.engine import DeviceElimination, HostResults  # noqa: E402
from paper_1308_1536_b200.synth import random_uniform_soa  # noqa: E402

for spec in sys.argv[1:]:
    n, p = map(int, spec.split("@"))
    A = random_uniform_soa(n, p, 1)
    L = (p + 31) // 32
    with DeviceElimination(n, p, "real") as eng:
        res = HostResults.alloc(n, 1, L, True)
        eng.load(A)
        t0 = time.perf_counter()
        rc, done = eng.run(True, True, 0, n, res)
        t1 = time.perf_counter()
        work = n * (n - 1) ** 2 / 2 * L * L
        print(f"n={n} p={p} done={done} wall={t1 - t0:.3f}s (incl. results D2H) "
              f"limb-MAC/s={work / (t1 - t0):.3e} launches={eng.launches()}", flush=True)
