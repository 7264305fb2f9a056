"""Quick timing probe of full eliminations on one GPU (not the bench).

usage: python tools/probe_perf.py 1000@4096 2000@4096 ...
Prints wall time, update-kernel time (profile events), the engine counters
(tensor-core fallback elements, which update engine ran)."""
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402,F401

from paper_1308_1536_b200.engine import DeviceElimination, HostResults  # noqa: E402
from paper_1308_1536_b200.synth import random_uniform_soa  # noqa: E402

series = True
fetch = True
specs = []
for arg in sys.argv[1:]:
    if arg == "--no-fetch":
        fetch = False  # results stay in HBM (no pinned host copy of the minors)
    elif arg == "--no-series":
        series = False  # minors emitted only at the last step (same update work)
    else:
        specs.append(arg)
for spec in specs:
    kind = "complex" if spec.endswith("c") else "real"  # 1000@4096c: complex elements
    n, p = map(int, spec.rstrip("c").split("@"))
    A = random_uniform_soa(n, p, 1, kind=kind)
    L = (p + 31) // 32
    with DeviceElimination(n, p, kind) as eng:
        res = HostResults.alloc(n, eng.ncomp, L, True, pinned=True) if fetch else None
        eng.load(A)
        eng.profile(True)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        rc, done = eng.run(True, series, 0, n, None)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        if fetch:
            eng.results(n, res)
        t2 = time.perf_counter()
        ms, nl, w = eng.profile_read()
        work = n * (n - 1) ** 2 / 2 * L * L * (4 if kind == "complex" else 1)
        print(f"n={n} p={p} kind={kind} series={series} done={done} device={t1 - t0:.3f}s results-D2H={t2 - t1:.3f}s "
              f"limb-MAC/s={work / (t1 - t0):.3e} update={ms / 1e3:.3f}s ({w / (ms * 1e-3):.3e}/s over {nl} launches) "
              f"launches={eng.launches()} {eng.counters()}", flush=True)
