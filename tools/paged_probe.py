"""Time the panel-paged executor against the in-core run on the same matrix
(device time incl. the host store round trips).  usage: paged_probe.py N BITS PANEL"""
import json
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1308_1536_b200.engine import DeviceElimination, HostResults  # noqa: E402
from paper_1308_1536_b200.paged import paged_eliminate_soa  # noqa: E402
from paper_1308_1536_b200.synth import random_uniform_soa  # noqa: E402

n, p, panel = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
A = random_uniform_soa(n, p, seed=11, pinned=True)
with DeviceElimination(n, p, "real") as e:
    e.load(A)
    res = HostResults.alloc(n, 1, e.L, True, pinned=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e.run(True, True, 0, n, res)
    fin = A.copy()
    e.fetch(fin)
    t_core = time.perf_counter() - t0
store = A.copy()
t0 = time.perf_counter()
pres, done = paged_eliminate_soa(store, n, p, "real", panel)
t_paged = time.perf_counter() - t0
same = bool(np.array_equal(store.limbs, fin.limbs) and np.array_equal(pres.dets.limbs, res.dets.limbs))
print(json.dumps({"n": n, "prec_bits": p, "panel_rows": panel, "panels": (n + panel - 1) // panel,
                  "in_core_s": t_core, "paged_s": t_paged, "bit_identical": same,
                  "pivot_row_reloads": sum(range(0, n, panel))}))
