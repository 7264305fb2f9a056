"""Kernel timeline of steps [START, STOP) of the Artless zero-power matrix (complex,
the bench's --family power input) -- where a complex elimination spends its time.

usage: python tools/trace_power.py N P START STOP"""
import collections
import json
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_1308_1536_b200 import hostgen  # noqa: E402
from paper_1308_1536_b200.engine import DeviceElimination, HostResults  # noqa: E402

n, p, start, stop = map(int, sys.argv[1:5])
ZEROS = "data/zeta_zeros_4096.txt"
from paper_1308_1536_b200.soa import SoA  # noqa: E402
M = n // 2
N = 2 * M + 1
full = hostgen.power_matrix_soa(ZEROS, M, p)
L = (p + 31) // 32
A = SoA(2, L, n * n)
A.limbs[...] = full.limbs.reshape(2, L, N, N)[:, :, :n, :n].reshape(2, L, -1)
A.exp[...] = full.exp.reshape(2, N, N)[:, :n, :n].reshape(2, -1)
A.cls[...] = full.cls.reshape(2, N, N)[:, :n, :n].reshape(2, -1)
with DeviceElimination(n, p, "complex") as eng:
    res = HostResults.alloc(n, 2, L, True)
    eng.load(A)
    if start:
        eng.run(True, True, 0, start, res)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        eng.run(True, True, start, stop, None)
        torch.cuda.synchronize()
    out = "gpurun_out/trace_power.json"
    prof.export_chrome_trace(out)
    print("counters", eng.counters())
ev = json.load(open(out))["traceEvents"]
agg = collections.defaultdict(lambda: [0, 0.0])
for e in ev:
    if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset"):
        name = e["name"].split("(")[0].replace("(anonymous namespace)::", "")
        agg[name][0] += 1
        agg[name][1] += e.get("dur", 0.0)
print(f"steps [{start}, {stop})")
for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:12]:
    print(f"  {k:40s} n={c:5d} total={t / 1e3:9.3f} ms")
