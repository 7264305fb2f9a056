"""Kernel timeline of a window of elimination steps (CUPTI via torch.profiler).

usage: python tools/trace_steps.py N P[c] START STOP [out.json]   (Pc: complex)
Runs steps [0, START) untraced, traces [START, STOP), prints per-kernel totals,
per-stream busy time and the idle gaps of the main stream."""
import collections
import json
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_1308_1536_b200.engine import DeviceElimination, HostResults  # noqa: E402
from paper_1308_1536_b200.synth import random_uniform_soa  # noqa: E402

kind = "complex" if sys.argv[2].endswith("c") else "real"  # P suffix c: complex elements
sys.argv[2] = sys.argv[2].rstrip("c")
n, p, start, stop = map(int, sys.argv[1:5])
out = sys.argv[5] if len(sys.argv) > 5 else "gpurun_out/trace.json"
A = random_uniform_soa(n, p, 1, kind=kind)
L = (p + 31) // 32
with DeviceElimination(n, p, kind) as eng:
    res = HostResults.alloc(n, eng.ncomp, L, True)
    eng.load(A)
    eng.run(True, True, 0, start, res)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
        eng.run(True, True, start, stop, None)
        torch.cuda.synchronize()
    prof.export_chrome_trace(out)
ev = json.load(open(out))["traceEvents"]
k = [e for e in ev if e.get("cat") in ("kernel", "gpu_memset", "gpu_memcpy")]
k.sort(key=lambda e: e["ts"])
tot = collections.defaultdict(lambda: [0, 0.0])
streams = collections.defaultdict(float)
for e in k:
    nm = e["name"].replace("(anonymous namespace)::", "").replace("void ", "").split("(")[0][:40]
    tot[nm][0] += 1
    tot[nm][1] += e["dur"]
    streams[e["args"].get("stream", -1)] += e["dur"]
span = (k[-1]["ts"] + k[-1]["dur"] - k[0]["ts"]) if k else 0
steps = stop - start
print(f"window {steps} steps, span {span / 1e3:.3f} ms ({span / steps:.1f} us/step)")
for nm, (c, d) in sorted(tot.items(), key=lambda x: -x[1][1]):
    print(f"  {nm:40s} n={c:5d} total={d / 1e3:9.3f} ms avg={d / c:8.1f} us  per-step={d / steps:8.1f} us")
for s, d in streams.items():
    print(f"  stream {s}: busy {d / 1e3:.3f} ms ({100 * d / span:.1f}% of span)")
# gaps on the busiest stream
main = max(streams, key=streams.get)
mk = [e for e in k if e["args"].get("stream", -1) == main]
gaps = [(mk[i + 1]["ts"] - (mk[i]["ts"] + mk[i]["dur"]), mk[i]["name"][:30], mk[i + 1]["name"][:30])
        for i in range(len(mk) - 1)]
g = [x for x in gaps if x[0] > 0]
print(f"main stream {main}: idle {sum(x[0] for x in g) / 1e3:.3f} ms in {len(g)} gaps; largest:")
for x in sorted(g, reverse=True)[:8]:
    print("   ", x)
