import sys, time, json, cProfile, pstats, io
sys.path.insert(0, ".")
import torch
from paper_1308_1536_b200 import MatrixBuffer, Precision, eliminate
from paper_1308_1536_b200.synth import random_uniform_soa
n, p = 2000, 4096
torch.cuda.synchronize()
for rep in range(3):
    soa = random_uniform_soa(n, p, seed=n)
    A = MatrixBuffer.from_soa(n, "real", Precision(p), soa)
    rows = []
    pr = cProfile.Profile() if rep == 2 else None
    t0 = time.perf_counter()
    if pr: pr.enable()
    eliminate(A, sink=rows.append)
    if pr: pr.disable()
    print("rep", rep, time.perf_counter() - t0, flush=True)
    del rows, A
s = io.StringIO(); pstats.Stats(pr, stream=s).sort_stats("cumulative").print_stats(25); print(s.getvalue())
