"""Per-rank device time of the row-cyclic sharded elimination, measured one rank at a
time on one GPU (the pool has one GPU per call): rank r of a world of W runs alone,
every non-owned step's pivot row arrives by ds_pivot_load (H2D of the final row i from
a world-1 run -- the bytes a broadcast delivers) and every owned step's row comes from
ds_pivot_stage, exactly as in dist_run.  Reports the rank's device time (CUDA events),
its update-kernel time and a bit-exact check of its rows against the world-1 result.
A projection for W GPUs: the rank's device time plus the per-step broadcast latency of
the real interconnect (not measured here).

usage: python tools/shard_projection.py [N] [BITS] [W ...]"""
import json
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1308_1536_b200.engine import DeviceElimination  # noqa: E402
from paper_1308_1536_b200.soa import SoA  # noqa: E402
from paper_1308_1536_b200.synth import random_uniform_soa  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
    p = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
    worlds = [int(x) for x in sys.argv[3:]] or [1, 2, 4, 8]
    A = random_uniform_soa(n, p, seed=n + p)
    L = (p + 31) // 32
    with DeviceElimination(n, p, "real") as e:
        e.load(A)
        e.run(True, True, 0, n, None)
        F = A.copy()
        e.fetch(F)
    rows = []
    for i in range(n):  # the final rows as count-n host SoAs (pinned: the H2D a broadcast replaces)
        r = SoA(1, L, n, pinned=True)
        r.limbs[...] = F.limbs[:, :, i * n:(i + 1) * n]
        r.exp[...] = F.exp[:, i * n:(i + 1) * n]
        r.cls[...] = F.cls[:, i * n:(i + 1) * n]
        rows.append(r)
    for W in worlds:
        for rank in sorted({0, W - 1}):
            with DeviceElimination(n, p, "real", 0, rank, W) as e:
                e.load(A)
                e.profile(True)
                e.profile_read()
                st = torch.cuda.ExternalStream(e.lib.ds_stream(e.ctx))
                ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                ev0.record(st)
                for i in range(n):
                    if i % W == rank:
                        e.stage(i)
                    else:
                        e.pivot_load(i, rows[i])
                    e.step(i, True, True)
                ev1.record(st)
                torch.cuda.synchronize()
                wall = time.perf_counter() - t0
                ms, nl, work = e.profile_read()
                fin = A.copy()
                e.fetch(fin)
            own = np.arange(rank, n, W)
            idx = (own[:, None] * n + np.arange(n)[None, :]).ravel()
            ok = bool(np.array_equal(fin.limbs[:, :, idx], F.limbs[:, :, idx]) and
                      np.array_equal(fin.exp[:, idx], F.exp[:, idx]) and np.array_equal(fin.cls[:, idx], F.cls[:, idx]))
            print(json.dumps({"n": n, "prec_bits": p, "world": W, "rank": rank, "rows": len(own),
                              "device_s": ev0.elapsed_time(ev1) / 1e3, "wall_s": wall, "update_s": ms / 1e3,
                              "update_launches": nl, "rows_bit_identical": ok}), flush=True)


if __name__ == "__main__":
    main()
