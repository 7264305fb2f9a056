"""Config-5-style run on one GPU (BASELINE config 5 is N=10,000 @33,220 b over
8 GPUs; this measures what one B200 does at the headline precision): the input
is generated on the device (ds_generate, counter-based random_uniform), the
minors rows stream off the device as they finalise (ds_stream_minors: only a
ring of rows in HBM), and the run is checked against the oracle on the
leading m x m block (prefix property) plus Laplace residuals of the largest
sizes.  One JSON line on stdout.

usage: python tools/bigrun.py --n 3000 --bits 33220 [--batch 8] [--keep 96] [--out minors.dsmr]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
if hasattr(sys, "set_int_max_str_digits"):
    sys.set_int_max_str_digits(0)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1308_1536_b200.engine import DeviceElimination, HostResults  # noqa: E402
from paper_1308_1536_b200.output import MinorsStream  # noqa: E402
from paper_1308_1536_b200.soa import SoA  # noqa: E402
from paper_1308_1536_b200.synth import counter_uniform_soa  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=3000)
    ap.add_argument("--bits", type=int, default=33220)
    ap.add_argument("--seed", type=int, default=5)
    ap.add_argument("--batch", type=int, default=8)
    ap.add_argument("--keep", type=int, default=96)
    ap.add_argument("--out", default=None)
    ap.add_argument("--no-parity", action="store_true")
    a = ap.parse_args()
    n, p = a.n, a.bits
    L = (p + 31) // 32
    free0, total = torch.cuda.mem_get_info()
    st = MinorsStream(n, p, "real", path=a.out, keep_upto=a.keep, keep_sizes={n, n - 1})  # fast checksum
    out = {"n": n, "prec_bits": p, "limbs": L, "seed": a.seed, "batch_steps": a.batch}
    with DeviceElimination(n, p, "real") as e:
        e.stream_minors(a.batch, st)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e.generate(a.seed)
        torch.cuda.synchronize()
        out["generate_s"] = time.perf_counter() - t0
        res = HostResults.alloc(n, 1, L, False)
        e.profile(True)
        t0 = time.perf_counter()
        rc, done = e.run(True, True, 0, n, res)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        ms, nl, w = e.profile_read()
        free1, _ = torch.cuda.mem_get_info()
        out.update({"done": done, "seconds": dt, "update_s": ms / 1e3,
                    "limb_mac_per_s": n * (n - 1) ** 2 / 2 * L * L / dt,
                    "hbm_used_gb": (total - free1) / 1e9, "hbm_total_gb": total / 1e9,
                    "matrix_gb": n * n * (4 * L + 5) / 1e9,
                    "resident_minors_would_be_gb": 2 * n * n * (4 * L + 5) / 1e9,
                    "streamed_rows": len(st.sizes), "streamed_bytes": st.bytes, "stream_checksum": st.digest,
                    "counters": e.counters()})
    st.close()
    if not a.no_parity and done == n:
        import parity_check as pc
        m = min(a.keep, n)
        Am = counter_uniform_soa(m, p, a.seed, rows=np.arange(m), cols=np.arange(m))
        # the leading block of the n x n matrix: generate rows/cols < m with the n x n indexing
        Am = counter_uniform_soa(n, p, a.seed, rows=np.arange(m), cols=np.arange(m))
        full = HostResults(res.pivots, res.dets, SoA(1, L, n * n), SoA(1, L, n * n), np.zeros(n, np.uint8))
        # scatter the kept streamed rows (sizes <= m) into an n x n results view for the checker
        for msz, (fl, sg, nm) in st.kept.items():
            if msz > m:
                continue
            base = (msz - 1) * n
            full.signed.limbs[:, :, base:base + msz] = sg.limbs
            full.signed.exp[:, base:base + msz] = sg.exp
            full.signed.cls[:, base:base + msz] = sg.cls
            if nm is not None:
                full.normalized.limbs[:, :, base:base + msz] = nm.limbs
                full.normalized.exp[:, base:base + msz] = nm.exp
                full.normalized.cls[:, base:base + msz] = nm.cls
            full.row_flags[msz - 1] = fl
        # prefix() slices A's leading block from an n x n SoA: hand it an m x m matrix as n = m
        pre = pc.prefix(Am, m, p, "real", m, _restride(full, n, m), None)
        out["parity_prefix"] = pre
        lap = {}
        for size in (n, n - 1):
            fl, sg, nm = st.kept[size]
            col = counter_uniform_soa(n, p, a.seed, rows=np.arange(size), cols=[size - 1])
            lap[str(size)] = _laplace(col, sg, res.dets, size, p)
        out["laplace_log2"] = lap
        out["parity_ok"] = bool(pre["ok"]) and all(v < -p / 2 for v in lap.values())
    print(json.dumps(out), flush=True)


def _restride(full: HostResults, n: int, m: int) -> HostResults:
    """Results of an n-wide layout restricted to sizes <= m in an m-wide layout."""
    def cut(s):
        return SoA(1, s.L, m * m, np.ascontiguousarray(s.limbs.reshape(1, s.L, n, n)[:, :, :m, :m].reshape(1, s.L, -1)),
                   np.ascontiguousarray(s.exp.reshape(1, n, n)[:, :m, :m].reshape(1, -1)),
                   np.ascontiguousarray(s.cls.reshape(1, n, n)[:, :m, :m].reshape(1, -1)))
    return HostResults(full.pivots, full.dets, cut(full.signed), cut(full.normalized), full.row_flags[:m].copy())


def _laplace(col: SoA, signed: SoA, dets: SoA, size: int, p: int) -> float:
    """log2 |sum_k signed_k a_{k,size} - det_size| / |det_size| (elim.py:232-248)."""
    from paper_1308_1536_b200 import mp
    with mp.context(precision=p):
        acc = None
        for k in range(size):
            t = signed.get(k, p) * col.get(k, p)
            acc = t if acc is None else acc + t
        det = dets.get(size - 1, p)
        num = abs(acc - det)
        return float("-inf") if num == 0 else float(mp.log2(num / abs(det)))


if __name__ == "__main__":
    main()
