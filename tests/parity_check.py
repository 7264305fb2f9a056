"""Parity checks of full-size device runs against the CPU oracle.

TEST INFRASTRUCTURE (imported by tests/ and by bench.py's `parity` field, as
the checker -- never on the measured path).  The oracle (oracle/ds_oracle.c)
restates elim.py:37-229 over MPFR and is pinned to the unmodified reference
by tests/golden/.

Three size-independent checks of one elimination of an n x n matrix whose
oracle run would take hours at full size:

  * leading steps -- the full matrix state after the first `steps` pivot steps
    (every element of every row, elim.py:203-218) against
    OracleRank(n, p).run(0, steps), compared as raw ds SoA arrays;
  * prefix       -- outputs for leading size m depend only on A[1..m,1..m]
    (elim.py:47-52; SURVEY.md 8(a) "prefix property"), so det_series[0..m),
    pivots[0..m), every minors row of size <= m (signed, normalized, None
    flags) and the final leading m x m block of the full run must equal an
    oracle run on that block;
  * Laplace      -- |sum_k signed_k a_{k,N} - det_N| / |det_N| on the original
    entries (elim.py:232-248), an independent check of any emitted size.

Arrays are compared byte for byte: the ds SoA form is canonical (left-aligned
mantissa with the MSB set and zero bits below p; zeros have zero limbs and
exponent), so equal bytes <=> equal canonical_bits (scalars.py:129-150).
"""
from __future__ import annotations

import math
import os
import time

import numpy as np

import oracle
from paper_1308_1536_b200 import mp
from paper_1308_1536_b200.engine import HostResults
from paper_1308_1536_b200.soa import SoA


def host_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:  # pragma: no cover
        return os.cpu_count() or 1


def block(s: SoA, n: int, m: int) -> SoA:
    """Leading m x m block of an n x n SoA matrix (row-major idx = row*n + col)."""
    nc, L = s.ncomp, s.L
    limbs = np.ascontiguousarray(s.limbs.reshape(nc, L, n, n)[:, :, :m, :m].reshape(nc, L, m * m))
    ex = np.ascontiguousarray(s.exp.reshape(nc, n, n)[:, :m, :m].reshape(nc, m * m))
    cl = np.ascontiguousarray(s.cls.reshape(nc, n, n)[:, :m, :m].reshape(nc, m * m))
    return SoA(nc, L, m * m, limbs, ex, cl)


def _mism(a: SoA, b: SoA, mask=None) -> int:
    """Number of elements whose (limbs, exp, cls) differ (optionally within mask)."""
    d = (a.limbs != b.limbs).any(axis=1).any(axis=0) | (a.exp != b.exp).any(axis=0) | (a.cls != b.cls).any(axis=0)
    if mask is not None:
        d &= mask
    return int(d.sum())


def leading_steps(A: SoA, n: int, p: int, kind: str, steps: int, device_final: SoA, device_res: HostResults,
                  collect_minors: bool = True) -> dict:
    """Full state after `steps` steps: device (already run and fetched) vs oracle."""
    t0 = time.perf_counter()
    r = oracle.OracleRank(n, p, kind, 0, 1, host_threads())
    r.load(A)
    res_o = HostResults.alloc(n, r.ncomp, r.L, collect_minors)
    rc, done = r.run(collect_minors, True, 0, steps, res_o)
    fin_o = A.copy()
    r.fetch(fin_o)
    r.close()
    out = {"steps": steps, "elements": n * n, "matrix_mismatches": _mism(fin_o, device_final),
           "trace_mismatches": _mism(_head(res_o.dets, done), _head(device_res.dets, done))
           + _mism(_head(res_o.pivots, done), _head(device_res.pivots, done)),
           "oracle_s": time.perf_counter() - t0}
    if collect_minors and device_res.signed is not None:
        out["minors_mismatches"] = _minors_mism(res_o, device_res, n, n, min(steps + 1, n))
    out["ok"] = out["matrix_mismatches"] == 0 and out["trace_mismatches"] == 0 and out.get("minors_mismatches", 0) == 0
    return out


def _head(s: SoA, k: int) -> SoA:
    return SoA(s.ncomp, s.L, k, np.ascontiguousarray(s.limbs[:, :, :k]), np.ascontiguousarray(s.exp[:, :k]),
               np.ascontiguousarray(s.cls[:, :k]))


def _minors_mism(ro: HostResults, rd: HostResults, no: int, nd: int, m: int) -> int:
    """Mismatches over minors rows of sizes 2..m: flags, signed[0..size), normalized when defined.
    ro has row stride no, rd row stride nd."""
    bad = int((ro.row_flags[:m] != rd.row_flags[:m]).sum())
    for name in ("signed", "normalized"):
        so, sd = getattr(ro, name), getattr(rd, name)
        if so is None or sd is None:
            continue
        bo, bd = block(so, no, m), block(sd, nd, m)
        rows = np.arange(m)[:, None]
        cols = np.arange(m)[None, :]
        mask = (cols <= rows) & (rows >= 1)  # row r <-> size r+1, columns 0..r
        if name == "normalized":
            mask &= ((ro.row_flags[:m] & 2) != 0)[:, None]
        bad += _mism(bo, bd, mask.reshape(-1))
    return bad


def prefix(A: SoA, n: int, p: int, kind: str, m: int, device_res: HostResults, device_final: SoA | None) -> dict:
    """Full-run outputs for leading sizes <= m vs an oracle run on A[1..m,1..m]."""
    t0 = time.perf_counter()
    Am = block(A, n, m)
    r = oracle.OracleRank(m, p, kind, 0, 1, host_threads())
    r.load(Am)
    res_o = HostResults.alloc(m, r.ncomp, r.L, True)
    rc, done = r.run(True, True, 0, m, res_o)
    fin_o = Am.copy()
    r.fetch(fin_o)
    r.close()
    out = {"m": m, "oracle_steps": done,
           "trace_mismatches": _mism(_head(res_o.dets, done), _head(device_res.dets, done))
           + _mism(_head(res_o.pivots, done), _head(device_res.pivots, done)),
           "minors_rows": m - 1, "minors_mismatches": _minors_mism(res_o, device_res, m, n, m),
           "oracle_s": time.perf_counter() - t0}
    if device_final is not None:
        out["block_mismatches"] = _mism(fin_o, block(device_final, n, m))
    out["ok"] = (out["trace_mismatches"] == 0 and out["minors_mismatches"] == 0
                 and out.get("block_mismatches", 0) == 0)
    return out


def laplace_log2(A: SoA, n: int, p: int, res: HostResults, size: int) -> float:
    """log2 of |sum_k signed[size][k] a_{k,size} - det_size| / |det_size| at precision p, with
    a_{k,size} the ORIGINAL entries (elim.py:232-248); -inf when the sum is exact."""
    base = (size - 1) * n
    with mp.context(precision=p):
        acc = None
        for k in range(size):
            s = res.signed.get(base + k, p)
            a = A.get(k * n + (size - 1), p)
            acc = s * a if acc is None else acc + s * a
        det = res.dets.get(size - 1, p)
        num = abs(acc - det)
        if num == 0:
            return -math.inf
        return float(mp.log2(num / abs(det)))


def laplace(A: SoA, n: int, p: int, res: HostResults, sizes) -> dict:
    vals = {int(s): laplace_log2(A, n, p, res, int(s)) for s in sizes}
    return {"sizes": sorted(vals), "log2_residual": {str(k): (None if v == -math.inf else round(v, 1))
                                                     for k, v in sorted(vals.items())},
            "worst_log2": max((v for v in vals.values()), default=-math.inf)}
