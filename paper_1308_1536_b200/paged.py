"""Out-of-core elimination by row panels (the role of the reference's
blockpager.py: paged_eliminate, schedule genmat/blockpager.py:224-241 and
505-529) for matrices larger than the device's memory.

The reference pages B x B blocks through a right-looking schedule over a
disk-resident block grid.  On the B200 the natural unit is a PANEL of
consecutive full-width rows [r0, r1) held in HBM (ds_create_block): the
panel is brought up to date left-looking -- for i < r0 the final pivot row i
is loaded from the host store (ds_pivot_load) and applied to every panel row
(exactly the update elim.py:216-218 applies to those rows in core, same op
order per element), then steps r0 <= i < r1 run inside the panel with their
pivot staged from it.  The finished rows go back to the host store, which may
be pinned RAM or a disk-backed numpy memmap (NVMe), and the next panel
starts.  Every element sees the in-core op sequence, so pivots, det_series,
minors and the final L\\U state are bit-identical to eliminate(); pivot rows
cost one host->device copy per (panel, earlier step).

Minors rows of size m are emitted by the panel holding row m-1 (elim.py:
220-226) and handed to `sink` as each panel finishes, in increasing m.
"""

from __future__ import annotations

import numpy as np

from .engine import DeviceElimination, HostResults
from .soa import SoA


def _rows(s: SoA, n: int, r0: int, r1: int) -> SoA:
    """View (copy) of rows [r0, r1) of an n x n SoA as a compact (r1-r0)*n SoA."""
    nc, L = s.ncomp, s.L
    sl = slice(r0 * n, r1 * n)
    return SoA(nc, L, (r1 - r0) * n, np.ascontiguousarray(s.limbs[:, :, sl]), np.ascontiguousarray(s.exp[:, sl]),
               np.ascontiguousarray(s.cls[:, sl]))


def _store_rows(dst: SoA, n: int, r0: int, src: SoA):
    nc = dst.ncomp
    cnt = src.count
    dst.limbs[:, :, r0 * n:r0 * n + cnt] = src.limbs
    dst.exp[:, r0 * n:r0 * n + cnt] = src.exp
    dst.cls[:, r0 * n:r0 * n + cnt] = src.cls
    del nc


def paged_eliminate_soa(A: SoA, n: int, prec_bits: int, kind: str, panel_rows: int, collect_minors: bool = True,
                        series: bool = True, device: int = 0, sink=None):
    """Eliminate the n x n matrix in host store A (ds SoA, updated in place to L\\U) panel by panel.

    Returns (HostResults with pivots/dets [0, done) and -- when sink is None -- every
    minors row, done).  sink(m, flags, signed SoA row, normalized SoA row or None) is
    called per emitted row instead of collecting them.  done < n: exact zero pivot at
    step `done` (the caller raises ZeroPivot, elim.py:209-212)."""
    if panel_rows < 1:
        raise ValueError("panel_rows must be >= 1")
    nc = 2 if kind == "complex" else 1
    L = (prec_bits + 31) // 32
    res = HostResults.alloc(n, nc, L, collect_minors and sink is None)
    done = n  # steps completed: the zero-pivot step when one is found
    for r0 in range(0, n, panel_rows):
        r1 = min(n, r0 + panel_rows)
        with DeviceElimination(n, prec_bits, kind, device, block=(r0, r1 - r0)) as e:
            e.load(_rows(A, n, r0, r1))
            failed = -1
            # after a zero pivot at step `done`, later panels still receive steps < done:
            # the reference leaves every row updated through the completed steps
            for i in range(min(r1, done)):
                if i < r0:
                    e.pivot_load(i, _rows(A, n, i, i + 1))
                else:
                    e.stage(i)
                e.step(i, collect_minors, series)
                if i >= r0 and (i - r0) % 64 == 63:  # surface a zero pivot without a sync per step
                    failed = e.status()
                    if failed >= 0:
                        break
            if failed < 0:
                failed = e.status()
            fin = SoA(nc, L, (r1 - r0) * n)
            e.fetch(fin)
            _store_rows(A, n, r0, fin)
            part = HostResults(SoA(nc, L, n), SoA(nc, L, n), SoA(nc, L, (r1 - r0) * n) if collect_minors else None,
                               SoA(nc, L, (r1 - r0) * n) if collect_minors else None, np.zeros(n, np.uint8))
            upto = failed if failed >= 0 else min(r1, done)
            e.results(upto, part)
        # trace entries of this panel's steps
        lo, hi = r0, max(r0, upto)
        if hi > lo:
            for dst, srcv in ((res.pivots, part.pivots), (res.dets, part.dets)):
                dst.limbs[:, :, lo:hi] = srcv.limbs[:, :, lo:hi]
                dst.exp[:, lo:hi] = srcv.exp[:, lo:hi]
                dst.cls[:, lo:hi] = srcv.cls[:, lo:hi]
        if collect_minors:
            for g in range(max(r0, 1), r1):  # row g holds the minors of size g+1
                fl = int(part.row_flags[g])
                if not fl & 1:
                    continue
                m = g + 1
                jl = g - r0
                sl = slice(jl * n, jl * n + m)
                sg = SoA(nc, L, m, np.ascontiguousarray(part.signed.limbs[:, :, sl]),
                         np.ascontiguousarray(part.signed.exp[:, sl]), np.ascontiguousarray(part.signed.cls[:, sl]))
                nm = None
                if fl & 2:
                    nm = SoA(nc, L, m, np.ascontiguousarray(part.normalized.limbs[:, :, sl]),
                             np.ascontiguousarray(part.normalized.exp[:, sl]),
                             np.ascontiguousarray(part.normalized.cls[:, sl]))
                if sink is not None:
                    sink(m, fl, sg, nm)
                else:
                    res.row_flags[g] = fl
                    res.signed.limbs[:, :, g * n:g * n + m] = sg.limbs
                    res.signed.exp[:, g * n:g * n + m] = sg.exp
                    res.signed.cls[:, g * n:g * n + m] = sg.cls
                    if nm is not None:
                        res.normalized.limbs[:, :, g * n:g * n + m] = nm.limbs
                        res.normalized.exp[:, g * n:g * n + m] = nm.exp
                        res.normalized.cls[:, g * n:g * n + m] = nm.cls
        if failed >= 0:
            done = failed
    return res, done


def paged_eliminate(A, panel_rows: int, collect_minors: bool = True, series: bool = True, sink=None,
                    device: int = 0):
    """Drop-in shaped like elim.eliminate for a MatrixBuffer too large for the device:
    returns (EliminationTrace, MinorSeries | None), A updated in place, ZeroPivot on an
    exactly singular leading block -- computed panel by panel (paged_eliminate_soa)."""
    from .elim import EliminationTrace, MinorRow, MinorSeries
    from .errors import ZeroPivot
    n, p = A.n, A.prec.bits
    soa = A.to_soa()
    out = MinorSeries(A.prec) if collect_minors else None
    emit = sink if sink is not None else (out.add if out is not None else None)

    def row_sink(m, fl, sg, nm):
        emit(MinorRow(m, sg.scalars(0, m, p), nm.scalars(0, m, p) if nm is not None else None))

    res, done = paged_eliminate_soa(soa, n, p, A.kind, panel_rows, collect_minors, series, device,
                                    row_sink if collect_minors else None)
    trace = EliminationTrace(n=n, prec=A.prec)
    trace.pivots = res.pivots.scalars(0, done, p)
    trace.det_series = res.dets.scalars(0, done, p)
    trace.step = done
    A._set_lazy(soa)
    if done < n:
        raise ZeroPivot(done + 1, trace=trace, series=out)
    return trace, out
