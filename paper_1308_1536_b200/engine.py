"""Device elimination context: a thin Python owner of one `ds_ctx`
(libdetseries_b200.so) holding this rank's row-cyclic shard in HBM.

world == 1 runs the whole step loop natively (`run`).  world > 1 exposes
the per-step building blocks (`stage`, `step`) and the broadcast buffer so a
driver can broadcast each pivot row from its owner (parexec.py:300-317
semantics) -- see parexec.py of this package.
"""

from __future__ import annotations

import ctypes
import threading
from dataclasses import dataclass

import numpy as np

from . import _native
from ._native import DS_INVALID, DS_OK, DS_OOM, DS_OVERFLOW, DS_ZERO_PIVOT, ds_results
from .errors import DeviceUnavailable, WorkerFailure
from .soa import SoA


@dataclass
class HostResults:
    """Host copies of one run's outputs, in the ds SoA layout."""

    pivots: SoA
    dets: SoA
    signed: SoA | None
    normalized: SoA | None
    row_flags: np.ndarray

    @classmethod
    def alloc(cls, n: int, ncomp: int, L: int, minors: bool, pinned: bool = False) -> "HostResults":
        return cls(SoA(ncomp, L, n, pinned=pinned), SoA(ncomp, L, n, pinned=pinned),
                   SoA(ncomp, L, n * n, pinned=pinned) if minors else None,
                   SoA(ncomp, L, n * n, pinned=pinned) if minors else None,
                   np.zeros(n, dtype=np.uint8))

    def c(self) -> ds_results:
        z = _native.ds_soa(0, 0, 0, 0)
        r = ds_results()
        r.pivots = self.pivots.c()
        r.dets = self.dets.c()
        r.signed_minors = self.signed.c() if self.signed is not None else z
        r.normalized = self.normalized.c() if self.normalized is not None else z
        r.row_flags = self.row_flags.ctypes.data
        return r


def _check(rc: int, ctx, what: str, rank: int = 0):
    if rc == DS_OK or rc == DS_ZERO_PIVOT:
        return
    msg = _native.last_error(ctx)
    if rc == DS_OOM:
        raise MemoryError(f"{what}: device allocation failed: {msg}")
    if rc == DS_INVALID:
        raise ValueError(f"{what}: invalid arguments {msg}")
    if rc == DS_OVERFLOW:
        raise OverflowError(f"{what}: exponent left MPFR's default range ({msg})")
    raise WorkerFailure(rank, f"{what} failed with code {rc}: {msg}")


_closing: list = []  # threads releasing contexts in the background (DeviceElimination.close_async)
_closing_lock = threading.Lock()


def wait_released():
    """Join every background context release (its HBM is free afterwards)."""
    with _closing_lock:
        threads = list(_closing)
        _closing.clear()
    for t in threads:
        t.join()


class DeviceElimination:
    """One rank's device context (ds_create .. ds_destroy)."""

    def __init__(self, n: int, prec_bits: int, kind: str, device: int = 0, rank: int = 0, world: int = 1,
                 block: tuple | None = None):
        """block=(row0, nrows): a row-block context of the panel-paged executor (ds_create_block)."""
        self.lib = _native.lib()
        wait_released()  # a context still being released holds its HBM
        self.n, self.prec_bits, self.kind = n, prec_bits, kind
        self.ncomp = 2 if kind == "complex" else 1
        self.L = (prec_bits + 31) // 32
        self.device, self.rank, self.world = device, rank, world
        self.block = block
        ctx = ctypes.c_void_p()
        kcode = _native.DS_KIND_COMPLEX if kind == "complex" else _native.DS_KIND_REAL
        if block is None:
            rc = self.lib.ds_create(ctypes.byref(ctx), n, prec_bits, kcode, device, rank, world)
        else:
            rc = self.lib.ds_create_block(ctypes.byref(ctx), n, prec_bits, kcode, device, int(block[0]),
                                          int(block[1]))
        if rc != DS_OK:
            _check(rc, None, "ds_create", rank)
        self.ctx = ctx

    def pivot_load(self, step: int, row: SoA):
        """Final pivot row `step` (host SoA, count n) into the pivot buffer (ds_pivot_load)."""
        s = row.c()
        _check(self.lib.ds_pivot_load(self.ctx, int(step), ctypes.byref(s)), self.ctx, "ds_pivot_load", self.rank)

    def close(self):
        if getattr(self, "ctx", None):
            self.lib.ds_destroy(self.ctx)
            self.ctx = None

    def close_async(self):
        """Release the context on a background thread: ds_destroy frees gigabytes of
        device and pinned memory (10-800 ms) that the caller need not wait for.  The
        next context creation (and interpreter exit: the thread is not a daemon) waits
        for it, so peak memory is as with close()."""
        ctx = getattr(self, "ctx", None)
        if not ctx:
            return
        self.ctx = None
        t = threading.Thread(target=self.lib.ds_destroy, args=(ctx,), name="ds_destroy")
        with _closing_lock:
            _closing.append(t)
        t.start()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # -- data movement ---------------------------------------------------
    def load(self, matrix: SoA):
        s = matrix.c()
        _check(self.lib.ds_load(self.ctx, ctypes.byref(s)), self.ctx, "ds_load", self.rank)

    def fetch(self, matrix: SoA):
        s = matrix.c()
        _check(self.lib.ds_fetch(self.ctx, ctypes.byref(s)), self.ctx, "ds_fetch", self.rank)

    def generate(self, seed: int, family: str = "random_uniform"):
        """Fill this rank's rows on the device (ds_generate): the counter-based twin of
        genmat.synth_matrix(family, n, seed) -- see synth.counter_uniform_soa."""
        code = {"random_uniform": 0}[family]
        _check(self.lib.ds_generate(self.ctx, code, int(seed) & (2 ** 64 - 1)), self.ctx, "ds_generate", self.rank)

    def update_rows(self, matrix: SoA):
        """Rows back into HBM without resetting the run (ds_update_rows)."""
        s = matrix.c()
        _check(self.lib.ds_update_rows(self.ctx, ctypes.byref(s)), self.ctx, "ds_update_rows", self.rank)

    def set_det(self, det: SoA):
        s = det.c()
        _check(self.lib.ds_set_det(self.ctx, ctypes.byref(s)), self.ctx, "ds_set_det", self.rank)

    # -- serial engine -----------------------------------------------------
    def run(self, collect_minors: bool, series: bool, start: int, stop: int, res: HostResults | None):
        """Steps [start, stop) on the device; returns (rc, steps_done).  res=None leaves
        the outputs in HBM (fetch them later with results())."""
        done = ctypes.c_int(0)
        rp = ctypes.byref(res.c()) if res is not None else None
        rc = self.lib.ds_run(self.ctx, int(collect_minors), int(series), start, stop, rp, ctypes.byref(done))
        _check(rc, self.ctx, "ds_run", self.rank)
        self.raise_stream_error()
        return rc, done.value

    def set_pivot_mode(self, mode: str):
        """pivot_mode of elim.eliminate (elim.py:184-208): "none" or "partial"."""
        code = {"none": 0, "partial": 1}[mode]
        _check(self.lib.ds_set_pivot_mode(self.ctx, code), self.ctx, "ds_set_pivot_mode", self.rank)

    def swaps(self, upto: int) -> list[bool]:
        """Per-step row-swap flags of a partial-pivoting run, steps [0, upto)."""
        buf = (ctypes.c_uint8 * max(upto, 1))()
        _check(self.lib.ds_swaps_fetch(self.ctx, upto, buf), self.ctx, "ds_swaps_fetch", self.rank)
        return [bool(buf[i]) for i in range(upto)]

    # -- sharded building blocks ---------------------------------------------
    def pivot_buffer(self):
        p = ctypes.c_void_p()
        nbytes = ctypes.c_size_t()
        _check(self.lib.ds_pivot_buffer(self.ctx, ctypes.byref(p), ctypes.byref(nbytes)), self.ctx,
               "ds_pivot_buffer", self.rank)
        return p.value, nbytes.value

    def stage(self, i: int):
        _check(self.lib.ds_pivot_stage(self.ctx, i), self.ctx, "ds_pivot_stage", self.rank)

    def step(self, i: int, collect_minors: bool, series: bool):
        _check(self.lib.ds_step(self.ctx, i, int(collect_minors), int(series)), self.ctx, "ds_step", self.rank)

    def status(self) -> int:
        f = ctypes.c_int(-1)
        _check(self.lib.ds_status(self.ctx, ctypes.byref(f)), self.ctx, "ds_status", self.rank)
        return f.value

    def results(self, upto: int, res: HostResults):
        r = res.c()
        _check(self.lib.ds_results_fetch(self.ctx, upto, ctypes.byref(r)), self.ctx, "ds_results_fetch",
               self.rank)

    def results_range(self, t0: int, t1: int, m0: int, m1: int, res: HostResults):
        """Trace entries [t0, t1) and minors rows of sizes [m0, m1) (ds_results_fetch_range)."""
        r = res.c()
        _check(self.lib.ds_results_fetch_range(self.ctx, int(t0), int(t1), int(m0), int(m1), ctypes.byref(r)),
               self.ctx, "ds_results_fetch_range", self.rank)

    # -- streaming of minors rows (ds_stream_minors / ds_stream_flush) ------------
    _ROWS_CB = ctypes.CFUNCTYPE(None, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.POINTER(_native.ds_soa),
                                ctypes.POINTER(_native.ds_soa), ctypes.POINTER(ctypes.c_uint8), ctypes.c_void_p)

    def stream_minors(self, batch_steps: int, callback):
        """Stream the minors rows off the device as they finalise (only a ring of rows
        stays in HBM).  callback(g0, stride, nrows, signed, normalized, flags) gets SoA
        VIEWS of pinned staging memory (valid during the call only): row r, leading size
        m = g0 + r*stride + 1, holds its m entries at [r*n, r*n + m).  batch_steps <= 0 or
        callback None turns streaming off."""
        if batch_steps <= 0 or callback is None:
            _check(self.lib.ds_stream_minors(self.ctx, 0, None, None), self.ctx, "ds_stream_minors", self.rank)
            self._stream_cb = None
            return
        nc, L = self.ncomp, self.L

        def view(sp):
            s = sp.contents
            cnt = int(s.count)
            limbs = np.ctypeslib.as_array(ctypes.cast(s.limbs, ctypes.POINTER(ctypes.c_uint32)), (nc, L, cnt))
            ex = np.ctypeslib.as_array(ctypes.cast(s.exp, ctypes.POINTER(ctypes.c_int32)), (nc, cnt))
            cl = np.ctypeslib.as_array(ctypes.cast(s.cls, ctypes.POINTER(ctypes.c_uint8)), (nc, cnt))
            return SoA(nc, L, cnt, limbs, ex, cl)

        def trampoline(g0, stride, nrows, sp, np_, fp, user):
            flags = np.ctypeslib.as_array(fp, (nrows,)) if nrows else np.zeros(0, np.uint8)
            try:
                callback(g0, stride, nrows, view(sp), view(np_), flags)
            except BaseException as exc:  # cannot propagate through C: keep it for the caller
                self._stream_exc = exc

        self._stream_exc = None
        self._stream_cb = self._ROWS_CB(trampoline)
        _check(self.lib.ds_stream_minors(self.ctx, int(batch_steps), self._stream_cb, None), self.ctx,
               "ds_stream_minors", self.rank)

    def stream_minors_native(self, batch_steps: int, cb_ptr: int, user_ptr: int):
        """Stream the minors rows to a native ds_rows_cb (e.g. hostgen.RowQueue, which
        builds the scalar structs off the interpreter)."""
        self._stream_cb = None
        self._stream_exc = None
        _check(self.lib.ds_stream_minors(self.ctx, int(batch_steps), ctypes.c_void_p(cb_ptr),
                                         ctypes.c_void_p(user_ptr)), self.ctx, "ds_stream_minors", self.rank)

    def stream_flush(self, upto_step: int, final: bool = False):
        _check(self.lib.ds_stream_flush(self.ctx, int(upto_step), int(final)), self.ctx, "ds_stream_flush",
               self.rank)
        self.raise_stream_error()

    def raise_stream_error(self):
        exc = getattr(self, "_stream_exc", None)
        if exc is not None:
            self._stream_exc = None
            raise exc

    def snapshot(self, save: bool):
        """save=True: keep a device copy of this rank's rows; save=False:
        restore it and reset the run state (resident re-runs)."""
        _check(self.lib.ds_snapshot(self.ctx, int(save)), self.ctx, "ds_snapshot", self.rank)

    def run_resident(self, collect_minors: bool, series: bool, start: int, stop: int):
        """Steps [start, stop) with results left in HBM (no D2H)."""
        done = ctypes.c_int(0)
        rc = self.lib.ds_run(self.ctx, int(collect_minors), int(series), start, stop, None, ctypes.byref(done))
        _check(rc, self.ctx, "ds_run", self.rank)
        return rc, done.value

    def profile(self, enable: bool):
        self.lib.ds_profile(self.ctx, int(enable))

    def profile_read(self):
        """(update kernel ms, launches, schoolbook limb-MACs) since the last read."""
        ms, n, w = ctypes.c_double(), ctypes.c_int64(), ctypes.c_double()
        _check(self.lib.ds_profile_read(self.ctx, ctypes.byref(ms), ctypes.byref(n), ctypes.byref(w)), self.ctx,
               "ds_profile_read", self.rank)
        return ms.value, n.value, w.value

    def counters(self) -> dict:
        """Internal engine counters (ds_counters): tensor-core fallback elements, active update engine."""
        out = (ctypes.c_int64 * 6)()
        _check(self.lib.ds_counters(self.ctx, out, 6), self.ctx, "ds_counters", self.rank)
        return {"tc_fallback_elements": int(out[0]), "tc_engine": bool(out[1]), "dfma_engine": bool(out[2]),
                "direct_mispredictions": int(out[3]), "h2d_bytes": int(out[4]), "d2h_bytes": int(out[5])}

    # -- multi-rank lookahead (ds_lookahead_*) ------------------------------
    def lookahead_enable(self, limit: int):
        _check(self.lib.ds_lookahead_enable(self.ctx, int(limit)), self.ctx, "ds_lookahead_enable", self.rank)

    def lookahead_stream(self) -> int:
        p = ctypes.c_void_p()
        _check(self.lib.ds_lookahead_stream(self.ctx, ctypes.byref(p)), self.ctx, "ds_lookahead_stream", self.rank)
        return p.value or 0

    def lookahead_pivot(self, i1: int, buf_ptr: int):
        _check(self.lib.ds_lookahead_pivot(self.ctx, int(i1), ctypes.c_void_p(buf_ptr)), self.ctx,
               "ds_lookahead_pivot", self.rank)

    def lookahead_mult(self, i1: int, buf_ptr: int):
        _check(self.lib.ds_lookahead_mult(self.ctx, int(i1), ctypes.c_void_p(buf_ptr)), self.ctx,
               "ds_lookahead_mult", self.rank)

    def stream(self) -> int:
        return self.lib.ds_stream(self.ctx) or 0

    def launches(self) -> int:
        return int(self.lib.ds_launch_count(self.ctx))


def scalar_op(op: str, kind: str, prec_bits: int, a: SoA, b: SoA, device: int = 0) -> SoA:
    """Element-wise correctly rounded op on the device (conformance surface)."""
    lib = _native.lib()
    code = {"mul": 0, "sub": 1, "div": 2, "add": 3}[op]
    out = SoA.like(a)
    sa, sb, so = a.c(), b.c(), out.c()
    rc = lib.ds_scalar_op(code, _native.DS_KIND_COMPLEX if kind == "complex" else _native.DS_KIND_REAL,
                          prec_bits, device, ctypes.byref(sa), ctypes.byref(sb), ctypes.byref(so))
    if rc not in (DS_OK,):
        _check(rc, None, "ds_scalar_op")
    return out


__all__ = ["DeviceElimination", "HostResults", "scalar_op", "DeviceUnavailable"]
