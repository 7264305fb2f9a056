"""ctypes binding of the CPU oracle (oracle/libds_oracle.so).

TEST INFRASTRUCTURE: only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / reference arm load this module, as the checker and the timed
CPU baseline.  The oracle is a C restatement of the reference hot path
(elim.py:37-229, parexec.py:244-333) over the system MPFR/MPC -- the libraries
gmpy2 wraps -- pinned against the unmodified reference (run through
oracle/gmpy2_shim) by tests/golden/.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libds_oracle.so")

DS_OK, DS_ZERO_PIVOT = 0, 1


class ds_soa(ctypes.Structure):
    _fields_ = [("limbs", ctypes.c_void_p), ("exp", ctypes.c_void_p), ("cls", ctypes.c_void_p),
                ("count", ctypes.c_int64)]


class ds_results(ctypes.Structure):
    _fields_ = [("pivots", ds_soa), ("dets", ds_soa), ("signed_minors", ds_soa), ("normalized", ds_soa),
                ("row_flags", ctypes.c_void_p)]


def build():
    """Compile libds_oracle.so (gcc, system runtime libs)."""
    subprocess.run(["make", "-C", HERE], check=True, capture_output=True)


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = ctypes.CDLL(LIB_PATH)
        VP, I, L64 = ctypes.c_void_p, ctypes.c_int, ctypes.c_long
        S = ctypes.POINTER(ds_soa)
        L.dso_create.restype = VP
        L.dso_create.argtypes = [I, L64, I, I, I, I]
        L.dso_destroy.argtypes = [VP]
        L.dso_load.argtypes = [VP, S]
        L.dso_fetch.argtypes = [VP, S]
        L.dso_pivot_buffer.restype = VP
        L.dso_pivot_buffer.argtypes = [VP, ctypes.POINTER(ctypes.c_size_t)]
        L.dso_pivot_stage.argtypes = [VP, I]
        L.dso_step.argtypes = [VP, I, I, I]
        L.dso_set_det.argtypes = [VP, S]
        L.dso_status.argtypes = [VP, ctypes.POINTER(I)]
        L.dso_results_fetch.argtypes = [VP, I, ctypes.POINTER(ds_results)]
        L.dso_run.argtypes = [VP, I, I, I, I, ctypes.POINTER(I)]
        L.dso_scalar_op.argtypes = [I, I, L64, S, S, S]
        L.dso_apply_pivot_rows.argtypes = [I, L64, I, I, I, S, S, I, I]
        L.dso_time_apply_pivot_rows.restype = ctypes.c_double
        L.dso_time_apply_pivot_rows.argtypes = [I, L64, I, I, I, S, S, I, I]
        L.dso_version.restype = ctypes.c_char_p
        _lib = L
    return _lib


def _soa_c(s) -> ds_soa:
    return ds_soa(s.limbs.ctypes.data, s.exp.ctypes.data, s.cls.ctypes.data, s.count)


class OracleRank:
    """One rank of the oracle's row-cyclic executor; same method names as
    paper_1308_1536_b200.engine.DeviceElimination (stage / step / status /
    results / fetch / load / set_det)."""

    def __init__(self, n: int, prec_bits: int, kind: str, rank: int = 0, world: int = 1, nthreads: int = 0):
        self.lib = lib()
        self.n, self.prec_bits, self.kind, self.rank, self.world = n, prec_bits, kind, rank, world
        self.ncomp = 2 if kind == "complex" else 1
        self.L = (prec_bits + 31) // 32
        self.ctx = self.lib.dso_create(n, prec_bits, 1 if kind == "complex" else 0, rank, world, nthreads)
        if not self.ctx:
            raise ValueError("dso_create failed")

    def close(self):
        if self.ctx:
            self.lib.dso_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def load(self, soa):
        s = _soa_c(soa)
        self.lib.dso_load(self.ctx, ctypes.byref(s))

    def fetch(self, soa):
        s = _soa_c(soa)
        self.lib.dso_fetch(self.ctx, ctypes.byref(s))

    def set_det(self, det):
        s = _soa_c(det)
        self.lib.dso_set_det(self.ctx, ctypes.byref(s))

    def pivot_array(self) -> np.ndarray:
        """The pivot buffer as a writable numpy uint8 array (host memory)."""
        nbytes = ctypes.c_size_t()
        ptr = self.lib.dso_pivot_buffer(self.ctx, ctypes.byref(nbytes))
        buf = (ctypes.c_uint8 * nbytes.value).from_address(ptr)
        return np.frombuffer(buf, dtype=np.uint8)

    def stage(self, i: int):
        self.lib.dso_pivot_stage(self.ctx, i)

    def step(self, i: int, collect_minors: bool, series: bool):
        self.lib.dso_step(self.ctx, i, int(collect_minors), int(series))

    def status(self) -> int:
        f = ctypes.c_int(-1)
        self.lib.dso_status(self.ctx, ctypes.byref(f))
        return f.value

    def results(self, upto: int, res):
        r = ds_results()
        z = ds_soa(0, 0, 0, 0)
        r.pivots = _soa_c(res.pivots)
        r.dets = _soa_c(res.dets)
        r.signed_minors = _soa_c(res.signed) if res.signed is not None else z
        r.normalized = _soa_c(res.normalized) if res.normalized is not None else z
        r.row_flags = res.row_flags.ctypes.data
        self.lib.dso_results_fetch(self.ctx, upto, ctypes.byref(r))

    def run(self, collect_minors: bool, series: bool, start: int, stop: int, res=None):
        done = ctypes.c_int(0)
        rc = self.lib.dso_run(self.ctx, int(collect_minors), int(series), start, stop, ctypes.byref(done))
        if res is not None:
            self.results(done.value, res)
        return rc, done.value


def eliminate_soa(matrix, n: int, prec_bits: int, kind: str, collect_minors=True, series=True, nthreads=0):
    """Serial oracle run on a SoA matrix (copied); returns (rc, done, results,
    final matrix SoA).  `matrix` is a paper_1308_1536_b200.soa.SoA (or any
    object with limbs/exp/cls/count numpy fields)."""
    from paper_1308_1536_b200.engine import HostResults
    r = OracleRank(n, prec_bits, kind, 0, 1, nthreads)
    r.load(matrix)
    res = HostResults.alloc(n, r.ncomp, r.L, collect_minors)
    rc, done = r.run(collect_minors, series, 0, n, res)
    final = matrix.copy()
    r.fetch(final)
    r.close()
    return rc, done, res, final


def scalar_op(op: str, kind: str, prec_bits: int, a, b):
    code = {"mul": 0, "sub": 1, "div": 2, "add": 3}[op]
    out = a.copy()
    sa, sb, so = _soa_c(a), _soa_c(b), _soa_c(out)
    lib().dso_scalar_op(code, 1 if kind == "complex" else 0, prec_bits, ctypes.byref(sa), ctypes.byref(sb),
                        ctypes.byref(so))
    return out


def time_apply_pivot_rows(n: int, prec_bits: int, kind: str, i: int, prow, rows, nrows: int, nthreads: int,
                          collect_minors: bool = True) -> float:
    """Seconds for the reference hot loop (elim.py:37-53) on `nrows` rows."""
    sp, sr = _soa_c(prow), _soa_c(rows)
    return lib().dso_time_apply_pivot_rows(n, prec_bits, 1 if kind == "complex" else 0, i, int(collect_minors),
                                           ctypes.byref(sp), ctypes.byref(sr), nrows, nthreads)
