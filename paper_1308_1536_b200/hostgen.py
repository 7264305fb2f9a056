"""Fast host builders (libds_hostgen.so) that produce benchmark-size inputs
directly in the ds SoA format.

beta_matrix_soa reproduces genmat.beta_matrix (reference genmat.py:156-190,
Artless Eq. 9) bit for bit -- same MPFR/MPC operation sequence and working
precisions -- in multi-threaded C with Gamma(1/4 - i t/2) memoised per column.
This is input generation (the reference builds inputs through gmpy2 the same
way); the elimination itself never runs on the CPU.
"""

from __future__ import annotations

import ctypes
import os

from .soa import SoA, ds_soa

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libds_hostgen.so")
_lib = None


def _load():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise FileNotFoundError(f"{LIB_PATH} missing: run make -C paper_1308_1536_b200/csrc")
        L = ctypes.CDLL(LIB_PATH)
        L.dsh_beta_matrix.restype = ctypes.c_int
        L.dsh_beta_matrix.argtypes = [ctypes.c_int, ctypes.c_long, ctypes.POINTER(ctypes.c_char_p), ctypes.c_int,
                                      ctypes.c_int, ctypes.POINTER(ds_soa), ctypes.POINTER(ds_soa)]
        L.dsh_beta_matrix_cols.restype = ctypes.c_int
        L.dsh_beta_matrix_cols.argtypes = [ctypes.c_int, ctypes.c_long, ctypes.POINTER(ctypes.c_char_p), ctypes.c_int,
                                           ctypes.c_int, ctypes.POINTER(ds_soa), ctypes.POINTER(ds_soa), ctypes.c_int,
                                           ctypes.c_int, ctypes.c_int, ctypes.c_int]
        L.dsh_beta_gammas.restype = ctypes.c_int
        L.dsh_beta_gammas.argtypes = [ctypes.c_int, ctypes.c_long, ctypes.POINTER(ctypes.c_char_p), ctypes.c_int,
                                      ctypes.c_int, ctypes.POINTER(ds_soa)]
        L.dsh_power_matrix.restype = ctypes.c_int
        L.dsh_power_matrix.argtypes = [ctypes.c_int, ctypes.c_long, ctypes.POINTER(ctypes.c_char_p), ctypes.c_long,
                                       ctypes.c_char_p, ctypes.c_long, ctypes.c_int, ctypes.c_int,
                                       ctypes.POINTER(ds_soa), ctypes.c_int, ctypes.c_int]
        L.dsh_mpfr_structs.restype = ctypes.c_int
        L.dsh_mpfr_structs.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                       ctypes.c_int64, ctypes.c_int, ctypes.c_long]
        L.dsh_mpfr_structs_planes.restype = ctypes.c_int
        L.dsh_mpfr_structs_planes.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
                                              ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
                                              ctypes.c_int, ctypes.c_long]
        L.dsh_rowq_create.restype = ctypes.c_void_p
        L.dsh_rowq_create.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_long, ctypes.c_int]
        L.dsh_rowq_close.restype = None
        L.dsh_rowq_close.argtypes = [ctypes.c_void_p]
        L.dsh_rowq_destroy.restype = None
        L.dsh_rowq_destroy.argtypes = [ctypes.c_void_p]
        L.dsh_rowq_pop.restype = ctypes.POINTER(_RowBatch)
        L.dsh_rowq_pop.argtypes = [ctypes.c_void_p, ctypes.POINTER(ctypes.c_int)]
        L.dsh_rowbatch_free.restype = None
        L.dsh_rowbatch_free.argtypes = [ctypes.POINTER(_RowBatch)]
        L.dsh_soa_to_mpfr_pool.restype = ctypes.c_int
        L.dsh_soa_to_mpfr_pool.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.POINTER(ds_soa), ctypes.c_int,
                                           ctypes.c_int64, ctypes.c_int64, ctypes.c_int, ctypes.c_long]
        L.dsh_soa_to_mpfr.restype = ctypes.c_int
        L.dsh_soa_to_mpfr.argtypes = [ctypes.c_void_p, ctypes.POINTER(ds_soa), ctypes.c_int, ctypes.c_int64,
                                      ctypes.c_int64, ctypes.c_int, ctypes.c_long]
        _lib = L
    return _lib


def read_zero_tokens(path: str, count: int) -> list:
    """First `count` zero ordinates of a zeros file as decimal strings
    (the tokens load_zeros parses, genmat.py:50-60)."""
    out = []
    with open(path) as f:
        for line in f:
            tok = line.strip()
            if not tok or tok.startswith("#"):
                continue
            out.append(tok)
            if len(out) == count:
                break
    if len(out) < count:
        from .errors import InsufficientZeros
        raise InsufficientZeros(f"{path} holds {len(out)} zeros, need {count}")
    return out


def beta_gammas_soa(zeros_path: str, N: int, prec_bits: int, nthreads: int = 0, guard_bits: int = 64) -> SoA:
    """Gamma(1/4 - i gamma_j / 2) at prec + guard bits for j < N (complex SoA):
    the column-only, expensive part of beta_entry (genmat.py:171)."""
    lib = _load()
    toks = read_zero_tokens(zeros_path, N)
    arr = (ctypes.c_char_p * N)(*[t.encode() for t in toks])
    out = SoA(2, (prec_bits + guard_bits + 31) // 32, N)
    c = out.c()
    if lib.dsh_beta_gammas(N, prec_bits, arr, guard_bits, nthreads, ctypes.byref(c)) != 0:
        from .errors import GammaEvaluationFailed
        raise GammaEvaluationFailed("Spouge Gamma did not stabilise")
    return out


def beta_matrix_soa(zeros_path: str, N: int, prec_bits: int, nthreads: int = 0, guard_bits: int = 64,
                    pinned: bool = False, gammas: SoA | None = None) -> SoA:
    lib = _load()
    toks = read_zero_tokens(zeros_path, N)
    arr = (ctypes.c_char_p * N)(*[t.encode() for t in toks])
    out = SoA(1, (prec_bits + 31) // 32, N * N, pinned=pinned)
    c = out.c()
    g = None
    if gammas is not None:
        assert gammas.ncomp == 2 and gammas.L == (prec_bits + guard_bits + 31) // 32 and gammas.count >= N
        g = ctypes.byref(gammas.c())
    rc = lib.dsh_beta_matrix(N, prec_bits, arr, guard_bits, nthreads, ctypes.byref(c), g)
    if rc != 0:
        from .errors import GammaEvaluationFailed
        raise GammaEvaluationFailed("Spouge Gamma did not stabilise")
    return out


class BetaBuilder:
    """Incremental builder: fill column ranges of the N x N beta matrix (so a
    caller can time the first chunk and decide whether to continue)."""

    def __init__(self, zeros_path: str, N: int, prec_bits: int, gammas: SoA | None = None, nthreads: int = 0,
                 guard_bits: int = 64, pinned: bool = False, row0: int = 0, rstep: int = 1):
        self.lib = _load()
        self.N, self.p, self.guard, self.nthreads = N, prec_bits, guard_bits, nthreads
        toks = read_zero_tokens(zeros_path, N)
        self._arr = (ctypes.c_char_p * N)(*[t.encode() for t in toks])
        # a rank of a sharded run (rstep > 1) holds only its rows: count nloc * N, the
        # layout ds_load accepts for owned rows
        nloc = (N - row0 + rstep - 1) // rstep if rstep > 1 else N
        self.out = SoA(1, (prec_bits + 31) // 32, nloc * N, pinned=pinned)
        self._c = self.out.c()
        self._g = gammas
        self._gc = gammas.c() if gammas is not None else None
        self.done = 0
        self.row0, self.rstep = row0, rstep

    def fill(self, j1: int):
        j1 = min(j1, self.N)
        if j1 <= self.done:
            return
        g = ctypes.byref(self._gc) if self._gc is not None else None
        rc = self.lib.dsh_beta_matrix_cols(self.N, self.p, self._arr, self.guard, self.nthreads,
                                           ctypes.byref(self._c), g, self.done, j1, self.row0, self.rstep)
        if rc != 0:
            from .errors import GammaEvaluationFailed
            raise GammaEvaluationFailed("Spouge Gamma did not stabilise")
        self.done = j1


def power_matrix_soa(zeros_path: str, M: int, prec_bits: int, t: str = "25", zero_prec: int = 2048,
                     t_prec: int = 2048, guard_bits: int = 32, nthreads: int = 0, pinned: bool = False,
                     row0: int = 0, rstep: int = 1) -> SoA:
    """genmat.power_matrix(load_zeros(zeros_path, Precision(zero_prec), M), M, mpfr(t) at t_prec,
    Precision(prec_bits), guard_bits) -- the (2M+1) x (2M+1) complex Artless zero-power matrix
    (reference genmat.py:193-223) -- bit for bit, in multi-threaded C (csrc/hostgen.c
    dsh_power_matrix).  rstep > 1: only rows row0, row0 + rstep, ... (owned-rows layout)."""
    lib = _load()
    toks = read_zero_tokens(zeros_path, M)
    arr = (ctypes.c_char_p * max(M, 1))(*[t_.encode() for t_ in toks])
    N = 2 * M + 1
    nloc = (N - row0 + rstep - 1) // rstep if rstep > 1 else N
    out = SoA(2, (prec_bits + 31) // 32, nloc * N, pinned=pinned)
    c = out.c()
    rc = lib.dsh_power_matrix(M, prec_bits, arr, zero_prec, str(t).encode(), t_prec, guard_bits, nthreads,
                              ctypes.byref(c), row0, rstep)
    if rc != 0:
        raise RuntimeError("power matrix builder failed")
    return out


# -- native consumer of the minors stream (csrc/hoststream.c) ---------------------------
class _RowBatch(ctypes.Structure):
    _fields_ = [("g0", ctypes.c_int32), ("stride", ctypes.c_int32), ("nrows", ctypes.c_int32),
                ("ncomp", ctypes.c_int32), ("m", ctypes.POINTER(ctypes.c_int32)),
                ("flags", ctypes.POINTER(ctypes.c_uint8)), ("off", ctypes.POINTER(ctypes.c_int64)),
                ("sg", ctypes.c_void_p * 2), ("nm", ctypes.c_void_p * 2), ("nel", ctypes.c_int64)]


class _BatchOwner:
    """Keeps one native batch (structs + limb pool) alive while any scalar wraps it."""
    __slots__ = ("ptr", "free")

    def __init__(self, ptr, free):
        self.ptr, self.free = ptr, free

    def __del__(self):
        self.free(self.ptr)


class RowQueue:
    """Minors-stream consumer whose callback (dsh_rowq_cb) runs natively on the thread
    that drives ds_run: each delivered batch becomes ready mpfr structs there, and
    pop_rows() on the caller's thread (GIL released while it waits) only wraps them
    in scalar objects.  Rows come back as (m, signed, normalized | None) in delivery
    (= increasing size) order."""

    def __init__(self, n: int, ncomp: int, L: int, prec: int, nthreads: int = 0):
        self.lib = _load()
        self.prec = prec
        self.q = self.lib.dsh_rowq_create(n, ncomp, L, prec, nthreads)
        if not self.q:
            raise ValueError("dsh_rowq_create: invalid shape")
        self.cb_ptr = ctypes.cast(self.lib.dsh_rowq_cb, ctypes.c_void_p).value

    def close(self):
        """Producer side done: pop_rows() returns None once drained."""
        self.lib.dsh_rowq_close(self.q)

    def pop_rows(self):
        """The next batch's rows, or None when the queue is closed and drained."""
        from . import mp
        failed = ctypes.c_int(0)
        bp = self.lib.dsh_rowq_pop(self.q, ctypes.byref(failed))
        if not bp:
            if failed.value:
                raise MemoryError("host memory for a streamed minors batch could not be allocated")
            return None
        b = bp.contents
        owner = _BatchOwner(bp, self.lib.dsh_rowbatch_free)
        T = mp._MPFR_T
        sz = ctypes.sizeof(T)
        out = []
        for r in range(b.nrows):
            m = b.m[r]
            if not m:
                continue
            off = b.off[r] * sz
            sg = [mp.wrap_pooled((T * m).from_address(b.sg[c] + off), owner, m) for c in range(b.ncomp)]
            nm = ([mp.wrap_pooled((T * m).from_address(b.nm[c] + off), owner, m) for c in range(b.ncomp)]
                  if b.flags[r] & 2 else None)
            if b.ncomp == 2:
                sg = [mp.mpc_from_parts(x, y) for x, y in zip(*sg)]
                nm = [mp.mpc_from_parts(x, y) for x, y in zip(*nm)] if nm is not None else None
            else:
                sg = sg[0]
                nm = nm[0] if nm is not None else None
            out.append((m, sg, nm))
        return out

    def __del__(self):
        q, self.q = getattr(self, "q", None), None
        if q:
            self.lib.dsh_rowq_destroy(q)
