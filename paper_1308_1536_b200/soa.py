"""Host side of the ds SoA scalar format (include/detseries_b200.h).

A real scalar x != 0 at precision p is (-1)^s * M * 2^(e - 32L) with M an
L-limb (32-bit, little-endian) integer whose MSB is set and whose low 32L-p
bits are zero; cls is the reference wire-format sign class (parexec.py:36:
0 = +, 1 = -, 2 = +0, 3 = -0).  Arrays are limb-plane major:
limbs[c, l, idx], exp[c, idx], cls[c, idx] with c the complex component.
This is the layout the device kernels read coalesced, and the layout the
C ABI takes from the caller.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import mp
from .mp import mpc, mpfr

CLS_POS, CLS_NEG, CLS_PZERO, CLS_NZERO = 0, 1, 2, 3


class paused_gc:
    """Cyclic garbage collection paused while millions of scalar objects are created
    (the boundary conversion of minors rows / the in-place buffer): the objects hold
    no reference cycles, and repeated full collections over a growing heap made the
    conversion ~4x slower.  Restores the previous state; nests."""

    def __enter__(self):
        import gc
        self._was = gc.isenabled()
        gc.disable()
        return self

    def __exit__(self, *exc):
        import gc
        if self._was:
            gc.enable()


class ds_soa(ctypes.Structure):
    _fields_ = [("limbs", ctypes.c_void_p), ("exp", ctypes.c_void_p), ("cls", ctypes.c_void_p),
                ("count", ctypes.c_int64)]


class SoA:
    """Numpy-backed ds SoA array of `count` scalars with `ncomp` components."""

    __slots__ = ("ncomp", "L", "count", "limbs", "exp", "cls")

    def __init__(self, ncomp: int, L: int, count: int, limbs=None, exp=None, cls=None, pinned=False):
        self.ncomp, self.L, self.count = int(ncomp), int(L), int(count)
        if limbs is None:
            if pinned:
                limbs = _pinned_empty((self.ncomp, self.L, self.count), np.uint32)
                limbs.fill(0)
            else:
                limbs = np.zeros((self.ncomp, self.L, self.count), dtype=np.uint32)
        if exp is None:
            if pinned:
                exp = _pinned_empty((self.ncomp, self.count), np.int32)
                exp.fill(0)
            else:
                exp = np.zeros((self.ncomp, self.count), dtype=np.int32)
        if cls is None:
            if pinned:
                cls = _pinned_empty((self.ncomp, self.count), np.uint8)
                cls.fill(CLS_PZERO)
            else:
                cls = np.full((self.ncomp, self.count), CLS_PZERO, dtype=np.uint8)
        self.limbs, self.exp, self.cls = limbs, exp, cls
        assert self.limbs.shape == (self.ncomp, self.L, self.count) and self.limbs.dtype == np.uint32
        assert self.limbs.flags.c_contiguous and self.exp.flags.c_contiguous and self.cls.flags.c_contiguous

    @classmethod
    def like(cls_, other: "SoA", count: int | None = None) -> "SoA":
        return cls_(other.ncomp, other.L, other.count if count is None else count)

    def copy(self) -> "SoA":
        return SoA(self.ncomp, self.L, self.count, self.limbs.copy(), self.exp.copy(), self.cls.copy())

    def c(self) -> ds_soa:
        """C view (pointers stay valid while self is alive)."""
        return ds_soa(self.limbs.ctypes.data, self.exp.ctypes.data, self.cls.ctypes.data, self.count)

    @property
    def nbytes(self) -> int:
        return self.limbs.nbytes + self.exp.nbytes + self.cls.nbytes

    # -- element access -------------------------------------------------
    def get(self, idx: int, prec: int):
        """Scalar object (mp.mpfr / mp.mpc) for element idx."""
        parts = [mp.from_limbs(self.limbs[c, :, idx].tobytes(), int(self.exp[c, idx]), int(self.cls[c, idx]), prec)
                 for c in range(self.ncomp)]
        return parts[0] if self.ncomp == 1 else mp.mpc_from_parts(parts[0], parts[1])

    def scalars(self, start: int, count: int, prec: int) -> list:
        """Scalar objects for the contiguous elements [start, start+count): the
        mpfr_t structs are filled by one native call (libds_hostgen.so,
        dsh_soa_to_mpfr) and wrapped, instead of one ctypes round trip per
        scalar -- the boundary conversion of whole minors rows."""
        if count <= 0:
            return []
        from .hostgen import _load
        lib = _load()
        n64 = (prec + 63) // 64
        pad = 2 * n64 - self.L
        parts = []
        for c in range(self.ncomp):
            # element-major limb pool, transposed from the planes natively and read in
            # place by the mpfr structs
            pool = np.empty((count, 2 * n64), dtype=np.uint32)
            planes = self.limbs[c]
            if planes.strides[1] != 4:
                planes = np.ascontiguousarray(planes)
            ex = np.ascontiguousarray(self.exp[c, start:start + count])
            cl = np.ascontiguousarray(self.cls[c, start:start + count])
            arr = (mp._MPFR_T * count)()
            if pad < 0 or lib.dsh_mpfr_structs_planes(arr, pool.ctypes.data, planes.ctypes.data + 4 * start,
                                                      planes.strides[0] // 4, self.L, ex.ctypes.data,
                                                      cl.ctypes.data, count, n64, prec) != 0:
                raise ValueError("SoA.scalars: precision %d does not hold %d limbs" % (prec, self.L))
            parts.append(mp.wrap_pooled(arr, pool, count))
        if self.ncomp == 1:
            return parts[0]
        return [mp.mpc_from_parts(a, b) for a, b in zip(parts[0], parts[1])]

    def set(self, idx: int, x, prec: int):
        comps = (x,) if self.ncomp == 1 else (x.real, x.imag)
        for c, v in enumerate(comps):
            raw, e, k = _real_limbs(v, prec, self.L)
            self.limbs[c, :, idx] = np.frombuffer(raw, dtype=np.uint32)
            self.exp[c, idx] = e
            self.cls[c, idx] = k

    def canonical(self, idx: int, prec: int):
        """canonical_bits of element idx straight from the limbs (scalars.py:129-145)."""
        parts = tuple(_canon_real(self.limbs[c, :, idx], int(self.exp[c, idx]), int(self.cls[c, idx]), prec, self.L)
                      for c in range(self.ncomp))
        return parts[0] if self.ncomp == 1 else ("c", parts[0], parts[1])

    def to_scalars(self, prec: int, indices=None) -> list:
        idxs = range(self.count) if indices is None else indices
        return [self.get(i, prec) for i in idxs]

    @classmethod
    def from_scalars(cls_, values, prec: int, kind: str) -> "SoA":
        ncomp = 2 if kind == "complex" else 1
        L = (prec + 31) // 32
        n = len(values)
        out = cls_(ncomp, L, n)
        raws = [bytearray() for _ in range(ncomp)]
        for i, x in enumerate(values):
            comps = (x,) if ncomp == 1 else (x.real, x.imag)
            for c, v in enumerate(comps):
                raw, e, k = _real_limbs(v, prec, L)
                raws[c] += raw
                out.exp[c, i] = e
                out.cls[c, i] = k
        for c in range(ncomp):
            if n:
                out.limbs[c] = np.frombuffer(bytes(raws[c]), dtype=np.uint32).reshape(n, L).T
        return out


def _real_limbs(v, prec: int, L: int):
    """(raw little-endian limb bytes, exp, cls) for a real scalar at `prec`."""
    if isinstance(v, mpfr):
        if v.precision != prec:
            with mp.context(precision=prec):
                v = mpfr(v)
        return mp.limbs_of(v)
    # foreign scalar (real gmpy2 or int/Fraction): go through the exact
    # mantissa/exponent pair
    with mp.context(precision=prec):
        w = mpfr(_foreign_to_mp(v, prec))
    return mp.limbs_of(w)


def _foreign_to_mp(v, prec):
    if hasattr(v, "as_mantissa_exp"):
        if v == 0:
            neg = str(v).startswith("-")
            return mpfr("-0") if neg else mpfr(0)
        m, e = v.as_mantissa_exp()
        return mp.mul_2exp(mpfr(int(m), max(64, abs(int(m)).bit_length())), int(e))
    return v


def _canon_real(limbs, exp, cls, prec, L):
    if cls == CLS_PZERO:
        return ("r", "+0")
    if cls == CLS_NZERO:
        return ("r", "-0")
    M = int.from_bytes(np.ascontiguousarray(limbs).tobytes(), "little")
    m = M >> (32 * L - prec)
    e = exp - prec
    if cls == CLS_NEG:
        m = -m
    tz = (m & -m).bit_length() - 1
    return ("r", m >> tz, e + tz)


_cudart = None


def _pinned_empty(shape, dtype):
    """Page-locked host array (for the timed e2e H2D/D2H copies); plain numpy
    when no CUDA runtime is available."""
    try:
        import torch
        if torch.cuda.is_available():
            count = int(np.prod(shape))
            t = torch.empty(count * np.dtype(dtype).itemsize, dtype=torch.uint8, pin_memory=True)
            arr = t.numpy().view(dtype).reshape(shape)
            _PINNED_KEEPALIVE[arr.ctypes.data] = t
            return arr
    except Exception:
        pass
    return np.empty(shape, dtype=dtype)


_PINNED_KEEPALIVE: dict = {}
