"""Result files of the reference CLI (cli.py:218-232), two ways.

* ``write_dets`` / ``write_minors``: the CLI's loops over result objects
  (EliminationTrace, MinorSeries) with ``format_scalar`` -- same text as
  ``_write_dets`` / ``_write_minors``.
* ``write_results``: the same files straight from a run's ``HostResults``
  (ds SoA), formatted and written by the native multi-threaded writer
  (csrc/hostio.c, libds_hostgen.so) -- no per-scalar Python objects, which
  at N=2000 @4096 b would be ~4 million mpfr conversions.

``digits`` defaults to the CLI's ``Precision.decimal_digits`` (cli.py:326).
"""

from __future__ import annotations

import ctypes
import os

from .elim import EliminationTrace, MinorSeries
from .engine import HostResults
from .hostgen import _load
from .scalars import Precision, format_scalar
from .soa import SoA, ds_soa

__all__ = ["write_dets", "write_minors", "write_results", "MinorsStream", "read_minors_binary"]


def _default_digits(prec_bits: int, digits):
    return digits if digits else Precision(prec_bits).decimal_digits


def write_dets(trace: EliminationTrace, path, digits):
    """cli._write_dets (cli.py:218-221)."""
    with open(path, "w") as f:
        for i, d in enumerate(trace.det_series, 1):
            f.write(f"{i} {format_scalar(d, digits)}\n")


def write_minors(minors: MinorSeries, outdir, digits):
    """cli._write_minors (cli.py:224-232)."""
    os.makedirs(outdir, exist_ok=True)
    for m in minors.sizes():
        row = minors.rows[m]
        with open(os.path.join(outdir, f"minors_{m}.txt"), "w") as f:
            for k in range(m):
                norm = "undefined" if row.normalized is None else format_scalar(row.normalized[k], digits)
                f.write(f"{k + 1} {format_scalar(row.signed[k], digits)} {norm}\n")


def _lib():
    L = _load()
    if not getattr(L, "_io_sigs", False):
        L.dsh_write_dets.restype = ctypes.c_int
        L.dsh_write_dets.argtypes = [ctypes.c_char_p, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_long,
                                     ctypes.POINTER(ds_soa), ctypes.c_int]
        L.dsh_write_minors.restype = ctypes.c_int
        L.dsh_write_minors.argtypes = [ctypes.c_char_p, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_long,
                                       ctypes.POINTER(ds_soa), ctypes.POINTER(ds_soa),
                                       ctypes.POINTER(ctypes.c_uint8), ctypes.c_int, ctypes.c_int]
        L._io_sigs = True
    return L


def write_results(res: HostResults, n: int, prec_bits: int, kind: str, outdir, steps_done: int,
                  digits=None, minors: bool = True, nthreads: int = 0, swaps=None):
    """dets.txt (the first ``steps_done`` leading minors) and, if ``minors``,
    minors_<m>.txt for every emitted size, from a run's host results -- the
    files the CLI writes for the same run (cli.py:330, 356-357).

    ``swaps``: the per-step row-swap flags of a pivot_mode="partial" run
    (DeviceElimination.swaps).  The device keeps the unsigned pivot product; the
    reference's det_series carries the swap sign (elim.py:207, 216), applied here
    as an exact sign flip before formatting.  Omitting it for a run that swapped
    rows would write wrong signs, so partial-pivot results must pass it."""
    digits = _default_digits(prec_bits, digits)
    L = (prec_bits + 31) // 32
    k = 1 if kind == "complex" else 0
    os.makedirs(outdir, exist_ok=True)
    lib = _lib()
    det_soa = res.dets
    if swaps is not None and any(swaps):
        det_soa = res.dets.copy()
        sign = 1
        for i, sw in enumerate(list(swaps)[:steps_done]):
            if sw:
                sign = -sign
            if sign < 0:
                for c in range(det_soa.ncomp):  # + <-> -, +0 <-> -0 (wire sign codes)
                    det_soa.cls[c, i] ^= 1
    dets = det_soa.c()
    rc = lib.dsh_write_dets(os.path.join(str(outdir), "dets.txt").encode(), int(steps_done), k, L, prec_bits,
                            ctypes.byref(dets), int(digits))
    if rc != 0:
        raise OSError(-rc, f"writing {outdir}/dets.txt failed")
    if minors and res.signed is not None:
        flags = (res.row_flags & 0xff).astype("uint8")
        # 0 / 1 (normalized None) / 3 (normalized present), as the engine flags them
        sig, nrm = res.signed.c(), res.normalized.c()
        rc = lib.dsh_write_minors(str(outdir).encode(), int(n), k, L, prec_bits, ctypes.byref(sig), ctypes.byref(nrm),
                                  flags.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8)), int(digits), int(nthreads))
        if rc != 0:
            raise OSError(-rc, f"writing minors into {outdir} failed")


def soa_of(values, prec_bits: int, kind: str) -> SoA:
    """SoA of scalar objects (helper for tests and small callers)."""
    return SoA.from_scalars(list(values), prec_bits, kind)


# ---------------------------------------------------------------- streamed minors
DSMR_MAGIC = b"DSMR"
DSMR_VERSION = 1


class MinorsStream:
    """Consumer of the device's minors stream (DeviceElimination.stream_minors):
    the rows arrive in increasing size straight from pinned staging, so the
    output path never needs all N^2 minors in HBM or host RAM (SURVEY 8(f)
    rank 1, config 5: ~416 GB).  Per row it can
      * append a binary record to ``path`` (format DSMR v1: header ``DSMR``, u32
        version, u32 n, u32 prec, u8 kind; then per emitted row u32 m, u8 flags,
        the signed minors as ds SoA (ncomp x L x m u32 limbs plane-major, ncomp x m
        i32 exponents, ncomp x m u8 classes) and, when flags bit1 is set, the
        normalized minors in the same layout) -- see read_minors_binary;
      * keep rows whose size is <= ``keep_upto`` or in ``keep_sizes`` as SoA rows
        (parity checks on the prefix / Laplace rows);
      * fold every row into a checksum (``digest``): by default a fast order-aware
        sum of 64-bit words (numpy; the callback runs on the thread that issues
        the elimination, so it must stay cheap), or sha256 with hash="sha256".
    The callback copies what it keeps: its arguments are views of staging memory
    the engine reuses after it returns."""

    def __init__(self, n: int, prec_bits: int, kind: str = "real", path=None, keep_upto: int = 0,
                 keep_sizes=(), hash: str = "sum"):
        import hashlib
        self.n, self.p, self.kind = n, prec_bits, kind
        self.ncomp = 2 if kind == "complex" else 1
        self.L = (prec_bits + 31) // 32
        self.keep_upto, self.keep_sizes = keep_upto, set(keep_sizes)
        self.kept: dict = {}
        self.sizes: list = []
        self.bytes = 0
        self._hash = hash
        self._h = hashlib.sha256() if hash == "sha256" else None
        self._sum = 0
        self._f = None
        if path is not None:
            import struct
            self._f = open(path, "wb")
            self._f.write(DSMR_MAGIC + struct.pack("<IIIB", DSMR_VERSION, n, prec_bits, self.ncomp - 1))

    def __call__(self, g0: int, stride: int, nrows: int, signed: SoA, normalized: SoA, flags):
        import struct
        import numpy as np
        n = self.n
        for r in range(nrows):
            m = g0 + r * stride + 1
            fl = int(flags[r])
            if not fl & 1:
                continue
            sl = slice(r * n, r * n + m)
            # copies: the arguments are views of staging memory the engine reuses after this call
            parts = [np.array(signed.limbs[:, :, sl]), np.array(signed.exp[:, sl]), np.array(signed.cls[:, sl])]
            if fl & 2:
                parts += [np.array(normalized.limbs[:, :, sl]), np.array(normalized.exp[:, sl]),
                          np.array(normalized.cls[:, sl])]
            head = struct.pack("<IB", m, fl)
            if self._h is not None:
                self._h.update(head)
                for a in parts:
                    self._h.update(a.data)
            else:  # Fletcher-style sums of the bytes (all words, and every other one), mod 2^64
                acc = m * 0x9E3779B97F4A7C15 + fl
                for j, a in enumerate(parts):
                    b = a.reshape(-1).view(np.uint8)
                    acc += (2 * j + 1) * int(b.sum(dtype=np.uint64)) + (2 * j + 2) * int(b[::2].sum(dtype=np.uint64))
                self._sum = (self._sum * 1000003 + acc) & 0xFFFFFFFFFFFFFFFF
            if self._f is not None:
                self._f.write(head)
                for a in parts:
                    self._f.write(a.data)
            self.bytes += len(head) + sum(a.nbytes for a in parts)
            self.sizes.append(m)
            if m <= self.keep_upto or m in self.keep_sizes:
                sg = SoA(self.ncomp, self.L, m, parts[0], parts[1], parts[2])
                nm = SoA(self.ncomp, self.L, m, parts[3], parts[4], parts[5]) if fl & 2 else None
                self.kept[m] = (fl, sg, nm)

    @property
    def digest(self) -> str:
        return self._h.hexdigest() if self._h is not None else f"sum64:{self._sum:016x}"

    def close(self):
        if self._f is not None:
            self._f.close()
            self._f = None


def read_minors_binary(path):
    """Iterate (m, flags, signed SoA, normalized SoA | None) over a DSMR v1 file."""
    import struct
    import numpy as np
    with open(path, "rb") as f:
        head = f.read(17)
        if head[:4] != DSMR_MAGIC:
            raise ValueError(f"{path}: not a DSMR file")
        version, n, p, kind = struct.unpack("<IIIB", head[4:])
        if version != DSMR_VERSION:
            raise ValueError(f"{path}: unsupported DSMR version {version}")
        nc, L = kind + 1, (p + 31) // 32

        def soa(m):
            limbs = np.frombuffer(f.read(4 * nc * L * m), dtype=np.uint32).reshape(nc, L, m).copy()
            ex = np.frombuffer(f.read(4 * nc * m), dtype=np.int32).reshape(nc, m).copy()
            cl = np.frombuffer(f.read(nc * m), dtype=np.uint8).reshape(nc, m).copy()
            return SoA(nc, L, m, limbs, ex, cl)

        while True:
            rec = f.read(5)
            if len(rec) < 5:
                return
            m, fl = struct.unpack("<IB", rec)
            sg = soa(m)
            nm = soa(m) if fl & 2 else None
            yield m, fl, sg, nm
