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

__all__ = ["write_dets", "write_minors", "write_results"]


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
                  digits=None, minors: bool = True, nthreads: int = 0):
    """dets.txt (the first ``steps_done`` leading minors) and, if ``minors``,
    minors_<m>.txt for every emitted size, from a run's host results -- the
    files the CLI writes for the same run (cli.py:330, 356-357)."""
    digits = _default_digits(prec_bits, digits)
    L = (prec_bits + 31) // 32
    k = 1 if kind == "complex" else 0
    os.makedirs(outdir, exist_ok=True)
    lib = _lib()
    dets = res.dets.c()
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
