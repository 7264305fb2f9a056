"""Checkpoint / resume in the reference CLI's format.

A checkpoint directory (cli._Checkpointer, cli.py:94-168) holds
``matrix.mpmat`` -- the mid-elimination buffer in the MPMAT text format
(matrix.py:109-140; the dead lower slots carry the L factor) -- and
``state.txt`` -- ``step <k>`` then one ``pivot <scalar>`` line per completed
step.  Resuming re-derives the determinant series from the pivots (elim.py
det chain, RN per product) and continues from step k.

Here the matrix file is written and parsed by the native multi-threaded
MPMAT code (csrc/hostio.c) straight from / into the ds SoA, so a checkpoint
of an N=2000 @4096 b run does not go through four million Python scalars.
Files are byte-identical to the reference's (tests/test_output.py), so
checkpoints move freely between the two implementations.
"""

from __future__ import annotations

import ctypes
import os

from .elim import EliminationTrace
from .errors import ParseError
from .hostgen import _load
from .matrix import MatrixBuffer
from .scalars import Precision, format_scalar, parse_scalar
from .soa import SoA, ds_soa

__all__ = ["Checkpoint", "save_mpmat", "load_mpmat"]

_KIND = {"real": 0, "complex": 1}


def _lib():
    L = _load()
    if not getattr(L, "_mpmat_sigs", False):
        L.dsh_write_mpmat.restype = ctypes.c_int
        L.dsh_write_mpmat.argtypes = [ctypes.c_char_p, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_long,
                                      ctypes.POINTER(ds_soa), ctypes.c_int]
        L.dsh_mpmat_header.restype = ctypes.c_int
        L.dsh_mpmat_header.argtypes = [ctypes.c_char_p, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int),
                                       ctypes.POINTER(ctypes.c_long)]
        L.dsh_read_mpmat.restype = ctypes.c_int
        L.dsh_read_mpmat.argtypes = [ctypes.c_char_p, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_long,
                                     ctypes.POINTER(ds_soa), ctypes.c_int]
        L._mpmat_sigs = True
    return L


def save_mpmat(soa: SoA, n: int, prec_bits: int, kind: str, path, nthreads: int = 0):
    """MatrixBuffer.save (matrix.py:109-115) of an n x n ds SoA."""
    L = (prec_bits + 31) // 32
    s = soa.c()
    rc = _lib().dsh_write_mpmat(str(path).encode(), int(n), _KIND[kind], L, int(prec_bits), ctypes.byref(s),
                                int(nthreads))
    if rc != 0:
        raise OSError(-rc, f"writing {path} failed")


def load_mpmat(path, nthreads: int = 0):
    """MatrixBuffer.load (matrix.py:117-140) into a ds SoA: (soa, n, prec_bits, kind)."""
    lib = _lib()
    n, k, bits = ctypes.c_int(), ctypes.c_int(), ctypes.c_long()
    rc = lib.dsh_mpmat_header(str(path).encode(), ctypes.byref(n), ctypes.byref(k), ctypes.byref(bits))
    if rc == -1:
        raise ParseError(f"{path}: not an MPMAT file")
    if rc != 0:
        raise ParseError(f"cannot read {path}: {os.strerror(-rc)}")
    kind = "complex" if k.value == 1 else "real"
    L = (bits.value + 31) // 32
    soa = SoA(2 if kind == "complex" else 1, L, n.value * n.value)
    s = soa.c()
    rc = lib.dsh_read_mpmat(str(path).encode(), n.value, k.value, L, bits.value, ctypes.byref(s), int(nthreads))
    if rc == -2:
        raise ParseError(f"{path}: truncated")
    if rc == -1:
        raise ParseError(f"{path}: malformed scalar")
    if rc != 0:
        raise ParseError(f"cannot read {path}: {os.strerror(-rc)}")
    return soa, n.value, int(bits.value), kind


class Checkpoint:
    """The reference CLI's checkpoint directory (cli._Checkpointer)."""

    def __init__(self, directory):
        self.dir = str(directory)
        os.makedirs(self.dir, exist_ok=True)

    def resumable(self) -> bool:
        return os.path.exists(os.path.join(self.dir, "state.txt"))

    def write_soa(self, soa: SoA, n: int, prec_bits: int, kind: str, step: int, pivots):
        """matrix.mpmat + state.txt for a run stopped after `step` steps, written to
        temporary names and moved into place (cli.py:110-120)."""
        tmp_m = os.path.join(self.dir, "matrix.mpmat.tmp")
        tmp_s = os.path.join(self.dir, "state.txt.tmp")
        save_mpmat(soa, n, prec_bits, kind, tmp_m)
        with open(tmp_s, "w") as f:
            f.write(f"step {step}\n")
            for p in pivots:
                f.write("pivot " + format_scalar(p) + "\n")
        os.replace(tmp_m, os.path.join(self.dir, "matrix.mpmat"))
        os.replace(tmp_s, os.path.join(self.dir, "state.txt"))

    def write(self, A: MatrixBuffer, trace: EliminationTrace):
        """cli._Checkpointer.write(A, trace)."""
        self.write_soa(A.to_soa(), A.n, A.prec.bits, A.kind, trace.step, trace.pivots)

    def load_soa(self):
        """(soa, n, prec_bits, kind, trace) with the determinant series re-derived
        from the pivots exactly as the reference does (cli.py:128-152)."""
        soa, n, bits, kind = load_mpmat(os.path.join(self.dir, "matrix.mpmat"))
        prec = Precision(bits)
        trace = EliminationTrace(n=n, prec=prec)
        with open(os.path.join(self.dir, "state.txt")) as f:
            header = f.readline().split()
            if len(header) != 2 or header[0] != "step":
                raise ParseError("corrupt checkpoint state file")
            step = int(header[1])
            with prec.context():
                det = None
                for line in f:
                    if not line.startswith("pivot "):
                        raise ParseError("corrupt checkpoint state file")
                    p = parse_scalar(line[6:], prec, kind)
                    trace.pivots.append(p)
                    det = p if det is None else det * p
                    trace.det_series.append(det)
        if len(trace.pivots) != step:
            raise ParseError("checkpoint pivot count does not match step")
        trace.step = step
        return soa, n, bits, kind, trace

    def load(self):
        """cli._Checkpointer.load(): (MatrixBuffer, trace, step)."""
        soa, n, bits, kind, trace = self.load_soa()
        A = MatrixBuffer.from_soa(n, kind, Precision(bits), soa)
        return A, trace, trace.step

