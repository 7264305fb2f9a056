"""Row-cyclic sharded elimination (reference parexec.py:1-424) over B200 ranks.

Rows are interleaved across T ranks (rank r owns rows i with i % T == r,
parexec.py:50-52 in 0-based form).  At step i the owner of row i stages that
row, UNNORMALIZED, into its pivot buffer; the buffer is broadcast to every
rank; every rank recomputes the det chain and applies the identical per-row
update to the rows it owns; the owner of row i+1 emits the minor row.  A row's
final value depends only on its own history and the broadcast pivot rows, so
results are bit-identical for every T (parexec.py:3-8) -- the G-invariance the
tests gate on.

Transports:
  * "local"  -- T virtual shards in this process, one device context each
                (round-robin over the visible GPUs); the broadcast is a
                device-to-device / peer copy of the pivot buffer.
  * "process" / "nccl" -- one process per GPU.  Inside an initialised
                torch.distributed group (torchrun) every rank calls
                par_eliminate and the broadcast is torch.distributed.broadcast
                of a device tensor that IS the pivot buffer (NCCL over
                NVLink), stream-ordered with the kernels on torch's current
                stream.  From a plain process, par_eliminate forks the worker
                ranks itself (torch.multiprocessing spawn, TCP rendezvous on
                127.0.0.1) like the reference coordinator (parexec.py:350-405):
                NCCL when every rank has its own GPU, else gloo with a pinned
                host staging copy (ranks sharing a GPU).
The wire format of the reference (pack_row / unpack_row, MPRW v1 with CRC32,
parexec.py:72-157) is kept for API compatibility; the device path does not
serialize -- HBM already holds the binary limb layout.
"""

from __future__ import annotations

import os

import struct
import zlib
from dataclasses import dataclass, field

import numpy as np

from . import mp
from .elim import EliminationTrace, MinorSeries, minor_rows_from_results
from .engine import DeviceElimination, HostResults
from .errors import CorruptPayload, ZeroPivot
from .matrix import MatrixBuffer
from .mp import mpc, mpfr
from .scalars import Precision
from .soa import SoA

WIRE_MAGIC = b"MPRW"
WIRE_VERSION = 1
ABORT_MAGIC = b"MPRA"
_SIGN_POS, _SIGN_NEG, _SIGN_PZERO, _SIGN_NZERO = 0, 1, 2, 3


@dataclass(frozen=True)
class WorkerTopology:
    """Row ownership for T workers (parexec.py:39-55), 1-based like the reference."""

    workers: int
    n: int

    def __post_init__(self):
        if self.workers < 1:
            raise ValueError("worker count must be >= 1")

    def owner(self, row: int) -> int:
        return ((row - 1) % self.workers) + 1

    def owned_rows(self, worker: int) -> list:
        return list(range(worker, self.n + 1, self.workers))


@dataclass
class CommStats:
    """Broadcast accounting (parexec.py:58-69); bytes are pivot-buffer bytes."""

    broadcasts: int = 0
    bytes_total: int = 0
    per_step_bytes: list = field(default_factory=list)
    minor_messages: int = 0
    fanout_deliveries: int = 0


# ------------------------------------------------------------------ wire format

def _pack_real(out: bytearray, x):
    if x == 0:
        out.append(_SIGN_NZERO if mp.is_signed(x) else _SIGN_PZERO)
        out += struct.pack("<qI", 0, 0)
        return
    m, e = x.as_mantissa_exp()
    m, e = int(m), int(e)
    out.append(_SIGN_NEG if m < 0 else _SIGN_POS)
    mag = abs(m)
    nl = (mag.bit_length() + 63) // 64
    out += struct.pack("<qI", e, nl)
    out += mag.to_bytes(nl * 8, "little")


def pack_row(step: int, scalars, kind: str) -> bytes:
    """MPRW v1: magic, u8 version, u32 step, u32 records, records, CRC32."""
    out = bytearray(WIRE_MAGIC)
    out += struct.pack("<BII", WIRE_VERSION, step, len(scalars) * (2 if kind == "complex" else 1))
    for x in scalars:
        for part in ((x.real, x.imag) if kind == "complex" else (x,)):
            _pack_real(out, part)
    out += struct.pack("<I", zlib.crc32(bytes(out)))
    return bytes(out)


def _unpack_real(data: bytes, off: int, bits: int):
    sign = data[off]
    e, nl = struct.unpack_from("<qI", data, off + 1)
    off += 13
    if sign in (_SIGN_PZERO, _SIGN_NZERO):
        if nl:
            raise CorruptPayload("zero record with nonzero limb count")
        return (mpfr("-0") if sign == _SIGN_NZERO else mpfr(0)), off
    if sign not in (_SIGN_POS, _SIGN_NEG):
        raise CorruptPayload(f"bad sign byte {sign}")
    if off + nl * 8 > len(data):
        raise CorruptPayload("truncated limb data")
    mag = int.from_bytes(data[off:off + nl * 8], "little")
    off += nl * 8
    if mag.bit_length() > bits:
        raise CorruptPayload("mantissa wider than the declared precision")
    x = mpfr(-mag if sign == _SIGN_NEG else mag)
    return mp.mul_2exp(x, e), off


def unpack_row(data: bytes, prec: Precision, kind: str):
    if len(data) < 17:
        raise CorruptPayload("payload shorter than the fixed header")
    if data[:4] != WIRE_MAGIC:
        raise CorruptPayload(f"bad magic {data[:4]!r}")
    (crc,) = struct.unpack_from("<I", data, len(data) - 4)
    if zlib.crc32(data[:-4]) != crc:
        raise CorruptPayload("CRC mismatch")
    version, step, records = struct.unpack_from("<BII", data, 4)
    if version != WIRE_VERSION:
        raise CorruptPayload(f"unsupported wire version {version}")
    if kind == "complex" and records % 2:
        raise CorruptPayload("odd record count for complex payload")
    off, reals = 13, []
    with prec.context():
        for _ in range(records):
            x, off = _unpack_real(data, off, prec.bits)
            reals.append(x)
        if off != len(data) - 4:
            raise CorruptPayload("trailing bytes after the last record")
        if kind == "complex":
            return step, [mpc(reals[k], reals[k + 1]) for k in range(0, records, 2)]
    return step, reals


def pack_abort(step: int, worker: int) -> bytes:
    return ABORT_MAGIC + struct.pack("<II", step, worker)


def is_abort(data: bytes) -> bool:
    return data[:4] == ABORT_MAGIC


def unpack_abort(data: bytes):
    return struct.unpack_from("<II", data, 4)


def block_reassign_plan(step: int, n: int, workers: int) -> list:
    """Contiguous blocks over rows step+1..n with sizes within one
    (parexec.py:173-194); provided for API parity, unused by the executors."""
    remaining = n - step
    if remaining <= 0:
        return []
    base, extra = divmod(remaining, workers)
    plan, row = [], step + 1
    for w in range(1, workers + 1):
        size = base + (1 if w <= extra else 0)
        if size == 0:
            break
        plan.append((w, row, row + size - 1))
        row += size
    return plan


# ------------------------------------------------------------------ executors

def _assemble(A: MatrixBuffer, trace: EliminationTrace, res: HostResults, done: int, collect_minors: bool,
              sink, out: MinorSeries | None):
    p = A.prec.bits
    from .soa import paused_gc
    with paused_gc():
        trace.pivots.extend(res.pivots.scalars(0, done, p))
        trace.det_series.extend(res.dets.scalars(0, done, p))
        rows = minor_rows_from_results(res, A.n, p) if collect_minors else []
    trace.step = done
    if collect_minors:
        emit = sink if sink is not None else out.add
        for row in rows:
            emit(row)


def _local_run(A: MatrixBuffer, workers: int, collect_minors: bool, series: bool, stats: CommStats, devices):
    import torch
    n, p = A.n, A.prec.bits
    devs = devices if devices is not None else list(range(max(1, torch.cuda.device_count())))
    soa = A.to_soa()
    ranks = [DeviceElimination(n, p, A.kind, devs[r % len(devs)], r, workers) for r in range(workers)]
    try:
        for e in ranks:
            e.load(soa)
        _, pbytes = ranks[0].pivot_buffer()
        lib = ranks[0].lib
        for i in range(n):
            owner = ranks[i % workers]
            owner.stage(i)
            for e in ranks:
                if e is not owner:
                    rc = lib.ds_pivot_copy(e.ctx, owner.ctx)
                    if rc != 0:
                        raise RuntimeError(f"ds_pivot_copy failed: {rc}")
            for e in ranks:
                e.step(i, collect_minors, series)
            stats.broadcasts += 1
            stats.bytes_total += pbytes
            stats.per_step_bytes.append(pbytes)
            stats.fanout_deliveries += workers
        failed = [e.status() for e in ranks]
        f = max(failed)
        done = f if f >= 0 else n
        res = HostResults.alloc(n, ranks[0].ncomp, ranks[0].L, collect_minors)
        for e in ranks:  # trace is replicated; each rank adds its owned minors rows
            e.results(done, res)
            e.fetch(soa)
        stats.minor_messages = sum(1 for m in range(2, n + 1) if res.row_flags[m - 1] & 1)
    finally:
        for e in ranks:
            e.close()
    A._set_lazy(soa)
    return res, done


def dist_run(engine, n: int, collect_minors: bool, series: bool, pivot, broadcast, stats: CommStats | None = None,
             lookahead: bool = True, stream_every: int = 0):
    """Generic per-rank step loop of the message-passing executor.

    engine    -- this rank's context (stage/step/status), a DeviceElimination
                 on a GPU; the CPU tests pass the C oracle's context instead.
    pivot     -- the tensor holding the pivot buffer bytes (device or host).
    broadcast -- callable(tensor, src_rank) (torch.distributed.broadcast).
    stream_every -- > 0 when the engine streams its minors rows (ds_stream_minors):
                 flush every that many steps and at the end.
    Returns the failed step (-1 if none).
    """
    world, rank = engine.world, engine.rank
    nbytes = pivot.numel() * pivot.element_size()
    la = _lookahead_setup(engine, n, pivot) if lookahead else None
    for i in range(n):
        owner = i % world
        if rank == owner:
            engine.stage(i)
        broadcast(pivot, owner)
        engine.step(i, collect_minors, series)
        if stats is not None:
            stats.broadcasts += 1
            stats.bytes_total += nbytes
            stats.per_step_bytes.append(nbytes)
            stats.fanout_deliveries += world
        if la is not None and i + 2 < n:
            # lookahead: the tile holding column i+1 is already updated on the
            # lookahead stream; the owner of row i+1 shares the next pivot there and
            # every rank computes step i+1's multipliers while step i's update runs
            ext, scal = la
            o1 = (i + 1) % world
            with _torch().cuda.stream(ext):
                if rank == o1:
                    engine.lookahead_pivot(i + 1, scal.data_ptr())
                broadcast(scal, o1)
            engine.lookahead_mult(i + 1, scal.data_ptr())
        if stream_every and (i + 1) % stream_every == 0:
            engine.stream_flush(i + 1)
    if la is not None:
        engine.lookahead_enable(0)
    failed = engine.status()
    if stream_every:
        engine.stream_flush(failed if failed >= 0 else n, final=True)
    return failed


def _lookahead_setup(engine, n: int, pivot):
    """(lookahead stream context, exchange buffer) for a multi-rank GPU run, or None
    (CPU engines, one rank, DS_NO_DIST_LOOKAHEAD)."""
    if not hasattr(engine, "lookahead_enable") or os.environ.get("DS_NO_DIST_LOOKAHEAD"):
        return None
    if not getattr(pivot, "is_cuda", False) or not engine.counters().get("tc_engine"):
        return None  # only the tensor-core engine splits its update for the lookahead
    torch = _torch()
    if engine.L > 2048:
        return None  # the lookahead multipliers need the warp division (L <= 2048 limbs)
    engine.lookahead_enable(n)
    ext = torch.cuda.ExternalStream(engine.lookahead_stream(), device=pivot.device)
    scal = torch.zeros(4 * engine.L + 8, dtype=torch.uint8, device=pivot.device)
    return ext, scal


def _torch():
    import torch
    return torch


def allreduce_gather(res: HostResults, soa: SoA | None, rank: int, world: int, allreduce):
    """Combine per-rank owned rows (minors and matrix rows) into full copies on
    every rank: non-owned entries are zeroed and an integer SUM all-reduce
    reassembles them exactly."""
    n = len(res.row_flags)
    own = np.zeros(n, dtype=bool)
    own[rank::world] = True

    def combine(a: SoA):
        count = a.count
        rows = count // n
        mask = np.repeat(own, rows) if rows > 1 else own
        if rows > 1:
            a.limbs[:, :, ~mask] = 0
            a.exp[:, ~mask] = 0
            a.cls[:, ~mask] = 0
        allreduce(a.limbs.view(np.int32))
        allreduce(a.exp)
        allreduce(a.cls.view(np.uint8))

    if res.signed is not None:
        combine(res.signed)
        combine(res.normalized)
    flags = res.row_flags.copy()
    flags[~own] = 0
    allreduce(flags)
    res.row_flags[:] = flags
    if soa is not None:
        mrows = np.repeat(own, n)
        soa.limbs[:, :, ~mrows] = 0
        soa.exp[:, ~mrows] = 0
        soa.cls[:, ~mrows] = 0
        allreduce(soa.limbs.view(np.int32))
        allreduce(soa.exp)
        allreduce(soa.cls)


def _rank_setup(eng, backend: str, rank: int):
    """Pivot tensor + broadcast callable for one device rank.  NCCL broadcasts the
    device buffer in place on torch's current stream (the context launches there);
    gloo (ranks sharing a GPU, or CPU-only process groups) stages it through a
    pinned host copy.  Returns (pivot, broadcast, lookahead_ok)."""
    import torch
    import torch.distributed as dist
    dev = torch.cuda.current_device()
    _, pbytes = eng.pivot_buffer()
    pivot = torch.empty(pbytes, dtype=torch.uint8, device=f"cuda:{dev}")
    _native_check(eng.lib.ds_use_pivot_buffer(eng.ctx, pivot.data_ptr(), pbytes), "ds_use_pivot_buffer")
    cur = torch.cuda.current_stream()
    if cur.cuda_stream == 0:
        # the legacy default stream has handle 0, which ds_set_stream reads as "own stream":
        # run on a dedicated torch stream so collectives and kernels share one stream order
        cur = torch.cuda.Stream()
        torch.cuda.set_stream(cur)
    _native_check(eng.lib.ds_set_stream(eng.ctx, cur.cuda_stream), "ds_set_stream")
    if backend == "nccl":
        return pivot, (lambda t, src: dist.broadcast(t, src=src)), True
    staging = {}

    def bcast(t, src):
        host = staging.get(t.numel())
        if host is None:
            host = staging[t.numel()] = torch.empty(t.numel(), dtype=t.dtype, pin_memory=True)
        if rank == src:
            host.copy_(t)  # synchronous w.r.t. the current stream: after the staging kernel
        dist.broadcast(host, src=src)
        if rank != src:
            t.copy_(host)
    return pivot, bcast, False


def _native_check(rc: int, what: str):
    if rc != 0:
        raise RuntimeError(f"{what} failed with code {rc}")


def _group_run(A: MatrixBuffer, workers: int, collect_minors: bool, series: bool, stats: CommStats):
    """Every rank of an already-initialised process group (e.g. torchrun) calls
    par_eliminate; each returns the full result, like the reference coordinator."""
    import torch
    import torch.distributed as dist
    world, rank = dist.get_world_size(), dist.get_rank()
    if world != workers:
        raise ValueError(f"workers={workers} but the process group has {world} ranks")
    n, p = A.n, A.prec.bits
    dev = torch.cuda.current_device()
    backend = dist.get_backend()
    eng = DeviceElimination(n, p, A.kind, dev, rank, world)
    caller_stream = torch.cuda.current_stream()
    try:
        soa = A.to_soa()
        eng.load(soa)
        pivot, bcast, la_ok = _rank_setup(eng, backend, rank)
        failed = dist_run(eng, n, collect_minors, series, pivot, bcast, stats, lookahead=la_ok)
        # agree on the failed step (identical on every rank by construction)
        f = torch.tensor([failed], dtype=torch.int64, device=f"cuda:{dev}" if backend == "nccl" else "cpu")
        dist.all_reduce(f, op=dist.ReduceOp.MAX)
        failed = int(f.item())
        done = failed if failed >= 0 else n
        res = HostResults.alloc(n, eng.ncomp, eng.L, collect_minors)
        eng.results(done, res)
        eng.fetch(soa)
        eng.lib.ds_set_stream(eng.ctx, None)
        eng.lib.ds_use_pivot_buffer(eng.ctx, None, 0)
    finally:
        eng.close()
        torch.cuda.set_stream(caller_stream)

    def allreduce(arr):
        t = torch.from_numpy(np.ascontiguousarray(arr))
        if backend == "nccl":
            t = t.to(f"cuda:{dev}")
        dist.all_reduce(t)
        arr[...] = t.cpu().numpy()

    allreduce_gather(res, soa, rank, world, allreduce)
    A._set_lazy(soa)
    return res, done


def _free_port() -> int:
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _spawn_worker(rank: int, world: int, port: int, d: str, n: int, p: int, kind: str, collect_minors: bool,
                  series: bool, engine_factory=None):
    """One worker process of par_eliminate(transport="process") without a process
    group (ref parexec.py:290-333): one GPU per rank when there are enough (NCCL),
    else ranks share the visible GPUs and broadcast over gloo.  Reads the input
    from the coordinator's scratch directory, writes back its owned rows."""
    import json
    import traceback
    try:
        import torch
        import torch.distributed as dist
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        ncomp = 2 if kind == "complex" else 1
        L = (p + 31) // 32
        src = SoA(ncomp, L, n * n, np.load(os.path.join(d, "limbs.npy")), np.load(os.path.join(d, "exp.npy")),
                  np.load(os.path.join(d, "cls.npy")))
        if engine_factory is None:
            ndev = torch.cuda.device_count()
            if ndev == 0:
                from .errors import DeviceUnavailable
                raise DeviceUnavailable("par_eliminate(transport='process') needs a CUDA device")
            dev = rank % ndev
            torch.cuda.set_device(dev)
            backend = "nccl" if ndev >= world and not os.environ.get("DS_PAR_FORCE_GLOO") else "gloo"
            kw = {"device_id": torch.device(f"cuda:{dev}")} if backend == "nccl" else {}
            dist.init_process_group(backend, rank=rank, world_size=world, **kw)
            eng = DeviceElimination(n, p, kind, dev, rank, world)
            eng.load(src)
            pivot, bcast, la_ok = _rank_setup(eng, backend, rank)
        else:  # test hook: a CPU engine with the same interface (gloo)
            backend = "gloo"
            dist.init_process_group(backend, rank=rank, world_size=world)
            eng = engine_factory(n, p, kind, rank, world)
            eng.load(src)
            pivot = torch.from_numpy(eng.pivot_array())
            bcast, la_ok = (lambda t, s_: dist.broadcast(t, src=s_)), False
        stats = CommStats()
        failed = dist_run(eng, n, collect_minors, series, pivot, bcast, stats, lookahead=la_ok)
        f = torch.tensor([failed], dtype=torch.int64, device=pivot.device if backend == "nccl" else "cpu")
        dist.all_reduce(f, op=dist.ReduceOp.MAX)
        failed = int(f.item())
        done = failed if failed >= 0 else n
        res = HostResults.alloc(n, eng.ncomp, eng.L, collect_minors)
        eng.results(done, res)
        fin = SoA.like(src)
        eng.fetch(fin)
        if hasattr(eng, "lib") and engine_factory is None:
            eng.lib.ds_set_stream(eng.ctx, None)
            eng.lib.ds_use_pivot_buffer(eng.ctx, None, 0)
        rows = np.arange(rank, n, world)

        def own(a: SoA):
            return (a.limbs.reshape(ncomp, L, n, n)[:, :, rows, :], a.exp.reshape(ncomp, n, n)[:, rows, :],
                    a.cls.reshape(ncomp, n, n)[:, rows, :])

        out = {}
        out["m_limbs"], out["m_exp"], out["m_cls"] = own(fin)
        if collect_minors:
            out["s_limbs"], out["s_exp"], out["s_cls"] = own(res.signed)
            out["n_limbs"], out["n_exp"], out["n_cls"] = own(res.normalized)
        out["flags"] = res.row_flags[rows]
        if rank == 0:
            for name, a in (("piv", res.pivots), ("det", res.dets)):
                out[name + "_limbs"], out[name + "_exp"], out[name + "_cls"] = a.limbs, a.exp, a.cls
            with open(os.path.join(d, "meta.json"), "w") as fh:
                json.dump({"done": done, "broadcasts": stats.broadcasts, "bytes_total": stats.bytes_total,
                           "per_step_bytes": stats.per_step_bytes[:1], "backend": backend}, fh)
        np.savez(os.path.join(d, f"out{rank}.npz"), **out)
        eng.close()
        dist.barrier()
        dist.destroy_process_group()
    except BaseException:
        with open(os.path.join(d, f"err{rank}.txt"), "w") as fh:
            fh.write(traceback.format_exc())
        raise


def _spawn_run(A: MatrixBuffer, workers: int, collect_minors: bool, series: bool, stats: CommStats,
               engine_factory=None):
    """par_eliminate(transport="process") from a plain process: fork `workers` ranks
    (torch.multiprocessing, spawn), as the reference's coordinator does
    (ref parexec.py:350-405), and assemble their owned rows."""
    import json
    import tempfile
    import torch.multiprocessing as tmp
    from .errors import WorkerFailure
    n, p = A.n, A.prec.bits
    soa = A.to_soa()
    nc, L = soa.ncomp, soa.L
    with tempfile.TemporaryDirectory(prefix="ds_par_") as d:
        np.save(os.path.join(d, "limbs.npy"), soa.limbs)
        np.save(os.path.join(d, "exp.npy"), soa.exp)
        np.save(os.path.join(d, "cls.npy"), soa.cls)
        ctx = tmp.get_context("spawn")
        port = _free_port()
        procs = [ctx.Process(target=_spawn_worker,
                             args=(r, workers, port, d, n, p, A.kind, collect_minors, series, engine_factory))
                 for r in range(workers)]
        for pr in procs:
            pr.start()
        # a rank that dies leaves the others blocked in a collective: stop them all
        import time as _time
        while any(pr.exitcode is None for pr in procs):
            if any(pr.exitcode not in (None, 0) for pr in procs):
                for pr in procs:
                    if pr.exitcode is None:
                        pr.terminate()
                for pr in procs:
                    pr.join(timeout=30)
                break
            _time.sleep(0.05)
        for pr in procs:
            pr.join()
        for r, pr in enumerate(procs):
            if pr.exitcode != 0:
                msg = ""
                ep = os.path.join(d, f"err{r}.txt")
                if os.path.exists(ep):
                    msg = open(ep).read().strip().splitlines()[-1]
                raise WorkerFailure(r + 1, f"worker exited with code {pr.exitcode}: {msg}")
        meta = json.load(open(os.path.join(d, "meta.json")))
        done = int(meta["done"])
        res = HostResults.alloc(n, nc, L, collect_minors)
        fin = SoA(nc, L, n * n)
        for r in range(workers):
            z = np.load(os.path.join(d, f"out{r}.npz"))
            rows = np.arange(r, n, workers)
            targets = [("m", fin)] + ([("s", res.signed), ("n", res.normalized)] if collect_minors else [])
            for key, a in targets:
                a.limbs.reshape(nc, L, n, n)[:, :, rows, :] = z[key + "_limbs"]
                a.exp.reshape(nc, n, n)[:, rows, :] = z[key + "_exp"]
                a.cls.reshape(nc, n, n)[:, rows, :] = z[key + "_cls"]
            res.row_flags[rows] = z["flags"]
            if r == 0:
                for key, a in (("piv", res.pivots), ("det", res.dets)):
                    a.limbs[...] = z[key + "_limbs"]
                    a.exp[...] = z[key + "_exp"]
                    a.cls[...] = z[key + "_cls"]
    stats.broadcasts = int(meta["broadcasts"])
    stats.bytes_total = int(meta["bytes_total"])
    stats.per_step_bytes = list(meta["per_step_bytes"]) * stats.broadcasts
    stats.fanout_deliveries = stats.broadcasts * workers
    stats.minor_messages = sum(1 for m in range(2, n + 1) if res.row_flags[m - 1] & 1)
    A._set_lazy(fin)
    return res, done


def _process_run(A: MatrixBuffer, workers: int, collect_minors: bool, series: bool, stats: CommStats,
                 engine_factory=None):
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized():
        return _group_run(A, workers, collect_minors, series, stats)
    return _spawn_run(A, workers, collect_minors, series, stats, engine_factory)


def par_eliminate(A: MatrixBuffer, workers: int, transport: str = "local", collect_minors: bool = True,
                  series: bool = True, sink=None, devices=None, _engine_factory=None):
    """Sharded elimination of A in place over `workers` ranks
    (parexec.py:408-424).  Returns (trace, minor_series, comm_stats), bit-
    identical to eliminate() for every worker count and transport."""
    if transport not in ("local", "process", "nccl"):
        raise ValueError(f"unknown transport {transport!r}")
    topo = WorkerTopology(workers, A.n)  # validates workers >= 1
    stats = CommStats()
    trace = EliminationTrace(n=A.n, prec=A.prec)
    out = MinorSeries(A.prec) if collect_minors else None
    if transport == "local":
        res, done = _local_run(A, topo.workers, collect_minors, series, stats, devices)
    else:
        res, done = _process_run(A, topo.workers, collect_minors, series, stats, _engine_factory)
    _assemble(A, trace, res, done, collect_minors, sink, out)
    if done < A.n:
        raise ZeroPivot(done + 1, trace=trace, series=out)
    return trace, out, stats
