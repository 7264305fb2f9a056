#!/usr/bin/env python
"""Benchmark of the hot path: all leading minors + last-column minors of an
N x N matrix at p bits, one pass of the unpivoted elimination per "step".

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload (BASELINE.json metric "limb-MAC/s + seconds to all minors
(N=2000 @4096b) at 1/2/4/8 B200 vs INT32 peak"): N=2000, p=4096 bits (L=128
limbs), collect_minors + series (every leading size emitted), real matrix.

value    = schoolbook limb-MACs of the whole elimination (n(n-1)^2/2 * L^2)
           / device time of one pass, inputs resident in HBM (restored from a
           device snapshot each step; minors stay in HBM), max over ranks.
e2e      = same metric through the C ABI with HOST buffers: per step the
           pinned host matrix is copied in (ds_load), the pass runs, and the
           pivots/dets/signed/normalized minors are copied out.
roofline = the update kernel (ds_tc.cu, tcgen05 kind::i8) timed live with
           CUDA events around every launch: algorithmic HBM bytes (read + write
           of every updated element) per second vs the measured HBM peak.
cpu_baseline / --impl reference = the reference hot loop (elim.py:37-53)
           restated over MPFR (oracle/), all host threads, bounded sample.
Multi-GPU (torchrun): row-cyclic shards, per-step NCCL broadcast of the pivot
row (parexec.py semantics), strong scaling of the same N x N problem.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


def measured_hbm_peak():
    """HBM GB/s from MEASURED_PEAKS.json (driver-written), else the profiling recipe's fallback."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs"
    except Exception:
        return 6650.0, "fallback 6.65 TB/s (B200_PROFILING.md)"


def committed_profile(n, prec):
    """The committed ncu --set full capture of one update launch of this workload
    (profiles/update_traffic.json): DRAM bytes per element (dram__bytes_read.sum +
    dram__bytes_write.sum), issue-active and tensor-pipe fractions, limiter."""
    try:
        with open(os.path.join(ROOT, "profiles", "update_traffic.json")) as f:
            d = json.load(f)
        if d.get("n") == n and d.get("prec_bits") == prec:
            return d
    except Exception:
        pass
    return None


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--dim", dest="n", type=int, default=2000)
    ap.add_argument("--bits", dest="prec", type=int, default=4096)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-parity", action="store_true", help="skip the oracle parity leg (outside the timed region)")
    ap.add_argument("--parity-m", type=int, default=256, help="leading block size of the prefix parity check")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="gloo: ranks may share a GPU (host-staged pivot broadcast; tests only)")
    ap.add_argument("--dist", action="store_true",
                    help="use the torch.distributed (NCCL) step loop even at world size 1 (testing)")
    ap.add_argument("--gen-budget", type=float, default=420.0,
                    help="max seconds of host time to build the Artless input before falling back to random")
    ap.add_argument("--family", default="beta", choices=["beta", "random", "power"],
                    help="beta: Artless-method beta matrix (genmat.beta_matrix, Eq. 9); random: random_uniform; "
                         "power: the complex Artless zero-power matrix (genmat.power_matrix, M = ceil((N-1)/2), "
                         "leading N x N block as the reference CLI's --limit-n)")
    return ap.parse_args()


ZEROS = os.path.join(ROOT, "data", "zeta_zeros_4096.txt")


def gamma_cache_path(n: int, p: int) -> str:
    return os.path.join(ROOT, "data", f"beta_gammas_p{p}_N{n}.npz")


def build_input(args, pinned: bool, rank: int = 0, world: int = 1, agree=None):
    """(SoA matrix, description, seconds).  beta: bit-identical to
    genmat.beta_matrix(load_zeros(zeros, Precision(p), n), n, SpougeGamma(),
    Precision(p)) (tests/test_hostgen.py), built by the multi-threaded C
    builder from the cached column Gammas when present."""
    import numpy as np
    t0 = time.perf_counter()
    if args.family == "beta":
        from paper_1308_1536_b200 import hostgen
        from paper_1308_1536_b200.soa import SoA
        gammas = None
        cp = gamma_cache_path(args.n, args.prec)
        if os.path.exists(cp):
            z = np.load(cp)
            gammas = SoA(2, int(z["L"]), int(z["count"]), np.ascontiguousarray(z["limbs"]),
                         np.ascontiguousarray(z["exp"]), np.ascontiguousarray(z["cls"]))
        # each rank builds only the rows it owns (row-cyclic); host threads shared by the local ranks
        local_world = int(os.environ.get("LOCAL_WORLD_SIZE", "1"))
        threads = max(1, len(os.sched_getaffinity(0)) // local_world)
        bb = hostgen.BetaBuilder(ZEROS, args.n, args.prec, gammas=gammas, pinned=pinned, nthreads=threads,
                                 row0=rank, rstep=world)
        probe = max(1, min(args.n, 2 * threads))
        bb.fill(probe)
        # later columns (larger ordinates) cost more per entry: 1.3x margin
        est = 1.3 * (time.perf_counter() - t0) * args.n / probe
        if agree is not None:  # every rank must build the same family: decide on the slowest rank's estimate
            est = agree(est)
        if est <= args.gen_budget:
            bb.fill(args.n)
            A = bb.out
            return A, workload_desc(args), time.perf_counter() - t0
        print(f"[bench] beta matrix generation would take ~{est:.0f}s > --gen-budget {args.gen_budget:.0f}s "
              f"on this host: using random_uniform (same shape, same work)", file=sys.stderr)
        args.family = "random"
    if args.family == "power":
        from paper_1308_1536_b200 import hostgen
        from paper_1308_1536_b200.soa import SoA
        M = args.n // 2  # 2M + 1 >= n rows: the leading n x n block (prefix property, cli.py:296-302)
        N = 2 * M + 1
        local_world = int(os.environ.get("LOCAL_WORLD_SIZE", "1"))
        threads = max(1, len(os.sched_getaffinity(0)) // local_world)
        full = hostgen.power_matrix_soa(ZEROS, M, args.prec, nthreads=threads, row0=rank, rstep=world)
        n, L = args.n, (args.prec + 31) // 32
        rows_here = len(range(rank, n, world))
        nrow_full = full.count // N
        lim = full.limbs.reshape(2, L, nrow_full, N)[:, :, :rows_here, :n]
        A = SoA(2, L, rows_here * n, pinned=pinned)
        A.limbs[...] = lim.reshape(2, L, -1)
        A.exp[...] = full.exp.reshape(2, nrow_full, N)[:, :rows_here, :n].reshape(2, -1)
        A.cls[...] = full.cls.reshape(2, nrow_full, N)[:, :rows_here, :n].reshape(2, -1)
        return A, workload_desc(args), time.perf_counter() - t0
    if args.family == "random":
        from paper_1308_1536_b200.synth import counter_uniform_soa, random_uniform_soa
        if world > 1:  # this rank's rows only (the counter-based draw is a function of (row, col))
            A = counter_uniform_soa(args.n, args.prec, 2000, rows=range(rank, args.n, world), pinned=pinned)
        else:
            A = random_uniform_soa(args.n, args.prec, 2000, pinned=pinned)
    return A, workload_desc(args), time.perf_counter() - t0


def workload_desc(args) -> str:
    if args.family == "beta":
        return (f"Artless beta matrix a[n][j] = beta_n(gamma_j) (genmat.beta_matrix, Eq. 9), N={args.n} "
                f"@{args.prec}b, zeros data/zeta_zeros_4096.txt")
    if args.family == "power":
        return (f"Artless zero-power matrix (genmat.power_matrix, complex, M={args.n // 2}, t=25), leading "
                f"N={args.n} block @{args.prec}b, zeros data/zeta_zeros_4096.txt (SURVEY 8d config 3)")
    return f"N={args.n} random_uniform real matrix @{args.prec}b (SURVEY 8d config 3')"


def kind_of(args) -> str:
    return "complex" if args.family == "power" else "real"


def work_limb_macs(n: int, L: int, complex_: bool = False) -> float:
    return n * (n - 1) ** 2 / 2 * L * L * (4 if complex_ else 1)


def workload(args, desc: str = "") -> dict:
    return {"workload": f"{desc}: all leading minors + last-column signed/normalized minors for every size "
                        f"(BASELINE config 3)",
            "family": args.family,
            "n": args.n, "prec_bits": args.prec, "limbs": (args.prec + 31) // 32, "kind": kind_of(args),
            "collect_minors": True, "series": True,
            "l2": "inputs larger than L2 (matrix %.1f GB)" % (args.n * args.n * (4 * ((args.prec + 31) // 32) + 5) / 1e9)}


class ClockSampler:
    """nvidia-smi clocks/throttle reasons during the timed region."""

    def __init__(self, index: int):
        self.index, self.rows, self.proc = index, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index),
                 "--query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm = [float(r[0]) for r in self.rows if r and r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if len(r) > 1 and r[1].replace(".", "").isdigit()]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            for k, name in enumerate(names):
                if len(r) > 4 + k and r[4 + k].lower() == "active":
                    reasons.add(name)
        sm_sorted = sorted(sm)
        return {"sm_mhz": sm_sorted[len(sm_sorted) // 2] if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


class _Soa:
    """Minimal ds SoA holder (limbs/exp/cls/count) for the CPU legs: they import
    nothing from the product package."""

    def __init__(self, limbs, exp, cls):
        self.limbs, self.exp, self.cls, self.count = limbs, exp, cls, limbs.shape[2]


def cpu_sample(n: int, p: int, rows: int, seed: int = 2000, ncomp: int = 1):
    """Pivot row + `rows` full-width rows at p bits in the ds SoA layout, drawn with
    numpy from the random_uniform family's distribution (genmat.py:242-246: sign
    uniform, |x| = U with a full p-bit mantissa).  MPFR's mul/sub cost at fixed p
    does not depend on the values, and this keeps the CPU legs free of the product's
    builders (the reference arm runs first, on a fresh box)."""
    import numpy as np
    L = (p + 31) // 32
    rng = np.random.default_rng(seed)
    out = []
    for count in (n, rows * n):
        limbs = rng.integers(0, 2 ** 32, size=(ncomp, L, count), dtype=np.uint32)
        zb = 32 * L - p
        if zb:
            limbs[:, zb // 32] &= np.uint32((0xFFFFFFFF << (zb % 32)) & 0xFFFFFFFF)
            limbs[:, :zb // 32] = 0
        limbs[:, L - 1] |= np.uint32(0x80000000)
        exp = (1 - rng.geometric(0.5, size=(ncomp, count))).astype(np.int32)
        cls = rng.integers(0, 2, size=(ncomp, count)).astype(np.uint8)
        out.append(_Soa(np.ascontiguousarray(limbs), np.ascontiguousarray(exp), np.ascontiguousarray(cls)))
    return out


def cpu_reference(n: int, p: int, seconds: float, kind: str = "real"):
    """Time the reference hot loop (oracle = elim.py:37-53 restated over MPFR) on a
    bounded sample of the workload: pivot step i applied to `rows` full-width rows,
    i = 0, 1, ... until ~`seconds` of timed MPFR work; all host threads."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle
    L = (p + 31) // 32
    threads = len(os.sched_getaffinity(0))
    rows_per_call = min(max(threads * 4, 64), n - 1)
    cx = kind == "complex"
    prow, rows = cpu_sample(n, p, rows_per_call, ncomp=2 if cx else 1)
    total_t, total_macs, calls, i = 0.0, 0.0, 0, 0
    while total_t < seconds and i < n - 1:
        # step i touches all n-1 columns of every sampled row (L and U slots)
        dt = oracle.time_apply_pivot_rows(n, p, kind, i, prow, rows, rows_per_call, threads, True)
        total_t += dt
        total_macs += rows_per_call * (n - 1)
        calls += 1
        i += 1
    rate = total_macs * L * L * (4 if cx else 1) / total_t
    return {"value": rate, "unit": "limb-MAC/s", "cores": threads, "kind": "port",
            "sample": f"{calls} pivot steps x {rows_per_call} full-width rows (n={n}, p={p}, {kind}, random_uniform "
                      f"distribution, numpy seed 2000), elim.py:37-53 restated over MPFR 4.2.1 / MPC 1.3.1 "
                      f"(oracle/ds_oracle.c), {total_macs:.3g} element MACs in {total_t:.2f}s on {threads} threads",
            "seconds_to_all_minors_extrapolated": work_limb_macs(n, L, cx) / rate}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    L = (args.prec + 31) // 32
    # timed MPFR seconds per step.  Every sampled pivot step also converts its rows into
    # MPFR values outside the timed region (measured: ~7x the timed seconds on the B200
    # box), so this keeps the whole --impl reference run to a few minutes
    per = max(2.0, min(args.cpu_seconds, 24.0 / max(1, args.steps + args.warmup)))
    desc = workload_desc(args)
    for _ in range(args.warmup):
        cpu_reference(args.n, args.prec, per / 4, kind_of(args))
    vals = []
    t0 = time.perf_counter()
    for _ in range(args.steps):
        vals.append(cpu_reference(args.n, args.prec, per, kind_of(args)))
    wall = time.perf_counter() - t0
    rate = sum(v["value"] for v in vals) / len(vals)
    base = vals[-1]
    out = {"metric": f"limb-MAC/s (schoolbook 32x32 limb products) of the all-minors elimination, "
                     f"N={args.n} @{args.prec}b",
           "value": rate, "unit": "limb-MAC/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
           "ms_per_step": wall / args.steps * 1e3, "higher_is_better": True, "scaling": "strong",
           "vs_baseline": None, "dtype": "mpfr (u64 limbs)",
           "data": "synthetic (random_uniform sample rows; MPFR cost is value-independent at fixed p)",
           "impl": "reference",
           "config": workload(args, desc),
           "seconds_to_all_minors": work_limb_macs(args.n, L, kind_of(args) == "complex") / rate,
           "cpu_baseline": {"value": rate, "unit": "limb-MAC/s", "cores": base["cores"], "kind": "port",
                            "sample": base["sample"]},
           "e2e": {"value": rate, "unit": "limb-MAC/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    emit_json(out)


def relaunch_under_torchrun(args) -> int:
    """`bench.py --gpus N` (N > 1) started as a plain process: re-exec under
    torch.distributed.run with N ranks (one per GPU), forwarding the JSON line."""
    import socket
    import torch
    if torch.cuda.device_count() < args.gpus:
        emit_json({"error": f"--gpus {args.gpus} needs {args.gpus} visible GPUs, found {torch.cuda.device_count()}",
                   "n_gpus": args.gpus})
        return 2
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(args.gpus),
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")  # NCCL's transport choice (NVLS / P2P) goes to the log
    r = subprocess.run(cmd, stdout=subprocess.PIPE, env=env, text=True)
    for line in r.stdout.splitlines():
        if line.startswith("{"):
            emit_json(json.loads(line))
    return r.returncode


def parity_leg(args, A, res, final, eng_factory):
    """Bit parity of THIS run against the oracle (tests/parity_check.py), outside every
    timed region: leading-steps state (a fresh device run of the first steps), the
    prefix property on the leading m x m block, and Laplace residuals."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import parity_check as pc
    from paper_1308_1536_b200.engine import HostResults
    t0 = time.perf_counter()
    n, p = args.n, args.prec
    out = {"checker": "oracle/ds_oracle.c (elim.py:37-229 over MPFR, pinned by tests/golden)"}
    head = 4 if p > 8192 else 8
    with eng_factory() as e2:
        e2.load(A)
        rh = HostResults.alloc(n, e2.ncomp, e2.L, False)
        e2.run(True, True, 0, head, rh)
        fh = A.copy()
        e2.fetch(fh)
    kind = kind_of(args)
    out["leading_steps"] = pc.leading_steps(A, n, p, kind, head, fh, rh)
    out["prefix"] = pc.prefix(A, n, p, kind, min(args.parity_m, n), res, final)
    sizes = sorted({n, n - 1, max(2, n // 2)})
    out["laplace"] = pc.laplace(A, n, p, res, sizes)
    out["ok"] = bool(out["leading_steps"]["ok"] and out["prefix"]["ok"])
    out["seconds"] = time.perf_counter() - t0
    return out


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch_under_torchrun(args))
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    local = local % max(1, torch.cuda.device_count())  # gloo test runs: ranks may share a GPU
    torch.cuda.set_device(local)
    dist = None
    use_dist = world > 1 or args.dist
    if use_dist:
        import torch.distributed as dist
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
        else:  # ranks sharing one GPU (tests): host-staged broadcasts
            dist.init_process_group("gloo")
    from paper_1308_1536_b200.engine import DeviceElimination, HostResults
    from paper_1308_1536_b200.soa import SoA

    n, p = args.n, args.prec
    L = (p + 31) // 32
    agree = None
    if use_dist:
        def agree(x: float) -> float:
            t = torch.tensor([x], dtype=torch.float64,
                             device=f"cuda:{local}" if args.dist_backend == "nccl" else "cpu")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            return float(t.item())
    A, desc, gen_s = build_input(args, pinned=True, rank=rank, world=world, agree=agree)  # this rank's rows
    kind = kind_of(args)
    nc = 2 if kind == "complex" else 1
    eng = DeviceElimination(n, p, kind, local, rank, world)
    # a dedicated stream (the legacy default stream's handle 0 would mean "own stream" to
    # ds_set_stream): kernels, NCCL broadcasts and the timing events share its order
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    pivot = None
    bcast, la_ok = None, True
    if use_dist:
        from paper_1308_1536_b200.parexec import dist_run
        _, pbytes = eng.pivot_buffer()
        pivot = torch.empty(pbytes, dtype=torch.uint8, device=f"cuda:{local}")
        eng.lib.ds_use_pivot_buffer(eng.ctx, pivot.data_ptr(), pbytes)
        if args.dist_backend == "nccl":
            bcast = lambda t, src: dist.broadcast(t, src=src)  # noqa: E731
        else:
            staging = {}
            la_ok = False

            def bcast(t, src):
                host = staging.get(t.numel())
                if host is None:
                    host = staging[t.numel()] = torch.empty(t.numel(), dtype=t.dtype, pin_memory=True)
                if rank == src:
                    host.copy_(t)
                dist.broadcast(host, src=src)
                if rank != src:
                    t.copy_(host)
    eng.lib.ds_set_stream(eng.ctx, stream.cuda_stream)
    # host buffers of this rank only: owned rows (count nloc * n) when sharded
    nloc = (n - rank + world - 1) // world
    res = HostResults.alloc(n, nc, L, True, pinned=True)
    if world > 1:
        res = HostResults(SoA(nc, L, n, pinned=True), SoA(nc, L, n, pinned=True), SoA(nc, L, nloc * n, pinned=True),
                          SoA(nc, L, nloc * n, pinned=True), res.row_flags)
    final = SoA(nc, L, nloc * n, pinned=True)

    def one_pass(resident: bool):
        if resident:
            eng.snapshot(False)
        else:
            eng.load(A)
        if not use_dist:
            if resident:
                eng.run_resident(True, True, 0, n)
            else:
                eng.run(True, True, 0, n, res)
                eng.fetch(final)  # the in-place L\\U state is part of the result (elim.py:19-22)
        else:
            dist_run(eng, n, True, True, pivot, bcast, lookahead=la_ok)
            if not resident:
                eng.results(n, res)
                eng.fetch(final)

    def barrier():
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x: float) -> float:
        if dist is None:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=f"cuda:{local}" if args.dist_backend == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def sum_over_ranks(x: float) -> float:
        if dist is None:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=f"cuda:{local}" if args.dist_backend == "nccl" else "cpu")
        dist.all_reduce(t)
        return float(t.item())

    eng.load(A)
    eng.snapshot(True)
    for _ in range(args.warmup):
        one_pass(True)
    barrier()
    # ---- timed: resident inputs (value), update kernel profiled live
    eng.profile(True)
    eng.profile_read()
    launches0 = eng.launches()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        barrier()
        ev0.record(stream)
        for _ in range(args.steps):
            one_pass(True)
        ev1.record(stream)
        barrier()
    ms = max_over_ranks(ev0.elapsed_time(ev1)) / args.steps
    upd_ms, upd_launches, upd_work = eng.profile_read()
    eng.profile(False)
    gpu_launches = eng.launches() - launches0
    total_work = work_limb_macs(n, L, kind == "complex")
    value = total_work / (ms / 1e3)
    # ---- timed: end to end through the C ABI with host buffers (pinned): H2D of the
    # matrix, the elimination, D2H of trace + minors (progressive) + final matrix
    e2e = None
    if not args.no_e2e:
        one_pass(False)
        barrier()
        c0 = eng.counters()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            one_pass(False)
        barrier()
        e2e_s = max_over_ranks(time.perf_counter() - t0) / args.steps
        c1 = eng.counters()
        h2d = sum_over_ranks(c1["h2d_bytes"] - c0["h2d_bytes"])  # whole job: every rank copies its own rows
        d2h = sum_over_ranks(c1["d2h_bytes"] - c0["d2h_bytes"])
        e2e = {"value": total_work / e2e_s, "unit": "limb-MAC/s",
               "h2d_bytes_per_step": int(h2d / args.steps),
               "d2h_bytes_per_step": int(d2h / args.steps),
               "bytes_counted_by": "ds_counters (every ABI host<->device copy of this context)",
               "seconds_to_all_minors": e2e_s,
               "includes": "H2D matrix, elimination, D2H pivots/dets/signed+normalized minors/final L\\U matrix"}
    # ---- roofline of the dominant kernel: the update (tensor-core engine)
    # algorithmic bytes per updated element: read + write a_jk (L limbs + exp + cls)
    cxw = 4 if kind == "complex" else 1  # component products per element
    elems = upd_work / (L * L * cxw) if L else 0.0
    upd_s = upd_ms / 1e3
    bytes_alg = elems * 2 * nc * (4 * L + 5)
    hbm_peak, peak_src = measured_hbm_peak()
    achieved_gbs = bytes_alg / upd_s / 1e9 if upd_s > 0 else 0.0
    counters = eng.counters()
    engine_name = ("k_prod_tcw x4 + k_tcw_finish_c (ds_tc.cu): complex component products on tcgen05 kind::i8 + "
                   "exact two-product sums and rounding" if kind == "complex" else
                   "k_update_tc (ds_tc.cu): tcgen05.mma kind::i8 digit products in TMEM + rounding epilogue"
                   if counters.get("tc_engine") else "k_fused (ds_update.cu): FP64 digit products + rounding epilogue")
    prof = committed_profile(n, p) if kind == "real" else None
    roof = {"kernel": engine_name, "bound": "hbm", "achieved": achieved_gbs, "peak": hbm_peak, "unit": "GB/s",
            "frac": achieved_gbs / hbm_peak if hbm_peak else None,
            "traffic": (prof["dram_bytes_per_element"] * elems / upd_launches) if prof and upd_launches else None,
            "traffic_per_element": prof.get("dram_bytes_per_element") if prof else None,
            "algorithmic_bytes_per_element": 2 * nc * (4 * L + 5),
            "elements_per_step": elems / args.steps if args.steps else None,
            "share_of_step": (upd_ms / args.steps) / ms if ms > 0 else None,
            "launches_per_step": upd_launches / args.steps,
            "limb_mac_rate": upd_work / upd_s if upd_s > 0 else None,
            "peak_source": peak_src,
            "limiter": prof.get("limiter") if prof else None,
            "issue_active_frac": prof.get("issue_active_frac") if prof else None,
            "tensor_pipe_frac": prof.get("tensor_pipe_frac") if prof else None,
            "ncu_source": prof.get("source") if prof else None,
            "tc_fallback_elements": counters.get("tc_fallback_elements"),
            "note": "achieved = algorithmic bytes (read+write of every updated a_jk) / summed update-kernel time "
                    "(CUDA events on the launch stream); bound = the HBM roof the kernel is measured against; "
                    "limiter / issue / tensor-pipe fractions from the committed ncu --set full capture"}
    parity = None
    if world == 1 and not args.no_parity and not args.no_e2e:
        try:
            parity = parity_leg(args, A, res, final, lambda: DeviceElimination(n, p, kind, local))
        except Exception as exc:  # reported, never hidden
            parity = {"ok": False, "error": repr(exc)}
    out = None
    if rank == 0:
        cpu = None
        if not args.no_cpu and world == 1:  # rank 0 at N=1 only
            try:
                cpu = cpu_reference(n, p, args.cpu_seconds, kind)
            except Exception as exc:  # never fail the GPU line on the baseline
                cpu = {"error": repr(exc)}
        out = {"metric": f"limb-MAC/s (schoolbook 32x32 limb products) of the all-minors elimination, N={n} @{p}b",
               "value": value, "unit": "limb-MAC/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
               "ms_per_step": ms, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
               "dtype": "u8 digit products (tcgen05 kind::i8, s32 accumulate) + u32 limbs",
               "data": {"random": "synthetic", "beta": "Artless beta matrix from data/ zeta zeros",
                        "power": "Artless zero-power matrix (complex) from data/ zeta zeros"}[args.family],
               "config": workload(args, desc), "seconds_to_all_minors": ms / 1e3,
               "input_generation_s": gen_s,
               "e2e": e2e, "roofline": roof, "parity": parity, "cpu_baseline": cpu, "gpu_launches": gpu_launches,
               "clocks": clk.summary(), "parallelism": f"row-cyclic x{world}"}
        emit_json(out)
    eng.close()
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


_JSON_FD = None


def emit_json(obj):
    """The one JSON line, on the process's original stdout."""
    line = (json.dumps(obj) + "\n").encode()
    if _JSON_FD is not None:
        os.write(_JSON_FD, line)
    else:
        sys.stdout.write(line.decode())
        sys.stdout.flush()


if __name__ == "__main__":
    # libraries (NCCL's version banner, CUDA/torch notices) print to fd 1: route
    # everything but the result line to stderr so stdout carries exactly one JSON line
    sys.stdout.flush()
    _JSON_FD = os.dup(1)
    os.dup2(2, 1)
    main()
