"""Phase breakdown of the drop-in eliminate() path (tools/dropin_e2e.py measures the
total): engine creation, H2D load, the streamed run (callback copying rows out of the
staging), trace fetch, state fetch, and the scalar conversion of the streamed rows --
each timed on its own, twice (cold and warm).

usage: python tools/dropin_phases.py [N] [BITS]"""
import json
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_1308_1536_b200 import MatrixBuffer, Precision, eliminate  # noqa: E402
from paper_1308_1536_b200.elim import _stream_batch  # noqa: E402
from paper_1308_1536_b200.hostgen import RowQueue  # noqa: E402
from paper_1308_1536_b200.engine import DeviceElimination, HostResults  # noqa: E402
from paper_1308_1536_b200.soa import paused_gc  # noqa: E402
from paper_1308_1536_b200.synth import random_uniform_soa  # noqa: E402


def phases(n, p, soa):
    t = {}
    c0 = time.perf_counter()
    eng = DeviceElimination(n, p, "real", 0)
    t["create"] = time.perf_counter() - c0
    c0 = time.perf_counter()
    eng.load(soa)
    t["load_h2d"] = time.perf_counter() - c0
    res = HostResults.alloc(n, eng.ncomp, eng.L, False)
    q = RowQueue(n, 1, eng.L, p)
    c0 = time.perf_counter()
    eng.stream_minors_native(_stream_batch(n), q.cb_ptr, q.q)
    t["stream_setup"] = time.perf_counter() - c0
    c0 = time.perf_counter()
    rc, d = eng.run(True, True, 0, n, res)
    t["run_streamed_native_structs"] = time.perf_counter() - c0
    c0 = time.perf_counter()
    eng.fetch(soa)
    t["fetch_d2h"] = time.perf_counter() - c0
    c0 = time.perf_counter()
    eng.close()
    t["close"] = time.perf_counter() - c0
    q.close()
    c0 = time.perf_counter()
    k = 0
    with paused_gc():
        while True:
            b = q.pop_rows()
            if b is None:
                break
            k += len(b)
    t["wrap_rows"] = time.perf_counter() - c0
    t["rows"] = k
    return t


def timeline(n, p, soa, nthreads=0):
    """eliminate()'s structure with timestamps: worker (stream run, fetch, close) against
    the caller's wrapping of each popped batch."""
    import threading
    ev = []
    T0 = time.perf_counter()

    def mark(what):
        ev.append((round(time.perf_counter() - T0, 4), what))

    eng = DeviceElimination(n, p, "real", 0)
    eng.load(soa)
    mark("loaded")
    res = HostResults.alloc(n, eng.ncomp, eng.L, False)
    q = RowQueue(n, 1, eng.L, p, nthreads)

    def work():
        eng.stream_minors_native(_stream_batch(n), q.cb_ptr, q.q)
        mark("stream set")
        eng.run(True, True, 0, n, res)
        mark("run done")
        eng.fetch(soa)
        mark("fetched")
        q.close()
        eng.close()
        mark("closed")

    th = threading.Thread(target=work)
    th.start()
    wrap = 0.0
    nb = 0
    first = None
    with paused_gc():
        while True:
            b = q.pop_rows.__self__.lib.dsh_rowq_pop  # noqa: F841  (keep the attribute hot)
            a = time.perf_counter()
            rows = q.pop_rows()
            w = time.perf_counter()
            if rows is None:
                break
            if first is None:
                first = round(a - T0, 4)
                mark("first batch popped")
            wrap += w - a
            nb += 1
    mark("main drained")
    th.join()
    mark("joined")
    return {"n": n, "nthreads": nthreads, "batches": nb, "pop_plus_wrap_s": round(wrap, 3), "events": ev}


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
    p = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
    torch.cuda.synchronize()
    for rep in range(2):
        soa = random_uniform_soa(n, p, seed=n)
        print(json.dumps({"n": n, "prec_bits": p, "rep": rep, **phases(n, p, soa)}))
    for nt in (0, 4):
        soa = random_uniform_soa(n, p, seed=n)
        print(json.dumps(timeline(n, p, soa, nt)))
    for rep in range(2):
        soa = random_uniform_soa(n, p, seed=n)
        A = MatrixBuffer.from_soa(n, "real", Precision(p), soa)
        rows = []
        c0 = time.perf_counter()
        eliminate(A, sink=rows.append)
        print(json.dumps({"n": n, "prec_bits": p, "rep": rep, "eliminate_s": time.perf_counter() - c0}))


if __name__ == "__main__":
    main()
