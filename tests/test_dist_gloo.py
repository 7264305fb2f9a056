"""Multi-process (gloo, world_size 2 and 3) run of the sharded executor's
host logic -- paper_1308_1536_b200.parexec.dist_run (per-step owner staging +
broadcast of the pivot buffer + per-rank step) and allreduce_gather (reassembly
of minors rows and matrix rows) -- with the CPU oracle as each rank's engine.
The reassembled trace / minors / final buffer must be bit-identical to the
reference goldens (parexec.py:3-8: identical for every worker count)."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as tmp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, name, out_dir):
    import sys
    for p in (ROOT, os.path.join(ROOT, "tests"), os.path.join(ROOT, "oracle")):
        sys.path.insert(0, p)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    from _util import build_input, load_golden, results_digest
    from paper_1308_1536_b200.engine import HostResults
    from paper_1308_1536_b200.parexec import CommStats, allreduce_gather, dist_run

    meta, arrays = load_golden(name)
    A = build_input(meta, arrays)
    n, p, kind = meta["n"], meta["prec"], meta["kind"]
    eng = oracle.OracleRank(n, p, kind, rank, world, 1)
    eng.load(A)
    pivot = torch.from_numpy(eng.pivot_array())  # shares the oracle's buffer
    stats = CommStats()
    failed = dist_run(eng, n, meta["collect_minors"], meta["series"], pivot,
                      lambda t, src: dist.broadcast(t, src=src), stats)
    done = failed if failed >= 0 else n
    res = HostResults.alloc(n, eng.ncomp, eng.L, meta["collect_minors"])
    eng.results(done, res)
    final = A.copy()
    eng.fetch(final)

    def allreduce(arr):
        t = torch.from_numpy(arr)
        dist.all_reduce(t)

    allreduce_gather(res, final, rank, world, allreduce)
    dig = results_digest(res, final, n, p, done)
    with open(os.path.join(out_dir, f"r{rank}.txt"), "w") as f:
        f.write(f"{dig} {done} {stats.broadcasts}\n")
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("name,world", [("uniform13_s5_p192", 2), ("uniform13_s5_p192", 3),
                                        ("complex8_s9_p192", 2), ("zero_pivot3", 2), ("int7_s1", 3),
                                        ("nominors_u9_p320", 2)])
def test_gloo_sharded_matches_reference(name, world, tmp_path):
    import sys
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from _util import load_golden
    meta, _ = load_golden(name)
    tmp.spawn(_worker, args=(world, _free_port(), name, str(tmp_path)), nprocs=world, join=True)
    for r in range(world):
        dig, done, bcast = open(tmp_path / f"r{r}.txt").read().split()
        assert dig == meta["digest"], (r, dig)
        assert int(bcast) == meta["n"]  # one broadcast per step (test_acceptance.py:157)
        if meta["zero_pivot_step"] is not None:
            assert int(done) + 1 == meta["zero_pivot_step"]


@pytest.mark.parametrize("name,world", [("uniform13_s5_p192", 2), ("complex8_s9_p192", 3), ("zero_pivot3", 2),
                                        ("nominors_u9_p320", 2), ("series_false_u6", 3)])
def test_spawned_process_transport_matches_reference(name, world):
    """par_eliminate(transport="process") from a plain process forks its own ranks (ref
    parexec.py:350-405), rendezvous over TCP, broadcasts per step over gloo and reassembles
    the owned rows into the caller's buffer -- oracle engines stand in for the GPUs here."""
    import sys
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import _oracle_engine
    from _util import build_input, load_golden
    from golden.digest import digest_parts
    from paper_1308_1536_b200 import MatrixBuffer, Precision, ZeroPivot, par_eliminate
    from paper_1308_1536_b200.scalars import canonical_bits
    meta, arrays = load_golden(name)
    A = MatrixBuffer.from_soa(meta["n"], meta["kind"], Precision(meta["prec"]), build_input(meta, arrays))
    got = []
    try:
        trace, minors, stats = par_eliminate(A, world, transport="process", collect_minors=meta["collect_minors"],
                                             series=meta["series"], sink=got.append,
                                             _engine_factory=_oracle_engine.make)
        assert stats.broadcasts == meta["n"]
    except ZeroPivot as exc:
        assert exc.step == meta["zero_pivot_step"]
        trace = exc.trace
    rows = [(r.n, [canonical_bits(x) for x in r.signed],
             None if r.normalized is None else [canonical_bits(x) for x in r.normalized]) for r in got]
    assert [r[0] for r in rows] == meta["emitted"]
    dig = digest_parts([canonical_bits(x) for x in trace.pivots], [canonical_bits(x) for x in trace.det_series],
                       rows, [canonical_bits(x) for row in A.rows for x in row])
    assert dig == meta["digest"]


def _dying_engine(n, p, kind, rank, world):
    """Engine factory whose rank 1 fails at creation (tests the coordinator's failure path)."""
    if rank == 1:
        raise RuntimeError("injected worker failure")
    import oracle
    return oracle.OracleRank(n, p, kind, rank, world, 1)


def test_spawned_process_transport_worker_failure():
    """A rank that dies raises WorkerFailure in the caller and the surviving ranks are stopped
    instead of waiting in a collective forever (ref parexec.py:395-405 raises WorkerFailure)."""
    import sys
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from _util import build_input, load_golden
    from paper_1308_1536_b200 import MatrixBuffer, Precision, par_eliminate
    from paper_1308_1536_b200.errors import WorkerFailure
    from test_dist_gloo import _dying_engine
    meta, arrays = load_golden("uniform13_s5_p192")
    A = MatrixBuffer.from_soa(meta["n"], meta["kind"], Precision(meta["prec"]), build_input(meta, arrays))
    with pytest.raises(WorkerFailure):
        par_eliminate(A, 2, transport="process", _engine_factory=_dying_engine)
