"""The drop-in Python entry points on the device, against the reference goldens.

`eliminate` (elim.py:158-229) with minors, `sink` order, `series=False`,
`collect_minors=False`, `step_hook` (stop + lazy A), `ZeroPivot` partials and
resume (`trace` / `start_step`), and `par_eliminate` (parexec.py:408-424)
with transport="local" for T in {1, 2, 3, 4, 8} virtual shards (criterion 5,
test_acceptance.py:143-159: bit-identical for every T, `broadcasts == n`).
Every check compares the digest of canonical_bits of the returned objects and
of the in-place buffer with the digest the unmodified reference produced.
"""
import pytest

from _util import build_input, load_golden
from golden.digest import digest_parts
from paper_1308_1536_b200 import MatrixBuffer, Precision, ZeroPivot, eliminate, par_eliminate
from paper_1308_1536_b200.elim import EliminationTrace, MinorSeries
from paper_1308_1536_b200.scalars import canonical_bits

pytestmark = pytest.mark.gpu


def _buffer(name):
    meta, arrays = load_golden(name)
    A = MatrixBuffer.from_soa(meta["n"], meta["kind"], Precision(meta["prec"]), build_input(meta, arrays))
    return meta, A


def _digest(trace, minors, A):
    rows = []
    if minors is not None:
        for m in minors.sizes():
            r = minors.rows[m]
            rows.append((m, [canonical_bits(x) for x in r.signed],
                         None if r.normalized is None else [canonical_bits(x) for x in r.normalized]))
    return digest_parts([canonical_bits(x) for x in trace.pivots], [canonical_bits(x) for x in trace.det_series],
                        rows, [canonical_bits(x) for row in A.rows for x in row])


def _run(A, meta, **kw):
    try:
        trace, minors = eliminate(A, collect_minors=meta["collect_minors"], series=meta["series"], **kw)
    except ZeroPivot as exc:
        assert meta["zero_pivot_step"] == exc.step
        assert exc.trace.step == exc.step - 1
        trace, minors = exc.trace, exc.series
    return trace, minors


@pytest.mark.parametrize("name", ["worked_2x2", "worked_3x3", "identity3", "zero_pivot3", "int7_s3", "rational_s1",
                                  "hilbert12_p100", "uniform24_s2_p4096", "series_false_u6", "nominors_u9_p320",
                                  "complex8_s9_p192", "complex_int6", "uniform128_s7_p1024", "beta64_p256"])
def test_eliminate_dropin(name):
    meta, A = _buffer(name)
    trace, minors = _run(A, meta)
    assert _digest(trace, minors, A) == meta["digest"]


@pytest.mark.parametrize("name", ["uniform128_s7_p1024", "zero_pivot3", "series_false_u6", "complex8_s9_p192"])
def test_sink_order(name):
    """sink receives every MinorRow exactly once, in increasing n (test_parexec.py:187-191)."""
    meta, A = _buffer(name)
    got = []
    trace, minors = _run(A, meta, sink=got.append)
    assert minors is None or not minors.rows  # rows went to the sink
    assert [r.n for r in got] == sorted(r.n for r in got)
    series = MinorSeries(A.prec)
    for r in got:
        series.add(r)
    assert _digest(trace, series if meta["collect_minors"] else None, A) == meta["digest"]
    assert [r.n for r in got] == meta["emitted"]


@pytest.mark.parametrize("name,stop", [("uniform128_s7_p1024", 37), ("complex8_s9_p192", 3),
                                       ("uniform24_s2_p4096", 10)])
def test_step_hook_stop_and_resume(name, stop):
    """step_hook(i, A, trace) after every step; returning True stops the run with A holding the
    mid-elimination state; resuming with trace/start_step (cli.py:194-206) ends bit-identical."""
    meta, A = _buffer(name)
    seen = []

    def hook(done, buf, tr):
        seen.append((done, len(tr.pivots)))
        return done == stop

    got = []
    trace, _ = eliminate(A, collect_minors=True, sink=got.append, step_hook=hook)
    assert trace.step == stop and seen == [(k, k) for k in range(1, stop + 1)]
    # the lazily materialised buffer is the reference's mid-run state: resume from it
    A2 = MatrixBuffer(A.n, A.kind, A.prec, [list(r) for r in A.rows])
    trace2 = EliminationTrace(n=A.n, prec=A.prec, pivots=list(trace.pivots), det_series=list(trace.det_series),
                              step=trace.step)
    trace3, _ = eliminate(A2, collect_minors=True, sink=got.append, trace=trace2, start_step=stop)
    series = MinorSeries(A.prec)
    for r in got:
        series.add(r)
    assert [r.n for r in got] == list(range(2, A.n + 1))
    assert _digest(trace3, series, A2) == meta["digest"]


def test_step_hook_checkpoint_save_matches_materialised(tmp_path):
    """A hook that saves the buffer (the reference CLI checkpointer, cli.py:108-118) writes the
    same MPMAT bytes whether the buffer is saved natively from the device copy or materialised."""
    meta, A = _buffer("uniform13_s5_p192")

    def hook(done, buf, tr):
        if done == 5:
            buf.save(str(tmp_path / "fast.mpmat"))
            rows = [list(r) for r in buf.rows]  # materialise
            MatrixBuffer(buf.n, buf.kind, buf.prec, rows).save(str(tmp_path / "slow.mpmat"))
        return False

    trace, minors = eliminate(A, step_hook=hook)
    assert (tmp_path / "fast.mpmat").read_bytes() == (tmp_path / "slow.mpmat").read_bytes()
    assert _digest(trace, minors, A) == meta["digest"]


@pytest.mark.parametrize("workers", [1, 2, 3, 4, 8])
def test_par_eliminate_local_criterion5(workers):
    """Criterion 5 (test_acceptance.py:143-159): N=128 @1024 seed 7, bit-identical for T in {1,2,4,8}
    (and 3), one broadcast per step."""
    meta, A = _buffer("uniform128_s7_p1024")
    trace, minors, stats = par_eliminate(A, workers, transport="local")
    assert stats.broadcasts == A.n
    assert _digest(trace, minors, A) == meta["digest"]


@pytest.mark.parametrize("name,workers", [("complex8_s9_p192", 3), ("zero_pivot3", 2), ("beta64_p256", 4),
                                          ("uniform24_s2_p4096", 8), ("nominors_u9_p320", 2)])
def test_par_eliminate_local_goldens(name, workers):
    meta, A = _buffer(name)
    try:
        trace, minors, stats = par_eliminate(A, workers, transport="local", collect_minors=meta["collect_minors"],
                                             series=meta["series"])
    except ZeroPivot as exc:
        assert exc.step == meta["zero_pivot_step"]
        trace, minors = exc.trace, exc.series
    assert _digest(trace, minors, A) == meta["digest"]


def test_par_eliminate_sink_order():
    meta, A = _buffer("uniform30_s4_p256")
    got = []
    par_eliminate(A, 3, transport="local", sink=got.append)
    assert [r.n for r in got] == list(range(2, A.n + 1))


@pytest.mark.parametrize("name,workers", [("uniform30_s4_p256", 2), ("complex8_s9_p192", 3), ("zero_pivot3", 2)])
def test_par_eliminate_process_spawns_its_own_ranks(name, workers):
    """transport="process" from a plain process forks the worker ranks itself (ref
    parexec.py:350-405); with fewer GPUs than ranks they share the GPU and broadcast over gloo
    through a pinned staging copy."""
    meta, A = _buffer(name)
    try:
        trace, minors, stats = par_eliminate(A, workers, transport="process")
        assert stats.broadcasts == A.n
    except ZeroPivot as exc:
        assert exc.step == meta["zero_pivot_step"]
        trace, minors = exc.trace, exc.series
    assert _digest(trace, minors, A) == meta["digest"]


def test_owned_rows_only_host_buffers():
    """ds_load / ds_fetch / ds_results_fetch with owned-rows-only host buffers (count nloc*n):
    three virtual shards driven step by step give the serial engine's bits."""
    import ctypes

    import numpy as np

    from paper_1308_1536_b200.engine import DeviceElimination, HostResults
    from paper_1308_1536_b200.soa import SoA
    from paper_1308_1536_b200.synth import random_uniform_soa
    n, p, world = 150, 1024, 3
    A = random_uniform_soa(n, p, seed=5)
    with DeviceElimination(n, p, "real") as e:
        e.load(A)
        ref = HostResults.alloc(n, 1, e.L, True)
        e.run(True, True, 0, n, ref)
        fin_ref = A.copy()
        e.fetch(fin_ref)
    L = (p + 31) // 32
    ranks = [DeviceElimination(n, p, "real", 0, r, world) for r in range(world)]
    try:
        for r, e in enumerate(ranks):
            rows = np.arange(r, n, world)
            own = SoA(1, L, len(rows) * n,
                      np.ascontiguousarray(A.limbs.reshape(1, L, n, n)[:, :, rows, :].reshape(1, L, -1)),
                      np.ascontiguousarray(A.exp.reshape(1, n, n)[:, rows, :].reshape(1, -1)),
                      np.ascontiguousarray(A.cls.reshape(1, n, n)[:, rows, :].reshape(1, -1)))
            e.load(own)
        for i in range(n):
            owner = ranks[i % world]
            owner.stage(i)
            for e in ranks:
                if e is not owner:
                    assert e.lib.ds_pivot_copy(e.ctx, owner.ctx) == 0
            for e in ranks:
                e.step(i, True, True)
        for r, e in enumerate(ranks):
            rows = np.arange(r, n, world)
            nloc = len(rows)
            fin = SoA(1, L, nloc * n)
            e.fetch(fin)
            res = HostResults(SoA(1, L, n), SoA(1, L, n), SoA(1, L, nloc * n), SoA(1, L, nloc * n),
                              np.zeros(n, dtype=np.uint8))
            e.results(n, res)
            assert np.array_equal(fin.limbs.reshape(1, L, nloc, n), fin_ref.limbs.reshape(1, L, n, n)[:, :, rows])
            assert np.array_equal(fin.exp.reshape(1, nloc, n), fin_ref.exp.reshape(1, n, n)[:, rows])
            assert np.array_equal(res.dets.limbs, ref.dets.limbs)
            for jl, g in enumerate(rows):
                m = g + 1
                if m < 2:
                    continue
                sl = slice(jl * n, jl * n + m)
                gl = slice(g * n, g * n + m)
                assert res.row_flags[g] == ref.row_flags[g]
                assert np.array_equal(res.signed.limbs[:, :, sl], ref.signed.limbs[:, :, gl])
                assert np.array_equal(res.normalized.exp[:, sl], ref.normalized.exp[:, gl])
            c = e.counters()
            assert c["h2d_bytes"] == nloc * n * (4 * L + 5)
    finally:
        for e in ranks:
            e.close()
