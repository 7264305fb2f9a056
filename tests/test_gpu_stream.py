"""Streaming of the minors rows off the device (ds_stream_minors /
ds_stream_flush): only a ring of rows stays in HBM, rows reach the host
consumer in increasing size, and every streamed row is bit-identical to the
resident run's.  Serial (ds_run flushes) and sharded (the driver flushes)."""
import numpy as np
import pytest

from _util import build_input, load_golden
from paper_1308_1536_b200.engine import DeviceElimination, HostResults
from paper_1308_1536_b200.output import MinorsStream, read_minors_binary
from paper_1308_1536_b200.synth import random_uniform_soa

pytestmark = pytest.mark.gpu


def _resident(A, n, p, kind):
    with DeviceElimination(n, p, kind) as e:
        e.load(A)
        res = HostResults.alloc(n, e.ncomp, e.L, True)
        rc, done = e.run(True, True, 0, n, res)
        fin = A.copy()
        e.fetch(fin)
    return res, fin, done


def _same_rows(stream: MinorsStream, res: HostResults, n: int, upto: int):
    assert stream.sizes == [m for m in range(2, upto + 1) if res.row_flags[m - 1] & 1]
    for m in stream.sizes:
        fl, sg, nm = stream.kept[m]
        assert fl == res.row_flags[m - 1]
        sl = slice((m - 1) * n, (m - 1) * n + m)
        assert np.array_equal(sg.limbs, res.signed.limbs[:, :, sl]), m
        assert np.array_equal(sg.exp, res.signed.exp[:, sl]) and np.array_equal(sg.cls, res.signed.cls[:, sl]), m
        if fl & 2:
            assert np.array_equal(nm.limbs, res.normalized.limbs[:, :, sl]), m
            assert np.array_equal(nm.exp, res.normalized.exp[:, sl]), m


@pytest.mark.parametrize("n,p,kind,batch", [(300, 1024, "real", 16), (150, 4096, "real", 5), (40, 256, "complex", 4),
                                            (96, 33220, "real", 8)])
def test_serial_stream_matches_resident(n, p, kind, batch, tmp_path):
    A = random_uniform_soa(n, p, seed=n + p, kind=kind)
    res, fin, _ = _resident(A, n, p, kind)
    path = tmp_path / "minors.dsmr"
    st = MinorsStream(n, p, kind, path=str(path), keep_upto=n)
    with DeviceElimination(n, p, kind) as e:
        e.stream_minors(batch, st)
        e.load(A)
        tr = HostResults.alloc(n, e.ncomp, e.L, False)
        rc, done = e.run(True, True, 0, n, tr)
        fin_s = A.copy()
        e.fetch(fin_s)
    st.close()
    assert done == n
    assert np.array_equal(fin_s.limbs, fin.limbs) and np.array_equal(tr.dets.limbs, res.dets.limbs)
    _same_rows(st, res, n, n)
    got = [(m, fl) for m, fl, _, _ in read_minors_binary(str(path))]
    assert got == [(m, int(res.row_flags[m - 1])) for m in range(2, n + 1)]


def test_serial_stream_zero_pivot():
    meta, arrays = load_golden("zero_pivot3")
    A = build_input(meta, arrays)
    n, p = meta["n"], meta["prec"]
    res, fin, done = _resident(A, n, p, meta["kind"])
    st = MinorsStream(n, p, meta["kind"], keep_upto=n)
    with DeviceElimination(n, p, meta["kind"]) as e:
        e.stream_minors(1, st)
        e.load(A)
        rc, d2 = e.run(True, True, 0, n, None)
    assert d2 == done == meta["zero_pivot_step"] - 1
    _same_rows(st, res, n, done + 1)


@pytest.mark.parametrize("world,batch", [(3, 8), (4, 16)])
def test_sharded_stream_matches_resident(world, batch):
    n, p = 200, 1024
    A = random_uniform_soa(n, p, seed=7)
    res, fin, _ = _resident(A, n, p, "real")
    ranks = [DeviceElimination(n, p, "real", 0, r, world) for r in range(world)]
    streams = [MinorsStream(n, p, "real", keep_upto=n) for _ in range(world)]
    try:
        for e, st in zip(ranks, streams):
            e.stream_minors(batch, st)
            e.load(A)
        for i in range(n):
            owner = ranks[i % world]
            owner.stage(i)
            for e in ranks:
                if e is not owner:
                    assert e.lib.ds_pivot_copy(e.ctx, owner.ctx) == 0
            for e in ranks:
                e.step(i, True, True)
            if (i + 1) % batch == 0:
                for e in ranks:
                    e.stream_flush(i + 1)
        for e in ranks:
            e.stream_flush(n, final=True)
    finally:
        for e in ranks:
            e.close()
    merged = MinorsStream(n, p, "real", keep_upto=n)
    for r, st in enumerate(streams):
        assert all((m - 1) % world == r for m in st.sizes)
        assert st.sizes == sorted(st.sizes)
        merged.kept.update(st.kept)
    merged.sizes = sorted(merged.kept)
    _same_rows(merged, res, n, n)
