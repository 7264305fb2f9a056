"""Panel-paged (out-of-core) executor (paged.py, ds_create_block /
ds_pivot_load): panels of consecutive rows brought up to date left-looking
from final pivot rows on the host give the in-core bits -- final L\\U state,
trace and every minors row -- for real and complex matrices, with the store
in RAM or in a disk-backed memmap, and through the MatrixBuffer drop-in
against the reference goldens."""
import numpy as np
import pytest

from _util import build_input, load_golden
from golden.digest import digest_parts
from paper_1308_1536_b200 import MatrixBuffer, Precision, ZeroPivot
from paper_1308_1536_b200.engine import DeviceElimination, HostResults
from paper_1308_1536_b200.paged import paged_eliminate, paged_eliminate_soa
from paper_1308_1536_b200.scalars import canonical_bits
from paper_1308_1536_b200.soa import SoA
from paper_1308_1536_b200.synth import random_uniform_soa

pytestmark = pytest.mark.gpu


def _in_core(A, n, p, kind):
    with DeviceElimination(n, p, kind) as e:
        e.load(A)
        res = HostResults.alloc(n, e.ncomp, e.L, True)
        rc, done = e.run(True, True, 0, n, res)
        fin = A.copy()
        e.fetch(fin)
    return res, fin, done


def _same(a: SoA, b: SoA):
    return np.array_equal(a.limbs, b.limbs) and np.array_equal(a.exp, b.exp) and np.array_equal(a.cls, b.cls)


@pytest.mark.parametrize("n,p,kind,panel", [(150, 1024, "real", 40), (131, 4096, "real", 64), (90, 333, "real", 1),
                                            (40, 256, "complex", 7), (24, 33220, "real", 10)])
def test_paged_matches_in_core(n, p, kind, panel):
    A = random_uniform_soa(n, p, seed=n + p, kind=kind)
    res, fin, done = _in_core(A, n, p, kind)
    store = A.copy()
    pres, pdone = paged_eliminate_soa(store, n, p, kind, panel)
    assert pdone == done == n
    assert _same(store, fin)
    assert _same(pres.pivots, res.pivots) and _same(pres.dets, res.dets)
    assert np.array_equal(pres.row_flags, res.row_flags)
    for m in range(2, n + 1):
        sl = slice((m - 1) * n, (m - 1) * n + m)
        assert np.array_equal(pres.signed.limbs[:, :, sl], res.signed.limbs[:, :, sl]), m
        assert np.array_equal(pres.normalized.exp[:, sl], res.normalized.exp[:, sl]), m


def test_paged_store_on_disk(tmp_path):
    """The host store is a disk-backed numpy memmap: only one panel is in memory at a time."""
    n, p = 100, 1024
    A = random_uniform_soa(n, p, seed=3)
    res, fin, _ = _in_core(A, n, p, "real")
    mm = lambda name, arr: np.lib.format.open_memmap(str(tmp_path / name), mode="w+", dtype=arr.dtype,  # noqa: E731
                                                     shape=arr.shape)
    limbs, ex, cl = mm("l.npy", A.limbs), mm("e.npy", A.exp), mm("c.npy", A.cls)
    limbs[...] = A.limbs
    ex[...] = A.exp
    cl[...] = A.cls
    store = SoA(1, A.L, n * n, limbs, ex, cl)
    pres, done = paged_eliminate_soa(store, n, p, "real", 30)
    limbs.flush()
    assert _same(SoA(1, A.L, n * n, np.asarray(limbs), np.asarray(ex), np.asarray(cl)), fin)
    assert _same(pres.dets, res.dets)


@pytest.mark.parametrize("name,panel", [("uniform128_s7_p1024", 50), ("complex8_s9_p192", 3), ("zero_pivot3", 1),
                                        ("beta64_p256", 16)])
def test_paged_dropin_matches_reference_goldens(name, panel):
    meta, arrays = load_golden(name)
    A = MatrixBuffer.from_soa(meta["n"], meta["kind"], Precision(meta["prec"]), build_input(meta, arrays))
    try:
        trace, minors = paged_eliminate(A, panel, collect_minors=meta["collect_minors"], series=meta["series"])
    except ZeroPivot as exc:
        assert exc.step == meta["zero_pivot_step"]
        trace, minors = exc.trace, exc.series
    rows = []
    if minors is not None:
        for m in minors.sizes():
            r = minors.rows[m]
            rows.append((m, [canonical_bits(x) for x in r.signed],
                         None if r.normalized is None else [canonical_bits(x) for x in r.normalized]))
    dig = digest_parts([canonical_bits(x) for x in trace.pivots], [canonical_bits(x) for x in trace.det_series], rows,
                       [canonical_bits(x) for row in A.rows for x in row])
    assert dig == meta["digest"]
