"""Native minors-stream consumer (csrc/hoststream.c, hostgen.RowQueue) on the CPU: the
callback is driven directly with staging SoAs laid out like ds_stream_minors delivers
them (include/detseries_b200.h ds_rows_cb), and the popped scalars must equal the
element-wise conversion of the same limbs."""
import ctypes
import threading

import numpy as np
import pytest

from paper_1308_1536_b200 import _native
from paper_1308_1536_b200.hostgen import RowQueue
from paper_1308_1536_b200.scalars import canonical_bits
from paper_1308_1536_b200.soa import SoA
from paper_1308_1536_b200.synth import random_uniform_soa

CB = ctypes.CFUNCTYPE(None, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.POINTER(_native.ds_soa),
                      ctypes.POINTER(_native.ds_soa), ctypes.POINTER(ctypes.c_uint8), ctypes.c_void_p)


def _staging(n, p, cap, ncomp, seed):
    side = int(np.ceil(np.sqrt(cap * n))) + 1  # random_uniform_soa(k) gives k*k elements
    base = random_uniform_soa(side, p, seed=seed)
    if ncomp == 2:
        im = random_uniform_soa(side, p, seed=seed + 1)
        base = SoA(2, base.L, base.count, np.concatenate([base.limbs, im.limbs]), np.concatenate([base.exp, im.exp]),
                   np.concatenate([base.cls, im.cls]))
    base.cls[:, ::7] = 2  # some +0
    base.cls[:, 3::11] = 3  # some -0
    return base


@pytest.mark.parametrize("p,ncomp,stride", [(256, 1, 1), (4096, 1, 1), (1000, 1, 3), (333, 2, 1), (64, 1, 2)])
def test_rowq_matches_elementwise(p, ncomp, stride):
    n, cap, g0, nrows = 40, 6, 5, 5
    sg = _staging(n, p, cap, ncomp, 11)
    nm = _staging(n, p, cap, ncomp, 23)
    flags = np.array([3, 1, 0, 3, 3], dtype=np.uint8)
    q = RowQueue(n, ncomp, sg.L, p)
    cb = CB(q.cb_ptr)
    cb(g0, stride, nrows, ctypes.byref(sg.c()), ctypes.byref(nm.c()),
       flags.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8)), ctypes.c_void_p(q.q))
    q.close()
    rows = q.pop_rows()
    assert q.pop_rows() is None
    want_m = [g0 + r * stride + 1 for r in range(nrows) if flags[r] & 1]
    assert [m for m, _, _ in rows] == want_m
    for m, s, z in rows:
        r = (m - 1 - g0) // stride
        assert len(s) == m
        assert [canonical_bits(x) for x in s] == [sg.canonical(r * n + k, p) for k in range(m)]
        if flags[r] & 2:
            assert [canonical_bits(x) for x in z] == [nm.canonical(r * n + k, p) for k in range(m)]
        else:
            assert z is None
    # the scalars outlive the queue and the staging
    del q, sg
    assert rows[-1][1][0] == rows[-1][1][0]


def test_rowq_pop_blocks_until_close():
    q = RowQueue(8, 1, 2, 64)
    got = []
    t = threading.Thread(target=lambda: got.append(q.pop_rows()))
    t.start()
    t.join(0.2)
    assert t.is_alive()
    q.close()
    t.join(5)
    assert got == [None]
