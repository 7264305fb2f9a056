"""Small elimination cases for compute-sanitizer (memcheck / racecheck / synccheck):
the fused tensor-core update (k_update_tc: TMA tiles, mbarriers, TMEM) and the
wide engine (k_prod_tcw + k_tcw_finish), a few steps each, checked against the
oracle so a sanitizer run also proves the instrumented kernels still compute
the same bits.   usage: compute-sanitizer --tool racecheck python tools/sanitize_case.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "tests"), os.path.join(ROOT, "oracle")):
    sys.path.insert(0, p)

import oracle  # noqa: E402
from paper_1308_1536_b200.engine import DeviceElimination, HostResults  # noqa: E402
from paper_1308_1536_b200.synth import random_uniform_soa  # noqa: E402

cases = [(140, 1024, 3), (132, 4096, 2), (40, 16384, 2)]
for n, p, steps in cases:
    A = random_uniform_soa(n, p, seed=n)
    with DeviceElimination(n, p, "real") as e:
        e.load(A)
        res = HostResults.alloc(n, 1, e.L, True)
        e.run(True, True, 0, steps, res)
        fin = A.copy()
        e.fetch(fin)
        c = e.counters()
    r = oracle.OracleRank(n, p, "real")
    r.load(A)
    r.run(True, True, 0, steps)
    fo = A.copy()
    r.fetch(fo)
    same = (fo.limbs == fin.limbs).all() and (fo.exp == fin.exp).all() and (fo.cls == fin.cls).all()
    print(f"n={n} p={p} steps={steps} tc_engine={c['tc_engine']} bit-identical={bool(same)}", flush=True)
    assert same
