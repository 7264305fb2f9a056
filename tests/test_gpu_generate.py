"""Device-side builder (ds_generate, csrc/ds_gen.cu): the counter-based
random_uniform matrix generated in HBM equals its host twin
(synth.counter_uniform_soa) bit for bit, for every rank of a row-cyclic
split, and the elimination of a device-generated matrix matches the oracle."""
import numpy as np
import pytest

import oracle
from _util import results_digest
from paper_1308_1536_b200.engine import DeviceElimination, HostResults
from paper_1308_1536_b200.soa import SoA
from paper_1308_1536_b200.synth import counter_uniform_soa

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,p,world", [(37, 100, 1), (50, 1024, 3), (33, 4096, 2), (12, 33220, 4), (64, 64, 1)])
def test_device_generator_matches_host_twin(n, p, world):
    L = (p + 31) // 32
    for rank in range(world):
        rows = np.arange(rank, n, world)
        with DeviceElimination(n, p, "real", 0, rank, world) as eng:
            eng.generate(seed=1234 + p)
            got = SoA(1, L, len(rows) * n)
            eng.fetch(got)
        ref = counter_uniform_soa(n, p, 1234 + p, rows=rows)
        assert np.array_equal(got.cls, ref.cls)
        assert np.array_equal(got.exp, ref.exp)
        assert np.array_equal(got.limbs, ref.limbs)


@pytest.mark.parametrize("n,p", [(120, 1024), (40, 4100)])
def test_generated_matrix_elimination_matches_oracle(n, p):
    A = counter_uniform_soa(n, p, 99)
    with DeviceElimination(n, p, "real") as eng:
        eng.generate(seed=99)
        res = HostResults.alloc(n, 1, eng.L, True)
        eng.run(True, True, 0, n, res)
        fin = A.copy()
        eng.fetch(fin)
    rc, done, res_o, fin_o = oracle.eliminate_soa(A, n, p, "real")
    assert results_digest(res_o, fin_o, n, p, done) == results_digest(res, fin, n, p, n)
