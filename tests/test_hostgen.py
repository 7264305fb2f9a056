"""The C host builder (libds_hostgen.so) reproduces the drop-in's and the
reference's Artless beta matrix bit for bit (input generation for config 3),
and the committed column-Gamma cache matches a fresh computation."""
import os

import numpy as np
import pytest

from _util import generate, load_golden
from paper_1308_1536_b200 import genmat, hostgen
from paper_1308_1536_b200.matrix import MatrixBuffer
from paper_1308_1536_b200.scalars import Precision
from paper_1308_1536_b200.soa import SoA

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_ZEROS = os.path.join(ROOT, "data", "zeta_zeros.txt")
ZEROS = os.path.join(ROOT, "data", "zeta_zeros_4096.txt")


def test_c_builder_matches_reference_golden():
    meta, _ = load_golden("beta64_p256")
    s = hostgen.beta_matrix_soa(REF_ZEROS, 64, 256)
    assert MatrixBuffer.from_soa(64, "real", Precision(256), s).fingerprint() == meta["fingerprint"]


@pytest.mark.parametrize("N,p", [(8, 1024), (6, 333)])
def test_c_builder_matches_python_builder(N, p):
    z = genmat.load_zeros(ZEROS, Precision(p), N)
    B = genmat.beta_matrix(z, N, genmat.SpougeGamma(), Precision(p))
    s = hostgen.beta_matrix_soa(ZEROS, N, p)
    assert MatrixBuffer.from_soa(N, "real", Precision(p), s).fingerprint() == B.fingerprint()


def test_gamma_cache_columns():
    path = os.path.join(ROOT, "data", "beta_gammas_p4096_N2000.npz")
    if not os.path.exists(path):
        pytest.skip("no cache")
    z = np.load(path)
    cache = SoA(2, int(z["L"]), int(z["count"]), np.ascontiguousarray(z["limbs"]), np.ascontiguousarray(z["exp"]),
                np.ascontiguousarray(z["cls"]))
    fresh = hostgen.beta_gammas_soa(ZEROS, 3, 4096)  # columns 0..2
    for j in range(3):
        assert cache.canonical(j, 4160) == fresh.canonical(j, 4160)
    # the cached path and the direct path give the same matrix (small N)
    a = hostgen.beta_matrix_soa(ZEROS, 3, 4096)
    b = hostgen.beta_matrix_soa(ZEROS, 3, 4096, gammas=cache)
    assert np.array_equal(a.limbs, b.limbs) and np.array_equal(a.exp, b.exp) and np.array_equal(a.cls, b.cls)
