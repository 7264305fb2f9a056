"""The CPU oracle (oracle/ds_oracle.c) against golden vectors recorded from the
UNMODIFIED reference (tests/golden/make_goldens.py): bit-identical trace,
minors and final buffer on every case.  This pins the checker every GPU
parity test relies on."""
import pytest

import oracle
from _util import build_input, golden_names, load_golden, results_digest


@pytest.mark.parametrize("name", golden_names())
def test_oracle_matches_reference(name):
    meta, arrays = load_golden(name)
    if meta["name"] == "beta64_p256" and "in_limbs" not in arrays:
        pytest.skip("input not stored")
    A = build_input(meta, arrays)
    n, p, kind = meta["n"], meta["prec"], meta["kind"]
    rc, done, res, final = oracle.eliminate_soa(A, n, p, kind, meta["collect_minors"], meta["series"])
    if meta["zero_pivot_step"] is not None:
        assert rc == oracle.DS_ZERO_PIVOT and done + 1 == meta["zero_pivot_step"]
    else:
        assert rc == oracle.DS_OK and done == n
    assert results_digest(res, final, n, p, done) == meta["digest"]


def test_oracle_version():
    assert b"MPFR" in oracle.lib().dso_version()
