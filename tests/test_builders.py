"""The drop-in's matrix builders reproduce the reference's inputs bit for bit
(MatrixBuffer.fingerprint of the reference run recorded in the goldens)."""
import pytest

from _util import generate, golden_names, load_golden

CASES = [n for n in golden_names() if load_golden(n)[0].get("gen")]


@pytest.mark.parametrize("name", CASES)
def test_builder_fingerprint(name):
    meta, _ = load_golden(name)
    if meta["gen"][0] == "beta":
        pytest.skip("beta64 regeneration is covered by test_beta_builder (slow)")
    A = generate(meta["gen"])
    assert A.fingerprint() == meta["fingerprint"]


@pytest.mark.slow
def test_beta_builder():
    meta, _ = load_golden("beta64_p256")
    assert generate(meta["gen"]).fingerprint() == meta["fingerprint"]
