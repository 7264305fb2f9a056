"""The C-ABI library loads (no GPU needed) and exports every function
include/detseries_b200.h declares; the product fails loudly without a GPU."""
import os
import re

import pytest

from paper_1308_1536_b200 import _native
from paper_1308_1536_b200.errors import DeviceUnavailable

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = open(os.path.join(ROOT, "include", "detseries_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ds_[a-z_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    lib = _native.load_library()
    declared = header_functions()
    assert len(declared) >= 15
    for name in declared:
        assert hasattr(lib, name), name
    assert set(declared) == set(_native.EXPORTS)
    assert lib.ds_version().startswith(b"detseries_b200")


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_1308_1536_b200 import Precision, eliminate, synth_matrix
    A = synth_matrix("random_uniform", 4, 1, Precision(128))
    with pytest.raises(DeviceUnavailable):
        eliminate(A)
