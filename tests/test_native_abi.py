"""The C-ABI library loads without a GPU and exports every symbol sgf.h declares."""
import os
import re

from paper_1907_03406_b200 import _native

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    text = open(os.path.join(ROOT, "include", "sgf.h")).read()
    return sorted(set(re.findall(r"\b(sgf_[a-z_]+)\s*\(", text)))


def test_library_exports_header_symbols():
    L = _native.load_library()
    declared = header_functions()
    assert declared, "no declarations parsed"
    for name in declared:
        assert hasattr(L, name), name
    assert set(declared) == set(_native.EXPORTS)


def test_context_without_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        return
    import pytest
    with pytest.raises(_native.NativeUnavailable):
        _native.context(0)
