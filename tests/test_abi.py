"""The C-ABI library loads without a GPU and exports every declared symbol."""

import os
import re

import pytest

from paper_2508_03148_b200 import engine

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    with open(os.path.join(ROOT, "include", "frontier_b200.h")) as fh:
        text = fh.read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(fs_[a-z_0-9]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    if not os.path.exists(engine.LIB_PATH):
        pytest.skip("engine library not built")
    lib = engine.load_library()  # also checks the struct sizes against numpy dtypes
    names = declared_functions()
    assert len(names) >= 15
    missing = [n for n in names if not hasattr(lib, n)]
    assert missing == []


def test_abi_version():
    if not os.path.exists(engine.LIB_PATH):
        pytest.skip("engine library not built")
    assert engine.load_library().fs_abi_version() == 2


def test_engine_fails_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    if not os.path.exists(engine.LIB_PATH):
        pytest.skip("engine library not built")
    with pytest.raises(engine.EngineUnavailable):
        engine.Engine(0)
