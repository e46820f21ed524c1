import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running")


def _ensure_built():
    lib = ROOT / "paper_2604_14650_b200" / "lib" / "liblpm6cu.so"
    orc = ROOT / "oracle" / "liblpm6oracle.so"
    if not lib.exists() or not orc.exists():
        import __graft_entry__
        __graft_entry__.build()


_ensure_built()


@pytest.fixture(scope="session")
def lpm():
    import paper_2604_14650_b200 as L
    return L


@pytest.fixture(scope="session")
def orc():
    from oracle.oracle import Oracle
    return Oracle()


@pytest.fixture(scope="session")
def ref():
    from oracle.oracle import REF_SO, RefOracle
    if not REF_SO.exists():
        pytest.skip("oracle/_ref not built (reference sources absent at build time)")
    return RefOracle()


@pytest.fixture(scope="session")
def cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch
