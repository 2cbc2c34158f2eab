import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
GOLDEN = os.path.join(ROOT, "tests", "golden", "golden.json")
EMU_LIB = os.path.join(ROOT, "tests", "emu", "libdashemu.so")
CUDA_LIB = os.path.join(ROOT, "paper_2302_06361_b200", "libdashgpu.so")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); runs the real libdashgpu.so")
    config.addinivalue_line("markers", "slow: longer CPU-side checks")


@pytest.fixture(scope="session")
def golden():
    with open(GOLDEN) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def oracle():
    from pyoracle import Oracle

    return Oracle()


@pytest.fixture(scope="session")
def emu():
    """CPU emulation of the device code (test infrastructure, tests/emu)."""
    if not os.path.exists(EMU_LIB):
        pytest.skip("tests/emu/libdashemu.so not built")
    from paper_2302_06361_b200.engine import Dash

    return Dash(lib_path=EMU_LIB, emulation=True)


@pytest.fixture(scope="session")
def gpu():
    """The product: libdashgpu.so on cuda:0 (fails loudly if it cannot load)."""
    from paper_2302_06361_b200.engine import Dash

    return Dash(0)
