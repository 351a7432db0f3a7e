import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")


def _has_gpu() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:  # pragma: no cover
        return False


@pytest.fixture(scope="session")
def engine():
    if not _has_gpu():
        pytest.fail("gpu test selected on a host without a CUDA device")
    from paper_2205_02473_b200.engine import Engine
    return Engine(int(os.environ.get("DPRO_TEST_DEVICE", "0")))


@pytest.fixture(scope="session")
def ref():
    from oracle import oracle
    if not oracle.ref_available():
        pytest.skip("oracle/_ref/libdpro_ref.so not built (needs /root/reference at build time)")
    return oracle


@pytest.fixture(scope="session")
def port():
    from oracle import oracle
    assert oracle.port_available(), "oracle/liboracle.so missing: run make -C oracle port"
    return oracle
