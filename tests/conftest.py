import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

ORACLE_LIB = os.path.join(ROOT, "oracle", "liboracle.so")
REF_LIB = os.path.join(ROOT, "oracle", "_ref", "libkvtier_ref.so")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built CUDA library")
    config.addinivalue_line("markers", "slow: long-running parity sweep")


def _gpu_available():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if _gpu_available():
        return
    skip = pytest.mark.skip(reason="no CUDA device visible")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


@pytest.fixture(scope="session")
def oracle_abi():
    from paper_2512_14946_b200 import _abi
    if not os.path.exists(ORACLE_LIB):
        pytest.fail("oracle/liboracle.so missing: run make -C oracle")
    return _abi.Abi(ORACLE_LIB, "orc_", codec=True)


@pytest.fixture(scope="session")
def ref_abi():
    from paper_2512_14946_b200 import _abi
    if not os.path.exists(REF_LIB):
        pytest.skip("oracle/_ref/libkvtier_ref.so not built (needs /root/reference here)")
    return _abi.Abi(REF_LIB, "ref_", codec=False)


@pytest.fixture(scope="session")
def gpu_abi():
    import paper_2512_14946_b200 as pkg
    return pkg.product()
