import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run with -m gpu on the GPU box)")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def ref():
    """The reference planner (oracle/_ref/libpoasref.so). Built here from
    /root/reference; travels prebuilt to the GPU box."""
    import oracle

    if not oracle.REF_SO.exists():
        if Path("/root/reference/proj/src").is_dir():
            oracle.build(with_ref=True)
        else:
            pytest.skip("reference planner library not built (no /root/reference here)")
    return oracle.ref


@pytest.fixture(scope="session")
def poas():
    from paper_2209_10245_b200 import poas as p

    return p


@pytest.fixture(scope="session")
def mach2_cfg():
    return (GOLDEN / "mach2.cfg").read_text()


def has_gpu():
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False
