import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


def _ensure_built():
    lib = ROOT / "paper_2302_02599_b200" / "libapl.so"
    if not lib.exists() and Path("/usr/local/cuda/bin/nvcc").exists():
        from paper_2302_02599_b200 import build

        build.build()
    ora = ROOT / "oracle" / "_build" / "libapl_oracle.so"
    if not ora.exists():
        import oracle

        oracle.build(ref=Path("/root/reference/proj/src").exists())


_ensure_built()


@pytest.fixture(scope="session")
def cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda:0")
