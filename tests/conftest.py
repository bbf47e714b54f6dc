import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) CUDA device")


@pytest.fixture(scope="session")
def gpu_ctx():
    import torch

    import paper_2305_08872_b200 as P

    assert torch.cuda.is_available(), "GPU test selected but no CUDA device is visible"
    ctx = P.Context(0)
    yield ctx
    ctx.close()


@pytest.fixture(scope="session")
def dry_ctx():
    import paper_2305_08872_b200 as P

    ctx = P.Context(dry_run=True)
    yield ctx
    ctx.close()
