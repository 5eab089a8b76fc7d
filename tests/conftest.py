import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a); parity tests through the C-ABI")
    config.addinivalue_line("markers", "slow: long-running (large-N) check")


@pytest.fixture(scope="session")
def hq():
    """The product binding (CUDA C-ABI library).  Only used by -m gpu tests."""
    import torch

    if not torch.cuda.is_available():
        pytest.fail("gpu test selected but CUDA is not available")
    from paper_2603_03019_b200 import hq as _hq

    return _hq
