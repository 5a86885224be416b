import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run with -m gpu via gpurun)")
    config.addinivalue_line("markers", "slow: longer CPU test")


@pytest.fixture(scope="session")
def oracle_lib():
    from oracle import cref
    cref.build()
    return cref


@pytest.fixture(scope="session")
def golden():
    import json

    import numpy as np
    here = os.path.join(ROOT, "tests", "golden")
    meta = json.load(open(os.path.join(here, "harris_golden.json")))
    arrays = dict(np.load(os.path.join(here, "harris_golden.npz")))
    return meta, arrays


@pytest.fixture(scope="session")
def cuda_ctx():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU test collected without a CUDA device (run -m gpu on a B200)")
    import paper_2212_12035_b200 as hb
    return hb.context(0)
