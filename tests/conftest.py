import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs on the GPU box)")
    config.addinivalue_line("markers", "multigpu: needs >= 2 GPUs")


def n_gpus():
    from paper_2602_21548_b200 import abi
    return abi.device_count()


@pytest.fixture(scope="session")
def gpus():
    n = n_gpus()
    if n < 1:
        pytest.fail("GPU test selected but no CUDA device is visible")
    import torch  # plumbing only: device buffers for block tables
    torch.cuda.init()
    return n


@pytest.fixture(scope="session")
def two_gpus(gpus):
    if gpus < 2:
        pytest.skip("needs >= 2 GPUs (run with gpurun --gpus 2)")
    return gpus
