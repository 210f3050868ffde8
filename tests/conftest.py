import os
import sys

import pytest

# PE and DE engines sharing one GPU run several streams each whose spin waits
# must never sit in one hardware queue in front of their producers: give
# every stream its own connection (set before the first CUDA call)
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

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


@pytest.fixture(params=["same_gpu", "peer_gpu"])
def de_dev(request, gpus):
    """Device of the DE side of a DE-read-path test.  'same_gpu' puts the DE
    engine (its store, its decode pool, its kernels) on the PE's own GPU —
    the kernels and their system-scope releases are the cross-GPU ones, the
    stores just land in local HBM — so the DE path is exercised on a 1-GPU
    box; 'peer_gpu' is the real NVLink case on device 1."""
    if request.param == "peer_gpu":
        request.applymarker(pytest.mark.multigpu)
        if gpus < 2:
            pytest.skip("needs >= 2 GPUs (run with gpurun --gpus 2)")
        return 1
    return 0
