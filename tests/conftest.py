import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a) device")


def bf16_round(x):
    """Round a float array to bf16 (round-to-nearest-even) and return float64."""
    import torch

    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).to(torch.bfloat16).to(torch.float64).numpy()


def make_batch(B, H, T, D, seed=0):
    """bf16-representable Q/K/V (B, H, T, D) float64 from consecutive reference seeds."""
    from paper_2306_01160_b200.tensors import random_tensor_np

    return tuple(bf16_round(random_tensor_np((B, H, T, D), seed + i)) for i in range(3))


@pytest.fixture
def cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda")
