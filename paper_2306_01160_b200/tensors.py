"""Layout helpers, tile geometry, sentinels and seeded synthetic inputs.

Mirrors the parts of pkg/src/scfa/tensors.py that the attention path uses:
``BlockSpec`` (:63-78), ``default_scale`` (:81-83), the pad sentinels
(:22-24), ``to_heads``/``from_heads`` (:157-164) and the per-(seed, domain,
index) Philox streams (:86-107) so that a seed names the same synthetic
tensor here and in the reference.  Tensors are torch tensors; the engine
layout is (B, H, T, D), the boundary layout (B, T, H, D).
"""

import os
from dataclasses import dataclass

import numpy as np
import torch

from .errors import ParameterError, ShapeError

KEY_PAD = 10**9
QUERY_PAD = -1

DOMAIN_VALUES = 0
DOMAIN_PROJECTIONS = 1
DOMAIN_KEEP = 2
DOMAIN_BUCKETS = 3

_M64 = (1 << 64) - 1


@dataclass(frozen=True)
class BlockSpec:
    """Reference tile geometry (B_m query rows x B_n key columns).

    The CUDA kernels run fixed 128-row tiles; a BlockSpec only changes the
    *reported* reference schedule (``FlashOutputs.tiles_computed``), never
    the numbers computed.
    """

    B_m: int = 64
    B_n: int = 64

    def __post_init__(self):
        if self.B_m < 1 or self.B_n < 1:
            raise ShapeError(f"block sizes must be >= 1, got {self.B_m}, {self.B_n}")

    def query_blocks(self, T_Q):
        return -(-T_Q // self.B_m)

    def key_blocks(self, T_KV):
        return -(-T_KV // self.B_n)


def default_scale(D):
    return 1.0 / float(np.sqrt(D))


def dtype_for(precision):
    if precision == 32:
        return torch.float32
    if precision == 64:
        return torch.float64
    if precision == 16:
        return torch.bfloat16
    raise ParameterError(f"precision must be 16, 32 or 64, got {precision}")


def to_heads(x):
    """(B, T, H, ...) -> (B, H, T, ...) contiguous."""
    return x.transpose(1, 2).contiguous()


def from_heads(x):
    """(B, H, T, ...) -> (B, T, H, ...) contiguous."""
    return x.transpose(1, 2).contiguous()


def stream(seed, domain, index=0):
    """numpy Generator for one (seed, domain, index) Philox key (tensors.py:86-93)."""
    key = ((seed & _M64) << 64) | ((domain & 0xFF) << 56) | (index & ((1 << 56) - 1))
    return np.random.Generator(np.random.Philox(key=key))


def random_tensor_np(shape, seed, dtype=np.float64):
    """(B, H, T, D) standard normal, one stream per (b, h) (tensors.py:96-107)."""
    B, H, T, D = (int(e) for e in shape)
    if min(B, H, T, D) < 1:
        raise ShapeError(f"all extents must be >= 1, got {shape}")
    out = np.empty((B, H, T, D), dtype=dtype)
    for b in range(B):
        for h in range(H):
            out[b, h] = stream(seed, DOMAIN_VALUES, b * H + h).standard_normal((T, D), dtype=dtype)
    return out


def random_tensor(shape, seed, device="cuda", dtype=torch.bfloat16):
    return torch.from_numpy(random_tensor_np(shape, seed)).to(device=device, dtype=dtype)


def worker_count():
    """Accepted for signature parity (tensors.py:167-175); the GPU path ignores it."""
    env = os.getenv("SCFA_WORKERS")
    if env:
        n = int(env)
        if n < 1:
            raise ParameterError(f"SCFA_WORKERS must be >= 1, got {n}")
        return n
    return 1


def pad128(T):
    return ((int(T) + 127) // 128) * 128
