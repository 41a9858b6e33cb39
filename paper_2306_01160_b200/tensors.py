"""Layout helpers, tile geometry, sentinels and seeded synthetic inputs.

Mirrors the parts of pkg/src/scfa/tensors.py that the attention path uses:
``BlockSpec`` (:63-78), ``default_scale`` (:81-83), the pad sentinels
(:22-24), ``to_heads``/``from_heads`` (:157-164) and the per-(seed, domain,
index) Philox streams (:86-107) so that a seed names the same synthetic
tensor here and in the reference.  Tensors are torch tensors; the engine
layout is (B, H, T, D), the boundary layout (B, T, H, D).
"""

import os
import struct
from dataclasses import dataclass

import numpy as np
import torch

from .errors import FormatError, ParameterError, ShapeError

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


# ---------------------------------------------------------------- SCFA tensor files

MAGIC = b"SCFA"
VERSION = 1
_HEADER = struct.Struct("<4sIB4Q")


def save_tensor(path, x):
    """Write a (B, H, T, D) float32 / float64 tensor in the reference's container format
    (tensors.py:110-125): magic "SCFA", u32 version 1, u8 bytes per element, four u64
    extents, then the little-endian values in row-major order.  Torch tensors (any device)
    are written from their host copy."""
    if isinstance(x, torch.Tensor):
        x = x.detach().cpu().numpy()
    x = np.asarray(x)
    if x.ndim != 4:
        raise ShapeError(f"tensor must be 4-D (B, H, T, D), got ndim={x.ndim}")
    if x.dtype not in (np.float32, np.float64):
        raise ShapeError(f"tensor must be float32 or float64, got {x.dtype}")
    if not np.isfinite(x).all():
        raise ShapeError("tensor must be finite")
    with open(path, "wb") as f:
        f.write(_HEADER.pack(MAGIC, VERSION, x.dtype.itemsize, *x.shape))
        f.write(np.ascontiguousarray(x, dtype=x.dtype.newbyteorder("<")).tobytes())


def load_tensor(path):
    """Read a file written by save_tensor (either implementation); FormatError with the
    byte offset of the first defect otherwise (tensors.py:128-154)."""
    with open(path, "rb") as f:
        raw = f.read()
    if len(raw) < _HEADER.size:
        raise FormatError("file truncated inside header", len(raw))
    magic, version, itemsize, B, H, T, D = _HEADER.unpack_from(raw, 0)
    if magic != MAGIC:
        raise FormatError(f"bad magic {magic!r}", 0)
    if version != VERSION:
        raise FormatError(f"unsupported version {version}", 4)
    if itemsize not in (4, 8):
        raise FormatError(f"bad precision byte {itemsize}", 8)
    for i, e in enumerate((B, H, T, D)):
        if e < 1:
            raise FormatError(f"extent {i} is {e}", 9 + 8 * i)
    count = B * H * T * D
    expected = _HEADER.size + count * itemsize
    if len(raw) != expected:
        raise FormatError(f"payload has {len(raw) - _HEADER.size} bytes, expected {count * itemsize}",
                          min(len(raw), expected))
    dtype = np.dtype("<f4" if itemsize == 4 else "<f8")
    data = np.frombuffer(raw, dtype=dtype, count=count, offset=_HEADER.size)
    return data.reshape(B, H, T, D).astype(dtype.newbyteorder("="))

