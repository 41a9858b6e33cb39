"""Dense causal flash attention on the same engine — the comparator.

API mirror of pkg/src/scfa/dense.py: the reference runs its tile loop with
``idx = arange(T)`` and the triangular schedule (dense.py:33-93); here the
same tcgen05 kernels run with arange index vectors, so every diagonal tile is
a masked boundary tile and every tile below it runs mask-free.
"""

import torch

from . import _lib
from ._kernel import Problem, as_operand, attention_backward, attention_forward, check_forward_operands
from .errors import ShapeError
from .tensors import BlockSpec, pad128
from ._headdim import padded_call


def dense_tile_count(T, blocks=BlockSpec()):
    """Tiles of the reference causal schedule for one head (dense.py:16-30)."""
    if T < 1:
        raise ShapeError(f"T must be >= 1, got {T}")
    n = blocks.key_blocks(T)
    total = 0
    for i in range(blocks.query_blocks(T)):
        last_q = min((i + 1) * blocks.B_m, T) - 1
        total += min(n, last_q // blocks.B_n + 1)
    return total


_ARANGE = {}


def _arange_aux(B, H, T, oob, device):
    key = (T, str(device))
    if key not in _ARANGE:
        _ARANGE[key] = torch.arange(T, dtype=torch.int32, device=device)
    src = _ARANGE[key]
    out = torch.empty((B * H, pad128(T)), dtype=torch.int32, device=device)
    _lib.call("scfa_pack_index", _lib.ptr(src), _lib.DT_I32, B * H, T, 0, 1, pad128(T), int(oob), _lib.ptr(out),
              _lib.stream_ptr())
    return out


def causal_problem(B, H, T, D, device):
    return Problem(B, H, T, T, D, _arange_aux(B, H, T, -1, device), _arange_aux(B, H, T, 0x7FFFFFFF, device))


@padded_call("flash_fwd")
def flash_forward(q, k, v, blocks=BlockSpec(), scale=None, workers=None, check=True):
    """Tiled causal attention over (B, H, T, D) operands (dense.py:33-63).

    check=False skips the read of the NumericError status word (graph capture)."""
    q, k, v = as_operand(q), as_operand(k), as_operand(v)
    check_forward_operands(q, k, v)
    B, H, T, D = q.shape
    if T != k.shape[2]:
        raise ShapeError("dense causal attention requires T_Q == T_KV")
    return attention_forward(causal_problem(B, H, T, D, q.device), q, k, v, scale, blocks, check=check)


@padded_call("flash_bwd")
def flash_backward(q, k, v, outputs, d_out, blocks=BlockSpec(), scale=None, workers=None):
    """Gradients of <O, dO> w.r.t. (Q, K, V), fp32 (dense.py:66-93)."""
    q, k, v = as_operand(q), as_operand(k), as_operand(v)
    check_forward_operands(q, k, v)
    B, H, T, D = q.shape
    if tuple(outputs.M.shape) != (B, H, T) or tuple(outputs.L.shape) != (B, H, T):
        raise ShapeError("stored M/L statistics do not match the operands")
    if tuple(d_out.shape) != tuple(q.shape):
        raise ShapeError(f"dO shape {tuple(d_out.shape)} does not match Q {tuple(q.shape)}")
    prob = getattr(outputs, "_problem", None)
    if prob is None or prob.T_q != T or prob.flags != 0:
        prob = causal_problem(B, H, T, D, q.device)
    return attention_backward(prob, q, k, v, outputs, d_out, scale)
