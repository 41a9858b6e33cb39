"""torch.autograd for the sparse attention calls.

The reference API is forward-only (qk_sparse.py:228-239, hash_sparse.py:223-238);
its backward exists only at kernel level (qk_backward_kernel / hash_backward_kernel).
These Functions compose the same path as the reference's kernel-level backward
(SURVEY.md §8c): the forward keeps the index preparation, bucket-ordered operands
and saved log-sum-exp, and the backward runs the dQ and dK/dV kernels, whose
epilogues write each gradient row straight back to its original position.
"""

import torch

from ._kernel import as_operand, attention_backward, attention_forward, check_status
from ._headdim import padded_call

__all__ = ["dense_causal_attention_autograd", "hash_sparse_attention_autograd", "qk_sparse_attention_autograd"]


class _HashSparseAttention(torch.autograd.Function):
    @staticmethod
    def forward(ctx, q, k, v, q_hash, k_hash, scale, exclude_self, check):
        # the same stages as hash_sparse_attention_fwd_bwd (copy-free bucket order for Q / dO)
        from .hash_sparse import _hash_forward_stage

        st = _hash_forward_stage(q, k, v, q_hash, k_hash, scale, exclude_self)
        if check:  # bucket ids (hash_sparse.py:112-113) and a non-finite output (softmax.py:63-64)
            check_status(st.err)
        ctx.state = (st, q.dtype, k.dtype, v.dtype)
        return st.outputs.O.to(q.dtype)

    @staticmethod
    def backward(ctx, d_out):
        from .hash_sparse import _hash_backward_stage

        st, qt, kt, vt = ctx.state
        dq, dk, dv = _hash_backward_stage(st, d_out.contiguous())
        ctx.state = None
        return dq.to(qt), dk.to(kt), dv.to(vt), None, None, None, None, None


class _QkSparseAttention(torch.autograd.Function):
    @staticmethod
    def forward(ctx, q, k, v, q_keep, k_keep, scale, check):
        # the same stages as qk_sparse_attention_fwd_bwd
        from .qk_sparse import _qk_forward_stage

        st = _qk_forward_stage(q, k, v, q_keep, k_keep, scale)
        if check:  # keep entries in {0, 1} (qk_sparse.py:54-55), a non-finite output (softmax.py:63-64)
            check_status(st.err, "keep entries must be 0 or 1")
        ctx.state = (st, q.dtype, k.dtype, v.dtype)
        return st.outputs.O.to(q.dtype)

    @staticmethod
    def backward(ctx, d_out):
        from .qk_sparse import _qk_backward_stage

        st, qt, kt, vt = ctx.state
        dq, dk, dv = _qk_backward_stage(st, d_out.contiguous())
        ctx.state = None
        return dq.to(qt), dk.to(kt), dv.to(vt), None, None, None, None


@padded_call("attn")
def hash_sparse_attention_autograd(q, k, v, q_hash, k_hash, scale=None, exclude_self=True, check=True):
    """hash_sparse_attention (hash_sparse.py:223-238) with gradients w.r.t. q, k, v.

    check=False skips the status read-back (one host sync per call: bucket ids, non-finite
    output) for callers whose ids are valid by construction, e.g. an argmax over LSH
    projections.
    """
    return _HashSparseAttention.apply(q, k, v, q_hash, k_hash, scale, exclude_self, check)


@padded_call("attn")
def qk_sparse_attention_autograd(q, k, v, q_keep, k_keep, scale=None, check=True):
    """qk_sparse_attention (qk_sparse.py:228-239) with gradients w.r.t. q, k, v.

    check=False skips the status read-back (one host sync per call)."""
    return _QkSparseAttention.apply(q, k, v, q_keep, k_keep, scale, check)


_DENSE_PROBLEMS = {}


class _DenseCausalAttention(torch.autograd.Function):
    """The comparator (dense.py:33-93) on boundary-layout (B, T, H, D) operands: the
    operands are transposed once into engine layout, the epilogues write O and the
    gradients straight back to (B, T, H, D)."""

    @staticmethod
    def forward(ctx, q, k, v, scale):
        from .dense import causal_problem

        B, T, H, D = q.shape
        eng = [as_operand(x).transpose(1, 2).contiguous() for x in (q, k, v)]
        key = (B, H, T, D, eng[0].device)
        prob = _DENSE_PROBLEMS.get(key)
        if prob is None:  # the causal schedule depends on the shape only
            prob = _DENSE_PROBLEMS[key] = causal_problem(B, H, T, D, eng[0].device)
            prob.schedule("fwd", "dq", "dkdv")
        out = attention_forward(prob, *eng, scale, boundary=(T, False))
        ctx.state = (prob, eng, out, scale, T, q.dtype, k.dtype, v.dtype)
        return out.O.to(q.dtype)

    @staticmethod
    def backward(ctx, d_out):
        prob, eng, out, scale, T, qt, kt, vt = ctx.state
        dq, dk, dv = attention_backward(prob, *eng, out, as_operand(d_out.contiguous()), scale, boundary=(T, T, False))
        ctx.state = None
        return dq.to(qt), dk.to(kt), dv.to(vt), None


@padded_call("attn")
def dense_causal_attention_autograd(q, k, v, scale=None):
    """Dense causal attention on (B, T, H, D) operands with gradients (dense.py:33-93)."""
    return _DenseCausalAttention.apply(q, k, v, scale)
