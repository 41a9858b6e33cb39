"""Hash-sparse attention: bucket sort, banded kernels, inverse scatter — on the GPU.

API mirror of pkg/src/scfa/hash_sparse.py.  Bucket ids arrive as (B, T, H)
(boundary) or (B, H, T) (engine) integer tensors; a stable per-(b, h) radix
sort by bucket (ties kept in position order, hash_sparse.py:89-94) produces
a permutation that drives a fused gather+transpose of Q/K/V, the exact tile
lists and the tcgen05 kernels; the inverse permutation routes outputs back.
"""

import ctypes
import os
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._kernel import (
    FlashOutputs,
    Problem,
    RowTables,
    make_row_tables,
    as_operand,
    attention_backward,
    attention_forward,
    check_forward_operands,
    check_status,
    pack_index,
)
from .errors import NumericError, ParameterError, ShapeError
from .tensors import DOMAIN_BUCKETS, DOMAIN_PROJECTIONS, BlockSpec, pad128, stream
from ._headdim import padded_call

_OOB_QI, _OOB_KI = -1, 0x7FFFFFFF
_OOB_QH, _OOB_KH = -3, -2


@dataclass
class SortedBatch:
    """Operands reordered by bucket plus provenance (hash_sparse.py:71-86).

    q/k/v (B, H, T, D) bf16; q_idx/k_idx (B, H, T) int32 original positions;
    q_hash/k_hash (B, H, T) int32 sorted bucket ids.
    """

    q: torch.Tensor
    k: torch.Tensor
    v: torch.Tensor
    q_idx: torch.Tensor
    k_idx: torch.Tensor
    q_hash: torch.Tensor
    k_hash: torch.Tensor
    problem: object = None
    q_rank: torch.Tensor = None  # (B*H, T_Q) position -> sorted slot
    k_rank: torch.Tensor = None
    q_perm: torch.Tensor = None  # (B*H, T_Q) sorted slot -> position
    k_perm: torch.Tensor = None


def random_buckets(B, T, H, nb, seed):
    """Uniform bucket ids, same stream as hash_sparse.py:55-60 (numpy, int64)."""
    if nb < 1:
        raise ParameterError(f"number of buckets must be >= 1, got {nb}")
    return stream(seed, DOMAIN_BUCKETS).integers(0, nb, size=(B, T, H), dtype=np.int64)


def lsh_buckets(x, nb, seed):
    """Angular LSH codes for (B, T, H, D) vectors (hash_sparse.py:34-52).

    The projections are drawn from the reference's Philox streams on the host (one
    D x nb/2 standard-normal matrix per (b, h), tensors.py:86-93), so ids agree with
    the reference; the projection and the argmax of [xR, -xR] run on the GPU in float64
    (scfa_lsh_buckets).  Returns int64 (B, T, H) on the device.
    """
    if nb < 2 or nb % 2 != 0:
        raise ParameterError(f"number of buckets must be even and >= 2, got {nb}")
    x = torch.as_tensor(x)
    if x.dim() != 4:
        raise ShapeError("lsh_buckets expects (B, T, H, D) vectors")
    B, T, H, D = x.shape
    dev = x.device if x.is_cuda else torch.device("cuda")
    if x.dtype not in (torch.float32, torch.float64, torch.bfloat16):
        x = x.to(torch.float64)
    x = x.to(dev)
    R = np.stack([stream(seed, DOMAIN_PROJECTIONS, b * H + h).standard_normal((D, nb // 2))
                  for b in range(B) for h in range(H)]) if B * H else np.zeros((0, D, nb // 2))
    R = torch.from_numpy(np.ascontiguousarray(R, dtype=np.float64)).to(dev)
    out = torch.empty((B, T, H), dtype=torch.int64, device=dev)
    dt = _lib.DT_BF16 if x.dtype == torch.bfloat16 else _lib.dtype_code(x)
    _lib.call("scfa_lsh_buckets", _lib.ptr(x), dt, B, T, H, D, *x.stride(), _lib.ptr(R), nb, _lib.ptr(out),
              *out.stride(), _lib.stream_ptr(dev))
    return out


def normalize_keys(q):
    """Shared-QK keys: rows scaled to unit norm (hash_sparse.py:63-68)."""
    q = torch.as_tensor(q)
    n = torch.linalg.vector_norm(q.float(), dim=-1, keepdim=True)
    if bool((n == 0).any()):
        raise NumericError("cannot normalize zero-norm rows")
    return (q.float() / n).to(q.dtype)


def _hash_view(h, B, H, T, layout):
    """Element strides (sb, st, sh) of a bucket tensor in 'bth' or 'bht' layout."""
    h = torch.as_tensor(h)
    if layout == "bht":
        if tuple(h.shape) != (B, H, T):
            raise ShapeError("hash tensors must be (B, H, T) matching the operands")
        return h, h.stride(0), h.stride(2), h.stride(1)
    if tuple(h.shape) != (B, T, H):
        raise ShapeError("hash tensors must be (B, T, H) matching the operands")
    return h, h.stride(0), h.stride(1), h.stride(2)


def _sort(hash_t, sb, st, sh, B, H, T, err, pos=None):
    dev = hash_t.device
    perm = torch.empty((B * H, T), dtype=torch.int32, device=dev)
    rank = torch.empty((B * H, T), dtype=torch.int32, device=dev)
    scratch = torch.empty((B * H, T), dtype=torch.int32, device=dev)
    if pos is not None:
        pos2 = pos.reshape(B * H, T)
        pargs = (_lib.ptr(pos2), _lib.dtype_code(pos2), pos2.stride(0), pos2.stride(1))
    else:
        pargs = (None, 0, 0, 0)
    _lib.call("scfa_hash_sort", _lib.ptr(hash_t), _lib.dtype_code(hash_t), B, T, H, sb, st, sh, *pargs,
              _lib.ptr(perm), _lib.ptr(rank), _lib.ptr(scratch), _lib.ptr(err), _lib.stream_ptr())
    return perm, rank


def _aux(perm, hash_t, sb, st, sh, B, H, T, oob_i, oob_h, pos=None):
    T_pad = pad128(T)
    dev = perm.device
    idx = torch.empty((B * H, T_pad), dtype=torch.int32, device=dev)
    hsh = torch.empty((B * H, T_pad), dtype=torch.int32, device=dev)
    if pos is not None:
        pos2 = pos.reshape(B * H, T)
        pargs = (_lib.ptr(pos2), _lib.dtype_code(pos2), pos2.stride(0), pos2.stride(1))
    else:
        pargs = (None, 0, 0, 0)
    _lib.call("scfa_build_aux", _lib.ptr(perm), None, B, H, T, T, T_pad, 0, int(oob_i),
              _lib.ptr(hash_t), _lib.dtype_code(hash_t), sb, st, sh, int(oob_h), *pargs,
              _lib.ptr(idx), _lib.ptr(hsh), _lib.stream_ptr())
    return idx, hsh


def _gather(x, perm, layout):
    """Rows of x ('bthd' or 'bhtd') in perm order -> (B, H, T, D)."""
    if layout == "bthd":
        B, T, H, D = x.shape
        sb, st, sh = x.stride(0), x.stride(1), x.stride(2)
    else:
        B, H, T, D = x.shape
        sb, st, sh = x.stride(0), x.stride(2), x.stride(1)
    out = torch.empty((B, H, perm.shape[1], D), dtype=x.dtype, device=x.device)
    _lib.call("scfa_gather_rows", _lib.ptr(x), x.element_size(), B, H, D, sb, st, sh, _lib.ptr(perm),
              perm.shape[1], perm.shape[1], _lib.ptr(out), _lib.stream_ptr())
    return out


def _scatter(src, rank, layout, out_dtype=None):
    """(B, H, T, D) sorted rows -> original positions, in 'bthd' or 'bhtd' layout."""
    B, H, T, D = src.shape
    src = src.contiguous()
    dt = out_dtype or src.dtype
    if layout == "bthd":
        out = torch.empty((B, T, H, D), dtype=dt, device=src.device)
        db, dtt, dh = out.stride(0), out.stride(1), out.stride(2)
    else:
        out = torch.empty((B, H, T, D), dtype=dt, device=src.device)
        db, dtt, dh = out.stride(0), out.stride(2), out.stride(1)
    _lib.call("scfa_scatter_rows", _lib.ptr(src), src.element_size(), B, H, T, D, _lib.ptr(rank), T,
              _lib.ptr(out), out.element_size(), db, dtt, dh, _lib.stream_ptr())
    return out


def _gather3(xs, perms, layout):
    """Rows of up to three tensors ('bthd' or 'bhtd') in their perm order, one launch."""
    outs, strides = [], []
    for x, perm in zip(xs, perms):
        if layout == "bthd":
            B, T, H, D = x.shape
            strides += [x.stride(0), x.stride(1), x.stride(2)]
        else:
            B, H, T, D = x.shape
            strides += [x.stride(0), x.stride(2), x.stride(1)]
        outs.append(torch.empty((B, H, perm.shape[1], D), dtype=x.dtype, device=x.device))
    n = len(xs)
    _lib.call("scfa_gather_rows3", n, _lib.ptr_array(xs), _lib.ptr_array(outs), _lib.ptr_array(perms),
              _lib.i64_array(strides), xs[0].element_size(), B, H, D,
              _lib.i64_array([p.shape[1] for p in perms]), _lib.i64_array([p.shape[1] for p in perms]),
              _lib.stream_ptr())
    return outs


def _permute3(xs, ranks, T_perm):
    """As _gather3 for boundary-layout ('bthd') tensors, driven from the source side:
    rows are read in memory order and each is written to its slot rank[bh, t]
    (scfa_permute_rows3; measured ~10% faster than the gather at cfg2, random-row
    writes instead of random-row reads)."""
    outs, strides = [], []
    for x in xs:
        B, T, H, D = x.shape
        strides += [x.stride(0), x.stride(1), x.stride(2)]
        outs.append(torch.empty((B, H, T_perm, D), dtype=x.dtype, device=x.device))
    _lib.call("scfa_permute_rows3", len(xs), _lib.ptr_array(xs), _lib.ptr_array(outs), _lib.ptr_array(ranks),
              _lib.i64_array(strides), xs[0].element_size(), B, T, H, D, _lib.i64_array([T_perm] * len(xs)),
              _lib.stream_ptr())
    return outs


_PREP_MAX_T = 16384
_Q_WRITEOUT = True  # forward gathers Q and writes the bucket-order copy (see _fwd_bwd)
_DO_WRITEOUT = True  # dQ gathers dO, fuses delta, writes the bucket-order dO copy (two-pass backward)
# dQ reads Q tiled from the forward's kernel-order copy (only dO through the row table);
# SCFA_DQ_Q_SORTED=0 gathers both (A/B)
_DQ_Q_SORTED = os.environ.get("SCFA_DQ_Q_SORTED", "1") != "0"


def _event_ptr(ev):
    """The cudaEvent_t of a torch.cuda.Event (created by a first record if needed)."""
    if ev is None:
        return None
    if not ev.cuda_event:
        ev.record()
    return ctypes.c_void_p(ev.cuda_event)


def _prepare_shared(hash_t, sb, st, sh, B, H, T, D, err, exclude_self, sorted_event=None):
    """Fused sort + sorted vectors + visibility runs for shared bucket ids (scfa_hash_prepare)."""
    dev = hash_t.device
    BH, T_pad = B * H, pad128(T)
    perm = torch.empty((BH, T), dtype=torch.int32, device=dev)
    rank = torch.empty((BH, T), dtype=torch.int32, device=dev)
    scratch = torch.empty((BH, T + 257), dtype=torch.int32, device=dev)
    vec = torch.empty((5, BH, T_pad), dtype=torch.int32, device=dev)
    runs = torch.empty((2, BH, T_pad, 2), dtype=torch.int32, device=dev)
    flags = _lib.FLAG_HASH | (_lib.FLAG_EXCLUDE_SELF if exclude_self else 0)
    _lib.call("scfa_hash_prepare", _lib.ptr(hash_t), _lib.dtype_code(hash_t), B, T, H, sb, st, sh, flags,
              _lib.ptr(perm), _lib.ptr(rank), _lib.ptr(scratch), _lib.ptr(vec[0]), _lib.ptr(vec[1]),
              _lib.ptr(vec[2]), _lib.ptr(vec[3]), _lib.ptr(runs[0]), _lib.ptr(runs[1]), _lib.ptr(vec[4]),
              _lib.ptr(err), _event_ptr(sorted_event), _lib.stream_ptr())
    problem = Problem(B, H, T, T, D, vec[0], vec[1], vec[2], vec[3], flags=flags)
    problem.set_runs(runs[0], runs[1])
    problem.rows = RowTables(vec[4], vec[4], B * T * H, B * T * H)
    return perm, rank, problem


def _sort_batch(q, k, v, q_hash, k_hash, layout, q_pos=None, k_pos=None, check=True, exclude_self=True,
                materialize=True, sorted_event=None, err=None):
    """Shared by sort_by_bucket (engine layout) and hash_sparse_attention (boundary layout).

    materialize=False (boundary layout only): no sorted copies of q / k / v; the
    problem carries row tables (problem.rows) for the gather-mode kernels instead.
    """
    if layout == "bhtd":
        check_forward_operands(q, k, v)
        B, H, T_Q, D = q.shape
        T_KV = k.shape[2]
        hl = "bht"
    else:
        if q.dim() != 4 or k.dim() != 4 or k.shape != v.shape or q.shape[0] != k.shape[0] or q.shape[2] != k.shape[
                2] or q.shape[3] != k.shape[3]:
            raise ShapeError(f"operand shapes disagree: {tuple(q.shape)}, {tuple(k.shape)}, {tuple(v.shape)}")
        B, T_Q, H, D = q.shape
        T_KV = k.shape[1]
        hl = "bth"
    dev = q.device
    qh, qsb, qst, qsh = _hash_view(torch.as_tensor(q_hash, device=dev), B, H, T_Q, hl)
    same = (k_hash is q_hash) and T_Q == T_KV and q_pos is None and k_pos is None
    if same:
        kh, ksb, kst, ksh = qh, qsb, qst, qsh
    else:
        kh, ksb, kst, ksh = _hash_view(torch.as_tensor(k_hash, device=dev), B, H, T_KV, hl)
    if err is None:
        err = torch.zeros(1, dtype=torch.int32, device=dev)
    if same and 0 < T_Q <= _PREP_MAX_T:
        q_perm, q_rank, problem = _prepare_shared(qh, qsb, qst, qsh, B, H, T_Q, D, err, exclude_self, sorted_event)
        k_perm, k_rank = q_perm, q_rank
        if check and int(err.item()):
            raise ShapeError("bucket ids must be non-negative (and < 2**31)")
        if materialize:
            q_s, k_s, v_s = _gather3([q, k, v], [q_perm, q_perm, q_perm], layout)
        else:
            q_s, k_s, v_s = q, k, v
            if layout != "bthd":
                problem.rows = None
                q_s, k_s, v_s = _gather3([q, k, v], [q_perm, q_perm, q_perm], layout)
        qi, ki, qhs, khs = problem.q_idx, problem.k_idx, problem.q_hash, problem.k_hash
    else:
        q_perm, q_rank = _sort(qh, qsb, qst, qsh, B, H, T_Q, err, q_pos)
        if same:
            k_perm, k_rank = q_perm, q_rank
        else:
            k_perm, k_rank = _sort(kh, ksb, kst, ksh, B, H, T_KV, err, k_pos)
        if check and int(err.item()):
            raise ShapeError("bucket ids must be non-negative (and < 2**31)")
        qi, qhs = _aux(q_perm, qh, qsb, qst, qsh, B, H, T_Q, _OOB_QI, _OOB_QH, q_pos)
        ki, khs = _aux(k_perm, kh, ksb, kst, ksh, B, H, T_KV, _OOB_KI, _OOB_KH, k_pos)
        problem = Problem(B, H, T_Q, T_KV, D, qi, ki, qhs, khs, flags=_lib.FLAG_HASH)
        if materialize or layout != "bthd":
            q_s, k_s, v_s = _gather3([q, k, v], [q_perm, k_perm, k_perm], layout)
        else:
            q_s, k_s, v_s = q, k, v
            problem.rows = make_row_tables(q_perm, k_perm, B, H, T_Q, T_KV, T_Q, T_KV, problem.Tq_pad, problem.Tkv_pad,
                                      shared=same)
    return SortedBatch(
        q=q_s, k=k_s, v=v_s,
        q_idx=qi[:, :T_Q].view(B, H, T_Q), k_idx=ki[:, :T_KV].view(B, H, T_KV),
        q_hash=qhs[:, :T_Q].view(B, H, T_Q), k_hash=khs[:, :T_KV].view(B, H, T_KV),
        problem=problem, q_rank=q_rank, k_rank=k_rank, q_perm=q_perm, k_perm=k_perm,
    )


@padded_call("sort")
def sort_by_bucket(q, k, v, q_hash, k_hash, q_idx=None, k_idx=None):
    """Reorder engine-layout operands by (bucket, position) (hash_sparse.py:97-133)."""
    q, k, v = as_operand(q), as_operand(k), as_operand(v)
    dev = q.device
    qp = None if q_idx is None else torch.as_tensor(q_idx, device=dev)
    kp = None if k_idx is None else torch.as_tensor(k_idx, device=dev)
    if qp is not None:
        qp = qp.expand(q.shape[0], q.shape[1], q.shape[2])
    if kp is not None:
        kp = kp.expand(k.shape[0], k.shape[1], k.shape[2])
    return _sort_batch(q, k, v, q_hash, k_hash, "bhtd", qp, kp)


def _own_views(sb, prob):
    """Whether the batch's index / bucket vectors are still the ones its cached Problem was
    built from (a caller may replace them, e.g. dataclasses.replace(sb, q_hash=...))."""
    pairs = ((sb.q_idx, prob.q_idx), (sb.k_idx, prob.k_idx), (sb.q_hash, prob.q_hash), (sb.k_hash, prob.k_hash))
    return all(isinstance(a, torch.Tensor) and b is not None and a.is_cuda and a.dtype == torch.int32
               and a.data_ptr() == b.data_ptr() for a, b in pairs)


def _problem_of(sb, exclude_self, validate=True):
    flags = _lib.FLAG_HASH | (_lib.FLAG_EXCLUDE_SELF if exclude_self else 0)
    prob = sb.problem
    if prob is not None and not _own_views(sb, prob):
        prob = None  # rebuilt from the batch and validated (_check_sorted, hash_sparse.py:136-142)
    if prob is not None and prob.rows is not None:  # operands stayed in (B, T, H, D)
        B, H, T_Q, D = prob.B, prob.H, prob.T_q, prob.D
        T_KV = prob.T_kv
    else:
        B, H, T_Q, D = sb.q.shape
        T_KV = sb.k.shape[2]
    if prob is None or prob.T_q != T_Q or prob.T_kv != T_KV:
        dev = sb.q.device
        BH = B * H
        prob = Problem(B, H, T_Q, T_KV, D,
                       pack_index(sb.q_idx, BH, T_Q, _OOB_QI, dev), pack_index(sb.k_idx, BH, T_KV, _OOB_KI, dev),
                       pack_index(sb.q_hash, BH, T_Q, _OOB_QH, dev), pack_index(sb.k_hash, BH, T_KV, _OOB_KH, dev),
                       flags=flags)
        if validate and BH:
            prob.validate("hash")
        return prob
    if prob.flags != flags:
        clone = Problem(prob.B, prob.H, prob.T_q, prob.T_kv, prob.D, prob.q_idx, prob.k_idx, prob.q_hash,
                        prob.k_hash, flags=flags)
        clone.rows = prob.rows
        prob = clone
    return prob


@padded_call("hash_fwd")
def hash_forward_kernel(sorted_batch, scale=None, blocks=BlockSpec(), exclude_self=True, workers=None):
    """Banded forward over a SortedBatch (hash_sparse.py:145-179)."""
    sb = sorted_batch
    sb.q, sb.k, sb.v = as_operand(sb.q), as_operand(sb.k), as_operand(sb.v)
    check_forward_operands(sb.q, sb.k, sb.v)
    prob = _problem_of(sb, exclude_self)
    return attention_forward(prob, sb.q, sb.k, sb.v, scale, blocks, check=True)


@padded_call("hash_bwd")
def hash_backward_kernel(sorted_batch, outputs, d_out_sorted, scale=None, blocks=BlockSpec(), exclude_self=True,
                         workers=None):
    """Gradients w.r.t. the sorted operands, fp32 (hash_sparse.py:182-213)."""
    sb = sorted_batch
    check_forward_operands(sb.q, sb.k, sb.v)
    if tuple(d_out_sorted.shape) != tuple(sb.q.shape):
        raise ShapeError(f"dO shape {tuple(d_out_sorted.shape)} != {tuple(sb.q.shape)}")
    prob = getattr(outputs, "_problem", None)
    want = _lib.FLAG_HASH | (_lib.FLAG_EXCLUDE_SELF if exclude_self else 0)
    if prob is None or prob.flags != want or prob.T_q != sb.q.shape[2] or not _own_views(sb, prob):
        prob = _problem_of(sb, exclude_self)
    return attention_backward(prob, as_operand(sb.q), as_operand(sb.k), as_operand(sb.v), outputs, d_out_sorted,
                              scale)


def hash_scatter(o_sorted, q_idx):
    """out[..., q_idx[p], :] = o_sorted[..., p, :] in engine layout (hash_sparse.py:216-220)."""
    o_sorted = torch.as_tensor(o_sorted)
    B, H, T, D = o_sorted.shape
    idx = torch.as_tensor(q_idx, device=o_sorted.device)
    rank = torch.empty((B * H, T), dtype=torch.int32, device=o_sorted.device)
    err = torch.zeros(1, dtype=torch.int32, device=o_sorted.device)
    # idx is (B, H, T): element (b, s, h) at b*s0 + s*s2 + h*s1
    _lib.call("scfa_invert_index", _lib.ptr(idx), _lib.dtype_code(idx), B, T, H, idx.stride(0), idx.stride(2),
              idx.stride(1), T, _lib.ptr(rank), _lib.ptr(err), _lib.stream_ptr())
    return _scatter(o_sorted, rank, "bhtd")


@padded_call("attn")
def hash_sparse_attention(q, k, v, q_hash, k_hash, scale=None, blocks=BlockSpec(), exclude_self=True,
                          workers=None):
    """End-to-end hash-sparse attention in boundary layout (hash_sparse.py:223-238).

    The forward epilogue writes each sorted row straight back to its original
    position (hash_scatter + from_heads fused).
    """
    q, k, v = as_operand(q), as_operand(k), as_operand(v)
    sb = _sort_batch(q, k, v, q_hash, k_hash, "bthd", exclude_self=exclude_self)
    prob = _problem_of(sb, exclude_self)
    return attention_forward(prob, sb.q, sb.k, sb.v, scale, blocks, boundary=(q.shape[1], False), check=True).O


class _HashState:
    """What the backward stage needs from the forward stage."""

    __slots__ = ("prob", "sb", "q", "xq", "xk", "xv", "outputs", "rows", "q_only", "scale", "T_Q", "T_KV", "err",
                 "single_pass")


def _hash_forward_stage(q, k, v, q_hash, k_hash, scale=None, exclude_self=True, row_tables=False,
                        single_pass=False, q_ready=None):
    """Preparation + forward of the boundary-layout hash path; returns a _HashState.

    Default (shared ids): Q / K / V are put in bucket order without copy passes for Q:
    K / V are permuted up front (`scfa_permute_rows3`, on a side stream started as soon as
    the sort is final, under the finishing / tile-list kernels), the forward reads Q
    through the row table (tile::gather4, once per 128-row item) and writes the
    bucket-order Q copy back with TMA stores.  Separate query / key ids: Q / K / V are
    copied (tiled loads everywhere).  row_tables=True: every load goes through the row
    tables (no copies at all; tile::gather4 sustains only ~1.6 TB/s, scripts/gather_bw.cu).
    Nothing here synchronises with the host: bad bucket ids (sort kernels) and non-finite
    outputs (forward) are flagged in the device word st.err, which the caller reads once
    its launches are queued (check_status).
    q_ready: an event after which Q's data is on the device (the host-streaming call uploads Q
    after the ids, K and V; the preparation needs only Q's shape, so only the forward waits).
    """
    if q_ready is not None and (q.dtype != torch.bfloat16 or not q.is_contiguous()):
        torch.cuda.current_stream(q.device).wait_event(q_ready)  # as_operand converts: it reads Q
        q_ready = None
    q, k, v = as_operand(q), as_operand(k), as_operand(v)
    sorted_ev = torch.cuda.Event() if not row_tables else None
    err = torch.zeros(1, dtype=torch.int32, device=q.device)
    sb = _sort_batch(q, k, v, q_hash, k_hash, "bthd", check=False, exclude_self=exclude_self, materialize=False,
                     sorted_event=sorted_ev, err=err)
    prob = _problem_of(sb, exclude_self)
    st = _HashState()
    st.prob, st.sb, st.q, st.scale = prob, sb, q, scale
    st.T_Q, st.T_KV = q.shape[1], k.shape[1]
    st.rows, st.q_only, st.err = (prob.rows if row_tables else None), None, err
    st.single_pass = False
    if row_tables:
        st.xq, st.xk, st.xv = q, k, v
        prob.schedule("fwd", "dq", "dkdv")  # runs + all three tile lists in one pass
        if q_ready is not None:
            torch.cuda.current_stream(q.device).wait_event(q_ready)
        st.outputs = attention_forward(prob, q, k, v, scale, boundary=(st.T_Q, False), rows=st.rows, err=err)
        return st
    main = torch.cuda.current_stream(q.device)
    side = _copy_streams(q.device)[2]
    shared = sb.q_rank is not None and sb.k_rank is sb.q_rank
    if sorted_ev.cuda_event and shared:
        side.wait_event(sorted_ev)  # perm / rank final: copy under the rest of the preparation
    else:
        side.wait_stream(main)
    q_writeout = prob.rows is not None and shared and st.T_Q == st.T_KV and _Q_WRITEOUT
    if q_ready is not None and not q_writeout:
        side.wait_event(q_ready)  # the side stream copies Q too
    with torch.cuda.stream(side):
        if q_writeout:
            xk, xv = _permute3([k, v], [sb.k_rank, sb.k_rank], st.T_KV)
            xq = None
        elif sb.q_rank is not None and sb.k_rank is not None and st.T_Q == st.T_KV:
            xq, xk, xv = _permute3([q, k, v], [sb.q_rank, sb.k_rank, sb.k_rank], st.T_Q)
        else:
            xq, xk, xv = _gather3([q, k, v], [sb.q_perm, sb.k_perm, sb.k_perm], "bthd")
    # overlaps the copies; the single-pass backward needs no dQ list
    st.single_pass = bool(single_pass and q_writeout and q.shape[3] == 64)
    prob.schedule(*(("fwd", "dkdv") if st.single_pass else ("fwd", "dq", "dkdv")))
    main.wait_stream(side)
    if q_ready is not None:
        main.wait_event(q_ready)
    for t in (xq, xk, xv):
        if t is not None:
            t.record_stream(main)
    if q_writeout:
        B, H, D = q.shape[0], q.shape[2], q.shape[3]
        xq = torch.empty((B, H, st.T_Q, D), dtype=torch.bfloat16, device=q.device)
        st.q_only = RowTables(prob.rows.q_rows, None, prob.rows.R_q, prob.rows.R_kv)
        st.outputs = attention_forward(prob, q, xk, xv, scale, boundary=(st.T_Q, False), rows=st.q_only, q_out=xq,
                                       err=err)
    else:
        st.outputs = attention_forward(prob, xq, xk, xv, scale, boundary=(st.T_Q, False), err=err)
    st.xq, st.xk, st.xv = xq, xk, xv
    return st


def _hash_backward_stage(st, d_out):
    """dQ, dK, dV (fp32, boundary layout) for a _HashState and the output gradient."""
    from ._kernel import dkdv_backward_sorted, dq_backward_gathered

    d_out = as_operand(d_out)
    prob, sb = st.prob, st.sb
    if tuple(d_out.shape) != tuple(st.q.shape):  # dO rows are addressed like Q's (hash_sparse.py:182-213)
        raise ShapeError(f"dO shape {tuple(d_out.shape)} != Q shape {tuple(st.q.shape)}")
    if st.single_pass:
        # single pass: delta = rowsum(dO * O) with dO moved into bucket order (read in memory
        # order, written to each position's slot), then dQ, dK, dV in one key-stationary sweep
        from ._kernel import backward_single_pass

        B, T, H, D = st.q.shape
        Tq_pad = prob.Tq_pad
        xdo = torch.empty_like(st.xq)
        delta = torch.empty((B * H, Tq_pad), dtype=torch.float32, device=d_out.device)
        _lib.call("scfa_bwd_prep_rank", _lib.ptr(st.outputs.O), _lib.ptr(d_out), B, T, H, D, Tq_pad,
                  _lib.ptr(sb.q_rank), _lib.ptr(xdo), _lib.ptr(delta), _lib.stream_ptr())
        return backward_single_pass(prob, st.xq, st.xk, st.xv, xdo, st.outputs._lse2, delta, st.scale, st.T_Q,
                                    st.T_KV)
    if st.q_only is not None and _DO_WRITEOUT:
        # dQ gathers Q / dO through the row table, fuses delta and writes dO back in
        # bucket order for dK/dV: no separate delta / dO pass
        xdo = torch.empty_like(st.xq)
        dq, delta = dq_backward_gathered(prob, st.q, st.xk, st.xv, st.outputs, d_out, st.q_only, st.scale, st.T_Q,
                                         xdo, q_sorted=st.xq if _DQ_Q_SORTED else None)
        dk, dv = dkdv_backward_sorted(prob, st.xq, st.xk, st.xv, xdo, st.outputs._lse2, delta, st.scale, st.T_KV)
        return dq, dk, dv
    shared = sb.q_rank is not None and sb.k_rank is sb.q_rank
    return attention_backward(prob, st.xq, st.xk, st.xv, st.outputs, d_out, st.scale,
                              boundary=(st.T_Q, st.T_KV, False), rows=st.rows, q_rank=sb.q_rank if shared else None)


def _fwd_bwd(q, k, v, q_hash, k_hash, d_out, scale=None, exclude_self=True, row_tables=False, check=False,
             single_pass=False):
    """The fused boundary-layout fwd + bwd; returns (FlashOutputs, dq, dk, dv, problem).

    check=False (graph capture, the bench's device-resident step) leaves the status word
    unread; check=True reads it once after the backward is queued.  single_pass=True (D = 64,
    shared ids) runs the one-sweep backward (scfa_attn_bwd: dQ reduced in fp32, order
    varies); the default two-pass backward (dQ pass + dK/dV pass) is bitwise reproducible
    and measured as fast or faster."""
    st = _hash_forward_stage(q, k, v, q_hash, k_hash, scale, exclude_self, row_tables, single_pass)
    dq, dk, dv = _hash_backward_stage(st, d_out)
    if check:
        check_status(st.err)
    st.outputs._err = st.err
    return st.outputs, dq, dk, dv, st.prob


@padded_call("fwd_bwd")
def hash_sparse_attention_fwd_bwd(q, k, v, q_hash, k_hash, d_out, scale=None, exclude_self=True, row_tables=False,
                                  out=None, check=True, single_pass=False):
    """Forward + backward through the whole hash path, boundary layout in and out.

    Returns (O bf16, dQ, dK, dV fp32), each (B, T, H, D).  The reference
    composes the same from sort_by_bucket -> hash_forward_kernel ->
    hash_backward_kernel(dO sorted by q order) -> inverse permutation; here the
    inverse permutation is fused into the kernels' epilogues (each row is stored at
    its original position) and, with row_tables=True, the forward permutation into
    their TMA gather loads.

    Host (CPU) inputs are streamed: the batch is split per b and host->device copies,
    the attention and device->host copies of consecutive batch elements overlap on
    three CUDA streams (every (b, h) slice is independent, hash_sparse.py:223-238, so
    the results are those of one call).  `out` may give the four host result tensors
    (pinned memory keeps the copies asynchronous).  Host results are complete when the
    call returns.

    check=True (the reference's behaviour): negative bucket ids raise ShapeError
    (hash_sparse.py:112-113) and a non-finite output NumericError (softmax.py:63-64).
    Both are flagged on the device and read once, after every launch of the call is
    queued, so the check adds no bubble to the GPU timeline.

    single_pass=True: at D = 64 the backward is one key-stationary pass whose dQ is reduced
    in fp32 (reduction order varies run to run, ~1 ulp); the default two-pass backward is
    bitwise reproducible.
    """
    if not (isinstance(q, torch.Tensor) and not q.is_cuda):
        outputs, dq, dk, dv, _ = _fwd_bwd(q, k, v, q_hash, k_hash, d_out, scale, exclude_self, row_tables, check,
                                          single_pass)
        return outputs.O, dq, dk, dv
    return _fwd_bwd_host(q, k, v, q_hash, k_hash, d_out, scale, exclude_self, out, check, single_pass)


_COPY_STREAMS = {}


def _copy_streams(dev):
    """Persistent H2D / D2H / side-work streams per device (the caching allocator pools
    by stream: fresh streams per call would mean fresh cudaMalloc's every call)."""
    if dev not in _COPY_STREAMS:
        _COPY_STREAMS[dev] = (torch.cuda.Stream(dev), torch.cuda.Stream(dev), torch.cuda.Stream(dev))
    return _COPY_STREAMS[dev]


_TRACE = None  # diagnostics: a list receives (name, stream event) marks of the host-streaming timeline


def _mark(name, stream):
    if _TRACE is not None:
        e = torch.cuda.Event(enable_timing=True)
        e.record(stream)
        _TRACE.append((name, e))


def _fwd_bwd_host(q, k, v, q_hash, k_hash, d_out, scale, exclude_self, out, check=True, single_pass=False):
    """Host tensors in, host results out: batch elements streamed over three CUDA streams —
    upload, attention, download of consecutive elements overlap (every (b, h) slice is
    independent, hash_sparse.py:223-238, so the results equal one whole-batch call).

    The call is bound by the download of the fp32 gradients; what the link cannot hide is
    the lead before the first download.  So each element's Q / K / V / ids go up before its
    dO, the forward runs as soon as they are there, and O goes down while dO is still on
    its way and the backward runs (the gradients follow)."""
    dev = torch.device("cuda", torch.cuda.current_device())
    B, T, H, D = q.shape
    same = k_hash is q_hash
    q_hash, k_hash = torch.as_tensor(q_hash), torch.as_tensor(k_hash)
    if out is None:
        pin = torch.cuda.is_available()
        out = [torch.empty((B, T, H, D), dtype=torch.bfloat16, pin_memory=pin)] + [
            torch.empty((B, k.shape[1] if i else T, H, D), dtype=torch.float32, pin_memory=pin) for i in range(3)]
    comp = torch.cuda.current_stream(dev)
    h2d, d2h, _ = _copy_streams(dev)
    h2d.wait_stream(comp)
    d2h.wait_stream(comp)
    keep, errs = [], []
    for b in range(B):
        sl = slice(b, b + 1)
        with torch.cuda.stream(h2d):
            _mark(f"h2d{b}", h2d)
            # ids, K, V first: the sort, the K / V permute and the tile lists run while Q
            # is still on its way (the forward alone waits for it)
            ids, xk, xv = (t[sl].to(dev, non_blocking=True) for t in (q_hash, k, v))
            kh = ids if same else k_hash[sl].to(dev, non_blocking=True)
            ready_p = torch.cuda.Event()
            ready_p.record(h2d)
            xq = q[sl].to(dev, non_blocking=True)
            xs = [xq, xk, xv, ids]
            ready_f = torch.cuda.Event()
            ready_f.record(h2d)
            do_b = d_out[sl].to(dev, non_blocking=True)
            ready_b = torch.cuda.Event()
            ready_b.record(h2d)
            _mark(f"h2d{b}-end", h2d)
        comp.wait_event(ready_p)
        for t in xs + [kh, do_b]:
            t.record_stream(comp)
        _mark(f"fwd{b}", comp)
        st = _hash_forward_stage(xs[0], xs[1], xs[2], xs[3], kh, scale, exclude_self, single_pass=single_pass,
                                 q_ready=ready_f)
        fwd_done = torch.cuda.Event()
        fwd_done.record(comp)
        with torch.cuda.stream(d2h):
            d2h.wait_event(fwd_done)
            _mark(f"d2h{b}", d2h)
            out[0][sl].copy_(st.outputs.O, non_blocking=True)
            st.outputs.O.record_stream(d2h)
        comp.wait_event(ready_b)
        _mark(f"bwd{b}", comp)
        dq, dk, dv = _hash_backward_stage(st, do_b)
        st.outputs._err = st.err
        errs.append(st.err)
        _mark(f"bwd{b}-end", comp)
        done = torch.cuda.Event()
        done.record(comp)
        with torch.cuda.stream(d2h):
            d2h.wait_event(done)
            for dst, src in zip(out[1:], (dq, dk, dv)):
                dst[sl].copy_(src, non_blocking=True)
                src.record_stream(d2h)
            _mark(f"d2h{b}-end", d2h)
        keep.append((xs, kh, do_b, st, dq, dk, dv))
    comp.wait_stream(d2h)
    # the reference API is synchronous: the host results are complete on return
    comp.synchronize()
    if check:
        for e in errs:
            check_status(e)
    return tuple(out)
