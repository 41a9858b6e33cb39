"""QK-sparse attention: per-head query/key dropping on the GPU.

API mirror of pkg/src/scfa/qk_sparse.py.  Boundary tensors are (B, T, H, D)
with keep indicators (B, T, H); the kernels run on compacted engine-layout
operands (B, H, T_c, D) whose original positions travel in padded int32
index vectors (query pad -1, key pad 10**9, qk_sparse.py:1-8).

Device work per call: one compaction kernel per side (stable keep-first
order), one row-gather per operand fused with the (B,T,H,D)->(B,H,T,D)
transpose, the padded index vectors, the tcgen05 attention kernels, and one
scatter fused with the inverse transpose.  The only host synchronisation is
the read of the buffer sizes (max kept count), which the reference also
needs before it can allocate (qk_sparse.py:58).
"""

from typing import NamedTuple

import numpy as np
import torch

from . import _lib
from ._kernel import (
    RowTables,
    FlashOutputs,
    Problem,
    as_operand,
    attention_backward,
    attention_forward,
    check_forward_operands,
    check_status,
    pack_index,
    make_row_tables,
)
from .errors import ShapeError
from .tensors import DOMAIN_KEEP, KEY_PAD, QUERY_PAD, BlockSpec, pad128, stream
from ._headdim import padded_call

_OOB_Q = QUERY_PAD
_OOB_K = 0x7FFFFFFF


class CompactResult(NamedTuple):
    compact: torch.Tensor  # (B, buffer_size, H, D) boundary layout
    index: torch.Tensor  # (B, buffer_size, H) original positions
    indices_per_head: torch.Tensor  # (B, H) kept counts; None when index was given


class QkPrepared(NamedTuple):
    q_c: torch.Tensor  # (B, H, T_cq, D) bf16
    k_c: torch.Tensor  # (B, H, T_ck, D)
    v_c: torch.Tensor  # (B, H, T_ck, D)
    q_idx: torch.Tensor  # (B, H, T_cq) int32 padded positions
    k_idx: torch.Tensor  # (B, H, T_ck)
    scatter_index: torch.Tensor  # (B, T_cq, H) unpadded query gather order
    T_Q: int
    problem: object = None  # engine Problem (padded vectors, schedules)
    q_rank: torch.Tensor = None  # (B*H, T_Q) position -> slot
    k_rank: torch.Tensor = None  # (B*H, T_KV)
    copy_event: object = None  # fused path: K / V compacted on a side stream; join before the forward


def _keep_tensor(keep, shape, device):
    keep = torch.as_tensor(keep, device=device)
    if tuple(keep.shape) != tuple(shape):
        raise ShapeError(f"keep shape {tuple(keep.shape)} != {tuple(shape)}")
    return keep


def _compact_perm(keep, B, T, H, counts_out, err):
    """Run the compaction kernel; returns (perm, rank) as (B*H, T) int32."""
    dev = keep.device
    perm = torch.empty((B * H, T), dtype=torch.int32, device=dev)
    rank = torch.empty((B * H, T), dtype=torch.int32, device=dev)
    _lib.call("scfa_qk_compact", _lib.ptr(keep), _lib.dtype_code(keep), B, T, H,
              keep.stride(0), keep.stride(1), keep.stride(2),
              _lib.ptr(perm), _lib.ptr(rank), _lib.ptr(counts_out), _lib.ptr(err), _lib.stream_ptr())
    return perm, rank


def _gather(x_btHd, perm, n_slots):
    """(B, T, H, D) boundary tensor -> (B, H, n_slots, D) rows in `perm` order."""
    B, T, H, D = x_btHd.shape
    out = torch.empty((B, H, n_slots, D), dtype=x_btHd.dtype, device=x_btHd.device)
    _lib.call("scfa_gather_rows", _lib.ptr(x_btHd), x_btHd.element_size(), B, H, D,
              x_btHd.stride(0), x_btHd.stride(1), x_btHd.stride(2), _lib.ptr(perm), perm.shape[1],
              n_slots, _lib.ptr(out), _lib.stream_ptr())
    return out


def _aux(perm, counts, B, H, n_slots, pad, oob):
    T_pad = pad128(n_slots)
    out = torch.empty((B * H, T_pad), dtype=torch.int32, device=perm.device)
    _lib.call("scfa_build_aux", _lib.ptr(perm), _lib.ptr(counts), B, H, perm.shape[1], n_slots, T_pad,
              int(pad), int(oob), None, 0, 0, 0, 0, 0, None, 0, 0, 0, _lib.ptr(out), None, _lib.stream_ptr())
    return out


def compact(keep, x, index=None):
    """Gather kept rows of x (B, T, H, D) into a dense prefix per head (qk_sparse.py:41-71)."""
    x = as_operand(x) if not (isinstance(x, torch.Tensor) and x.is_cuda) else x.contiguous()
    B, T, H, D = x.shape
    dev = x.device
    if index is None:
        keep = _keep_tensor(keep, (B, T, H), dev)
        cnt = torch.zeros(B * H + 1, dtype=torch.int32, device=dev)
        perm, _ = _compact_perm(keep, B, T, H, cnt[: B * H], cnt[B * H:])
        host = cnt.cpu()
        if int(host[B * H]):
            raise ShapeError("keep entries must be 0 or 1")
        counts = host[: B * H].to(torch.int64).reshape(B, H)
        buffer = int(counts.max()) if counts.numel() else 0
        index = perm[:, :buffer].reshape(B, H, buffer).transpose(1, 2)
        counts_out = counts.to(dev)
    else:
        index = torch.as_tensor(index, device=dev)
        if index.dim() != 3 or index.shape[0] != B or index.shape[2] != H:
            raise ShapeError(f"index shape {tuple(index.shape)} incompatible with x")
        if index.numel() and (int(index.min()) < 0 or int(index.max()) >= T):
            raise ShapeError("supplied index out of range")
        buffer = index.shape[1]
        perm = index.transpose(1, 2).reshape(B * H, buffer).to(torch.int32).contiguous()
        counts_out = None
    g = _gather(x, perm, buffer)  # (B, H, buffer, D)
    return CompactResult(g.transpose(1, 2), index, counts_out)


def pad_index(index, indices_per_head, pad_idx):
    """Slots past each head's kept count -> pad_idx (qk_sparse.py:74-83); returns a copy."""
    index = torch.as_tensor(index)
    B, buf, H = index.shape
    counts = torch.as_tensor(indices_per_head, device=index.device)
    slot = torch.arange(buf, device=index.device).view(1, buf, 1)
    out = index.to(torch.int64).clone()
    out[slot >= counts.view(B, 1, H)] = int(pad_idx)
    return out


def qk_tile_schedule(q_idx, k_idx, blocks=BlockSpec()):
    """Reference j_stop per query block for one head's padded index vectors (qk_sparse.py:86-92)."""
    from ._kernel import causal_j_stops

    return causal_j_stops(q_idx, k_idx, blocks)


@padded_call("prep")
def qk_preprocess(q, k, v, q_keep, k_keep, materialize=True):
    """Compact, pad and transpose boundary-layout inputs (qk_sparse.py:196-211).

    materialize=False: no compacted copies; q_c / k_c / v_c are the (B, T, H, D) inputs
    and problem.rows holds the row tables the gather-mode kernels read them through.
    materialize="kv": compacted K / V only (q_c is the input Q, problem.rows set).
    """
    q, k, v = as_operand(q), as_operand(k), as_operand(v)
    if q.dim() != 4 or k.dim() != 4 or k.shape != v.shape:
        raise ShapeError(f"operand shapes disagree: {tuple(q.shape)}, {tuple(k.shape)}, {tuple(v.shape)}")
    B, T_Q, H, D = q.shape
    T_KV = k.shape[1]
    if T_KV >= KEY_PAD:
        raise ShapeError(f"T_KV must be < {KEY_PAD}")
    dev = q.device
    qk_ = _keep_tensor(q_keep, (B, T_Q, H), dev)
    kk_ = _keep_tensor(k_keep, (B, T_KV, H), dev)
    BH = B * H
    cnt = torch.zeros(2 * BH + 1, dtype=torch.int32, device=dev)
    q_perm, q_rank = _compact_perm(qk_, B, T_Q, H, cnt[:BH], cnt[2 * BH:])
    k_perm, k_rank = _compact_perm(kk_, B, T_KV, H, cnt[BH: 2 * BH], cnt[2 * BH:])
    host = cnt.cpu()  # the one host sync: buffer sizes
    if int(host[2 * BH]):
        raise ShapeError("keep entries must be 0 or 1")
    T_cq = int(host[:BH].max()) if BH else 0
    T_ck = int(host[BH: 2 * BH].max()) if BH else 0
    q_aux = _aux(q_perm, cnt[:BH], B, H, T_cq, QUERY_PAD, _OOB_Q)
    k_aux = _aux(k_perm, cnt[BH: 2 * BH], B, H, T_ck, KEY_PAD, _OOB_K)
    problem = Problem(B, H, T_cq, T_ck, D, q_aux, k_aux)
    if materialize == "kv":  # compacted K / V; Q stays in place behind the row tables
        q_c, k_c, v_c = q, _gather(k, k_perm, T_ck), _gather(v, k_perm, T_ck)
        problem.rows = make_row_tables(q_perm, k_perm, B, H, T_cq, T_ck, T_Q, T_KV, problem.Tq_pad, problem.Tkv_pad)
    elif materialize:
        q_c = _gather(q, q_perm, T_cq)
        k_c = _gather(k, k_perm, T_ck)
        v_c = _gather(v, k_perm, T_ck)
    else:
        q_c, k_c, v_c = q, k, v
        problem.rows = make_row_tables(q_perm, k_perm, B, H, T_cq, T_ck, T_Q, T_KV, problem.Tq_pad, problem.Tkv_pad)
    return QkPrepared(
        q_c=q_c, k_c=k_c, v_c=v_c,
        q_idx=q_aux[:, :T_cq].view(B, H, T_cq),
        k_idx=k_aux[:, :T_ck].view(B, H, T_ck),
        scatter_index=q_perm[:, :T_cq].view(B, H, T_cq).transpose(1, 2),
        T_Q=T_Q, problem=problem, q_rank=q_rank, k_rank=k_rank,
    )


_QK_PREP_MAX_T = 16384  # scfa_qk_prepare (one CTA per slice, both sides' prefix counts in shared memory)


def _prepare_static(q, k, v, q_keep, k_keep, err):
    """qk_preprocess for the fused paths with every size static: the compacted buffers hold
    T_Q / T_KV slots (kept rows first, in position order, then pad slots — QUERY_PAD /
    KEY_PAD in the index vectors, the dropped rows' data in the operands) instead of the
    reference's max kept count (qk_sparse.py:58), so nothing is read back to the host and
    the whole fwd + bwd can be captured in a CUDA graph.  Pad slots have empty visibility
    runs: no tile lists them, their outputs are zero.  Keep entries outside {0, 1} are
    flagged SCFA_ERR_SHAPE in the device status word `err` (qk_sparse.py:54-55).

    One launch (scfa_qk_prepare) builds perm / rank, the padded index vectors, the row
    tables and the visibility runs of both sides; the K / V compaction (one rank read per
    row, scfa_permute_rows3) then runs on a side stream under the tile-list build — the
    caller joins it (`prep.copy_event`) before the forward."""
    B, T_Q, H, D = q.shape
    T_KV = k.shape[1]
    if T_KV >= KEY_PAD:
        raise ShapeError(f"T_KV must be < {KEY_PAD}")
    dev = q.device
    qk_ = _keep_tensor(q_keep, (B, T_Q, H), dev)
    kk_ = _keep_tensor(k_keep, (B, T_KV, H), dev)
    BH = B * H
    contiguous_kv = k.stride(3) == 1 and k.is_contiguous() and v.is_contiguous()
    if T_Q > _QK_PREP_MAX_T or T_KV > _QK_PREP_MAX_T or BH > 65535 or not contiguous_kv:
        return _prepare_static_passes(q, k, v, qk_, kk_, err)
    Tq_pad, Tkv_pad = pad128(T_Q), pad128(T_KV)
    i32 = dict(dtype=torch.int32, device=dev)
    perm_q, rank_q = torch.empty((BH, T_Q), **i32), torch.empty((BH, T_Q), **i32)
    perm_k, rank_k = torch.empty((BH, T_KV), **i32), torch.empty((BH, T_KV), **i32)
    q_aux, k_aux = torch.empty((BH, Tq_pad), **i32), torch.empty((BH, Tkv_pad), **i32)
    q_runs, k_runs = torch.empty((BH, Tq_pad, 2), **i32), torch.empty((BH, Tkv_pad, 2), **i32)
    q_rows, k_rows = torch.empty((BH, Tq_pad), **i32), torch.empty((BH, Tkv_pad), **i32)
    cnt = torch.empty(2 * BH, **i32)
    _lib.call("scfa_qk_prepare", _lib.ptr(qk_), _lib.dtype_code(qk_), *qk_.stride(), _lib.ptr(kk_),
              _lib.dtype_code(kk_), *kk_.stride(), B, T_Q, T_KV, H, _lib.ptr(perm_q), _lib.ptr(rank_q),
              _lib.ptr(perm_k), _lib.ptr(rank_k), _lib.ptr(q_aux), _lib.ptr(k_aux), _lib.ptr(q_runs),
              _lib.ptr(k_runs), _lib.ptr(q_rows), _lib.ptr(k_rows), _lib.ptr(cnt), _lib.ptr(err), _lib.stream_ptr())
    problem = Problem(B, H, T_Q, T_KV, D, q_aux, k_aux)
    problem.set_runs(q_runs, k_runs)
    problem.rows = RowTables(q_rows, k_rows, B * T_Q * H, B * T_KV * H)
    # every key position has a slot: K / V rows move in memory order to their slots, on a
    # side stream under the tile-list build
    from .hash_sparse import _copy_streams, _permute3

    main = torch.cuda.current_stream(dev)
    side = _copy_streams(dev)[2]
    side.wait_stream(main)
    with torch.cuda.stream(side):
        k_c, v_c = _permute3([k, v], [rank_k, rank_k], T_KV)
        ev = torch.cuda.Event()
        ev.record(side)
    for t in (k_c, v_c):
        t.record_stream(main)
    prep = QkPrepared(
        q_c=q, k_c=k_c, v_c=v_c,
        q_idx=q_aux[:, :T_Q].view(B, H, T_Q), k_idx=k_aux[:, :T_KV].view(B, H, T_KV),
        scatter_index=perm_q.view(B, H, T_Q).transpose(1, 2),
        T_Q=T_Q, problem=problem, q_rank=rank_q, k_rank=rank_k, copy_event=ev,
    )
    return prep


def _prepare_static_passes(q, k, v, qk_, kk_, err):
    """_prepare_static as separate passes (compaction per side, aux vectors, row maps; the
    runs come from scfa_build_schedule): T above scfa_qk_prepare's limit or strided K / V."""
    B, T_Q, H, D = q.shape
    T_KV = k.shape[1]
    dev = q.device
    BH = B * H
    cnt = torch.empty(2 * BH, dtype=torch.int32, device=dev)
    q_perm, q_rank = _compact_perm(qk_, B, T_Q, H, cnt[:BH], err)
    k_perm, k_rank = _compact_perm(kk_, B, T_KV, H, cnt[BH:], err)
    q_aux = _aux(q_perm, cnt[:BH], B, H, T_Q, QUERY_PAD, _OOB_Q)
    k_aux = _aux(k_perm, cnt[BH:], B, H, T_KV, KEY_PAD, _OOB_K)
    problem = Problem(B, H, T_Q, T_KV, D, q_aux, k_aux)
    if k.stride(3) == 1 and k.is_contiguous() and v.is_contiguous():
        from .hash_sparse import _permute3

        k_c, v_c = _permute3([k, v], [k_rank, k_rank], T_KV)
    else:
        k_c, v_c = _gather(k, k_perm, T_KV), _gather(v, k_perm, T_KV)
    problem.rows = make_row_tables(q_perm, k_perm, B, H, T_Q, T_KV, T_Q, T_KV, problem.Tq_pad, problem.Tkv_pad)
    prep = QkPrepared(
        q_c=q, k_c=k_c, v_c=v_c,
        q_idx=q_aux[:, :T_Q].view(B, H, T_Q), k_idx=k_aux[:, :T_KV].view(B, H, T_KV),
        scatter_index=q_perm.view(B, H, T_Q).transpose(1, 2),
        T_Q=T_Q, problem=problem, q_rank=q_rank, k_rank=k_rank,
    )
    return prep


def _problem_from(q_c, k_c, q_idx, k_idx, validate=True):
    check_forward_operands(q_c, k_c, k_c)
    B, H, T_Q, D = q_c.shape
    T_KV = k_c.shape[2]
    dev = q_c.device
    pq = pack_index(q_idx, B * H, T_Q, _OOB_Q, dev)
    pk = pack_index(k_idx, B * H, T_KV, _OOB_K, dev)
    prob = Problem(B, H, T_Q, T_KV, D, pq, pk)
    if validate and B * H:
        prob.validate("qk")
    return prob


@padded_call("qk_fwd")
def qk_forward_kernel(q_c, k_c, v_c, q_idx, k_idx, scale=None, blocks=BlockSpec(), workers=None):
    """Irregular-causal forward over compacted operands (qk_sparse.py:120-148)."""
    q_c, k_c, v_c = as_operand(q_c), as_operand(k_c), as_operand(v_c)
    check_forward_operands(q_c, k_c, v_c)
    B, H, T_Q, _ = q_c.shape
    if tuple(torch.as_tensor(q_idx).shape) != (B, H, T_Q) or tuple(torch.as_tensor(k_idx).shape) != (
            B, H, k_c.shape[2]):
        raise ShapeError("index tensors do not match the compacted operands")
    prob = _problem_from(q_c, k_c, q_idx, k_idx)
    return attention_forward(prob, q_c, k_c, v_c, scale, blocks, check=True)


@padded_call("qk_bwd")
def qk_backward_kernel(q_c, k_c, v_c, outputs, d_out_c, q_idx, k_idx, scale=None, blocks=BlockSpec(),
                       workers=None):
    """Gradients w.r.t. compacted operands, fp32 (qk_sparse.py:151-183)."""
    q_c, k_c, v_c = as_operand(q_c), as_operand(k_c), as_operand(v_c)
    check_forward_operands(q_c, k_c, v_c)
    if tuple(d_out_c.shape) != tuple(q_c.shape):
        raise ShapeError(f"dO shape {tuple(d_out_c.shape)} != {tuple(q_c.shape)}")
    prob = getattr(outputs, "_problem", None)
    if prob is None or prob.T_q != q_c.shape[2] or prob.T_kv != k_c.shape[2]:
        prob = _problem_from(q_c, k_c, q_idx, k_idx)
    return attention_backward(prob, q_c, k_c, v_c, outputs, d_out_c, scale)


def _scatter(o_kernel, rank, T_Q, out_dtype=None):
    """(B, H, T_c, D) -> (B, T_Q, H, D); positions whose slot is >= T_c get zeros."""
    B, H, T_c, D = o_kernel.shape
    o_kernel = o_kernel.contiguous()
    dt = out_dtype or o_kernel.dtype
    out = torch.empty((B, T_Q, H, D), dtype=dt, device=o_kernel.device)
    _lib.call("scfa_scatter_rows", _lib.ptr(o_kernel), o_kernel.element_size(), B, H, T_Q, D,
              _lib.ptr(rank), T_c, _lib.ptr(out), out.element_size(),
              out.stride(0), out.stride(1), out.stride(2), _lib.stream_ptr())
    return out


def _rank_from_index(scatter_index, T_Q):
    idx = torch.as_tensor(scatter_index)
    B, T_c, H = idx.shape
    rank = torch.empty((B * H, T_Q), dtype=torch.int32, device=idx.device)
    err = torch.zeros(1, dtype=torch.int32, device=idx.device)
    _lib.call("scfa_invert_index", _lib.ptr(idx), _lib.dtype_code(idx), B, T_c, H,
              idx.stride(0), idx.stride(1), idx.stride(2), T_Q, _lib.ptr(rank), _lib.ptr(err), _lib.stream_ptr())
    return rank


def qk_postprocess(o_kernel, scatter_index, T_Q, rank=None):
    """Scatter kernel outputs back to (B, T, H, D); dropped rows are zero (qk_sparse.py:214-225)."""
    o_kernel = torch.as_tensor(o_kernel)
    if rank is None:
        rank = _rank_from_index(scatter_index, T_Q)
    return _scatter(o_kernel, rank, T_Q)


@padded_call("attn")
def qk_sparse_attention(q, k, v, q_keep, k_keep, scale=None, blocks=BlockSpec(), workers=None):
    """End-to-end QK-sparse attention in boundary layout (qk_sparse.py:228-239).

    The forward epilogue writes every kept query row straight to its original
    position (the inverse scatter of qk_postprocess is fused); dropped rows are zero.
    """
    prep = qk_preprocess(q, k, v, q_keep, k_keep)
    return attention_forward(prep.problem, prep.q_c, prep.k_c, prep.v_c, scale, blocks,
                             boundary=(prep.T_Q, True), check=True).O


class _QkState:
    """What the QK backward stage needs from the forward stage."""

    __slots__ = ("prob", "prep", "q", "xq", "outputs", "rows", "q_only", "scale", "T_Q", "T_KV", "q_keep", "k_keep",
                 "err", "static")


def _qk_forward_stage(q, k, v, q_keep, k_keep, scale=None, row_tables=False):
    """Preparation + forward of the boundary-layout QK path; returns a _QkState.

    Default: static sizes (_prepare_static, no host synchronisation, graph-capturable);
    only K / V are compacted up front; the forward reads Q through the row table and writes
    the compacted Q back (as the hash path).  row_tables=True: the reference's sizing (one
    read-back of the kept counts) and every load through the row tables.  Dropped rows of O
    are zeroed here (not zero-filled up front).
    """
    st = _QkState()
    st.T_Q, st.T_KV, st.scale, st.q_keep, st.k_keep = q.shape[1], k.shape[1], scale, q_keep, k_keep
    st.q_only, st.xq, st.rows = None, None, None
    q, k, v = as_operand(q), as_operand(k), as_operand(v)
    if q.dim() != 4 or k.dim() != 4 or k.shape != v.shape or q.shape[0] != k.shape[0] or q.shape[2:] != k.shape[2:]:
        raise ShapeError(f"operand shapes disagree: {tuple(q.shape)}, {tuple(k.shape)}, {tuple(v.shape)}")
    st.err = torch.zeros(1, dtype=torch.int32, device=q.device)
    st.static = False
    if row_tables:
        st.prep, mode = qk_preprocess(q, k, v, q_keep, k_keep, materialize=False), "rows"
    elif st.T_Q == 0:
        st.prep, mode = qk_preprocess(q, k, v, q_keep, k_keep), "sorted"
    else:
        st.prep, mode = _prepare_static(q, k, v, q_keep, k_keep, st.err), "gathered"
        st.static = True
    st.prob = prob = st.prep.problem
    prob.schedule("fwd", "dq", "dkdv")
    if getattr(st.prep, "copy_event", None) is not None:
        torch.cuda.current_stream(q.device).wait_event(st.prep.copy_event)  # K / V compacted
    st.q = q
    if mode == "gathered":
        st.q_only = RowTables(prob.rows.q_rows, None, prob.rows.R_q, prob.rows.R_kv)
        st.xq = torch.empty((prob.B, prob.H, prob.T_q, prob.D), dtype=torch.bfloat16, device=st.q.device)
        st.outputs = attention_forward(prob, st.q, st.prep.k_c, st.prep.v_c, scale, boundary=(st.T_Q, False),
                                       rows=st.q_only, q_out=st.xq, err=st.err)
    else:
        st.rows = prob.rows if mode == "rows" else None
        st.outputs = attention_forward(prob, st.prep.q_c, st.prep.k_c, st.prep.v_c, scale,
                                       boundary=(st.T_Q, False), rows=st.rows, err=st.err)
    if not st.static:
        # static sizing: every dropped position has a pad slot whose (zero) output row the
        # epilogue writes through the row table, so nothing is left to clear
        _zero_dropped_rows(q_keep, st.outputs.O)
    return st


def _qk_backward_stage(st, d_out):
    """dQ, dK, dV (fp32, boundary layout; dropped rows zero) for a _QkState."""
    from ._kernel import dkdv_backward_sorted, dq_backward_gathered

    prob, prep = st.prob, st.prep
    d_b = as_operand(d_out)
    if tuple(d_b.shape) != tuple(st.q.shape):  # the kernels address dO like Q (qk_sparse.py:151-183)
        raise ShapeError(f"dO shape {tuple(d_b.shape)} != Q shape {tuple(st.q.shape)}")
    if st.q_only is not None:
        xdo = torch.empty_like(st.xq)
        from .hash_sparse import _DQ_Q_SORTED

        dq, delta = dq_backward_gathered(prob, st.q, prep.k_c, prep.v_c, st.outputs, d_b, st.q_only, st.scale,
                                         st.T_Q, xdo, q_sorted=st.xq if _DQ_Q_SORTED else None)
        dk, dv = dkdv_backward_sorted(prob, st.xq, prep.k_c, prep.v_c, xdo, st.outputs._lse2, delta, st.scale,
                                      st.T_KV, out_rows=prob.rows.k_rows if st.static else None)
    else:
        dq, dk, dv = attention_backward(prob, prep.q_c, prep.k_c, prep.v_c, st.outputs, d_b, st.scale,
                                        boundary=(st.T_Q, st.T_KV, False), rows=st.rows)
    if not st.static:  # (static: pad slots wrote the dropped rows' zeros)
        _zero_dropped_rows(st.q_keep, dq)
        _zero_dropped(st.k_keep, dk, dv)
    return dq, dk, dv


@padded_call("fwd_bwd")
def qk_sparse_attention_fwd_bwd(q, k, v, q_keep, k_keep, d_out, scale=None, row_tables=False, check=True):
    """Forward + backward through the whole QK path in boundary layout.

    Returns (O bf16, dQ, dK, dV fp32), all (B, T, H, D); dropped positions get
    zero outputs and zero gradients.  The reference composes the same thing
    from qk_preprocess -> qk_forward_kernel -> qk_backward_kernel.  check=True reads
    the device status word once, after every launch is queued, and raises
    NumericError for a non-finite output (softmax.py:63-64).
    """
    st = _qk_forward_stage(q, k, v, q_keep, k_keep, scale, row_tables)
    dq, dk, dv = _qk_backward_stage(st, d_out)
    if check:
        check_status(st.err, "keep entries must be 0 or 1")
    return st.outputs.O, dq, dk, dv


def _zero_dropped_rows(keep, out):
    B, T, H, D = out.shape
    keep = torch.as_tensor(keep, device=out.device)
    _lib.call("scfa_zero_dropped", _lib.ptr(keep), _lib.dtype_code(keep), B, T, H, *keep.stride(), _lib.ptr(out),
              D * out.element_size(), None, 0, _lib.stream_ptr())


def _zero_dropped(keep, out0, out1):
    B, T, H, D = out0.shape
    keep = torch.as_tensor(keep, device=out0.device)
    _lib.call("scfa_zero_dropped", _lib.ptr(keep), _lib.dtype_code(keep), B, T, H, *keep.stride(), _lib.ptr(out0),
              D * out0.element_size(), _lib.ptr(out1), D * out1.element_size(), _lib.stream_ptr())


def random_keep(B, T, H, drop_prob, seed):
    """Keep indicators with drop probability drop_prob, same stream as qk_sparse.py:242-247 (numpy)."""
    if not 0.0 <= drop_prob <= 1.0:
        raise ShapeError(f"drop probability must be in [0, 1], got {drop_prob}")
    g = stream(seed, DOMAIN_KEEP)
    return (g.random((B, T, H)) >= drop_prob).astype(np.float64)
