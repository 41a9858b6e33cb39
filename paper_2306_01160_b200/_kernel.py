"""The shared tile engine: problem description, schedules, fwd/bwd launches.

Counterpart of pkg/src/scfa/_kernel.py.  The reference runs one NumPy tile
loop per (b, h) (``forward_head`` :92-123, ``backward_head`` :139-193) over a
contiguous key-block range per query block (``causal_j_stops`` :45-53,
``hash_tile_ranges`` :56-79).  Here a :class:`Problem` carries the padded
int32 index / bucket vectors of every (b, h) slice, builds exact tile lists
on the device, and launches the tcgen05 kernels of
``csrc/scfa_attn.cu`` through the C ABI.
"""

import ctypes

import torch

from . import _lib
from .errors import ShapeError
from .tensors import BlockSpec, default_scale, pad128


class FlashOutputs:
    """Forward results (``_kernel.py:18-30``).

    O (B, H, T_Q, D) bf16, normalised output; M (B, H, T_Q) f32 running max of
    the scaled logits (-inf for stranded queries); L (B, H, T_Q) f32 softmax
    denominator relative to M (0 for stranded queries).  ``tiles_computed``
    is the reference schedule's tile count at the caller's BlockSpec,
    computed on first access; ``tiles_executed`` counts the 128x128 tiles the
    kernel actually ran.
    """

    def __init__(self, O, M, L, tiles_computed=None, *, problem=None, blocks=None, lse2=None):
        self.O = O
        self.M = M
        self.L = L
        self._tiles = tiles_computed
        self._problem = problem
        self._blocks = blocks if blocks is not None else BlockSpec()
        self._lse2 = lse2

    @property
    def tiles_computed(self):
        if self._tiles is None:
            self._tiles = self._problem.ref_tiles(self._blocks) if self._problem is not None else 0
        return self._tiles

    @tiles_computed.setter
    def tiles_computed(self, v):
        self._tiles = v

    @property
    def tiles_executed(self):
        return self._problem.executed_tiles() if self._problem is not None else 0

    def __repr__(self):
        return f"FlashOutputs(O={tuple(self.O.shape)}, tiles_computed={self.tiles_computed})"


class Problem:
    """Index/bucket vectors of all (b, h) slices, padded to 128 per slice.

    q_idx (B*H, Tq_pad) / k_idx (B*H, Tkv_pad) int32 carry original positions
    (QUERY_PAD/KEY_PAD in pad slots, sentinels past the end); q_hash/k_hash
    carry bucket ids when ``flags`` has FLAG_HASH.
    """

    def __init__(self, B, H, T_q, T_kv, D, q_idx, k_idx, q_hash=None, k_hash=None, flags=0):
        self.B, self.H, self.T_q, self.T_kv, self.D = int(B), int(H), int(T_q), int(T_kv), int(D)
        self.q_idx, self.k_idx, self.q_hash, self.k_hash = q_idx, k_idx, q_hash, k_hash
        self.flags = int(flags)
        self.rows = None  # RowTables for gather-mode kernels, when the operands stay in (B, T, H, D)
        self._lists = {}

    @property
    def BH(self):
        return self.B * self.H

    @property
    def Tq_pad(self):
        return pad128(self.T_q)

    @property
    def Tkv_pad(self):
        return pad128(self.T_kv)

    def set_runs(self, q_runs, k_runs):
        """Adopt visibility runs computed elsewhere (scfa_hash_prepare) for this problem's flags."""
        self._lists["q_runs"] = q_runs
        self._lists["k_runs"] = k_runs

    def _hash_ptrs(self):
        if self.flags & _lib.FLAG_HASH:
            return _lib.ptr(self.q_hash), _lib.ptr(self.k_hash)
        return _lib.ptr(self.q_idx), _lib.ptr(self.k_idx)

    @property
    def _tiles_total(self):
        """Listed tiles per list (fwd, dq, dkdv; int64, device), summed from the counts on
        demand (the list kernel keeps no running total: no fill launch, no atomics)."""
        parts = []
        for name in ("fwd", "dq", "dkdv"):
            ent = self._lists.get(name)
            parts.append(ent[1].sum(dtype=torch.int64) if ent is not None
                         else torch.zeros((), dtype=torch.int64, device=self.q_idx.device))
        return torch.stack(parts)

    # list name -> (rows are queries, streamed tile width, tiles_total slot)
    LISTS = {"fwd": (True, 128, 0), "dq": (True, 64, 1), "dkdv": (False, 64, 2)}

    def schedule(self, *which):
        """Visibility runs + exact tile lists (scfa_build_schedule), built once per Problem.

        Returns {name: (list, count, stride)} for the requested lists plus the
        runs under "q_runs" / "k_runs".
        """
        which = which or tuple(self.LISTS)
        want = [w for w in which if w not in self._lists]
        if want:
            dev = self.q_idx.device
            ready = (1 if "q_runs" in self._lists else 0) | (2 if "k_runs" in self._lists else 0)
            if any(self.LISTS[w][0] for w in want) and "q_runs" not in self._lists:
                self._lists["q_runs"] = torch.empty((self.BH, self.Tq_pad, 2), dtype=torch.int32, device=dev)
            if any(not self.LISTS[w][0] for w in want) and "k_runs" not in self._lists:
                self._lists["k_runs"] = torch.empty((self.BH, self.Tkv_pad, 2), dtype=torch.int32, device=dev)
            args = []
            for name in ("fwd", "dq", "dkdv"):
                rq, cb, _ = self.LISTS[name]
                if name in want:
                    T_rows = self.T_q if rq else self.T_kv
                    T_cols = self.T_kv if rq else self.T_q
                    n_rb = max(-(-T_rows // 128), 1)
                    stride = max(-(-T_cols // cb), 1)
                    lst = torch.empty((self.BH, n_rb, stride), dtype=torch.int16, device=dev)
                    # counts (BH, n_rb), the attention kernels' work counter pair, then the item
                    # order (longest first, {item, count} pairs, 8-byte aligned); the list
                    # kernels write all of it (no fill launch)
                    n_it = self.BH * n_rb
                    cnt = torch.empty(3 * n_it + 4, dtype=torch.int32, device=dev)[:n_it].view(
                        self.BH, n_rb)  # same base address; pair and order live past the view
                    self._lists[name] = (lst, cnt, stride)
                    args += [_lib.ptr(lst), _lib.ptr(cnt), stride]
                else:
                    args += [None, None, 0]
            qh, kh = self._hash_ptrs()
            _lib.call(
                "scfa_build_schedule",
                _lib.ptr(self.q_idx), qh, _lib.ptr(self.k_idx), kh,
                self.BH, self.T_q, self.T_kv, self.Tq_pad, self.Tkv_pad, self.flags,
                _lib.ptr(self._lists.get("q_runs")), _lib.ptr(self._lists.get("k_runs")), ready,
                *args, None, _lib.stream_ptr(),
                kernels=(0 if ready == 3 else 1) + 2,
            )
        return self._lists

    def executed_tiles(self):
        """128x128 tiles run by the forward kernel (non-empty tiles only)."""
        self.schedule("fwd")
        return int(self._tiles_total[0].item())

    def ref_schedule(self, blocks=BlockSpec()):
        """Reference per-query-block ranges at BlockSpec granularity (all heads)."""
        nQ = blocks.query_blocks(self.T_q) if self.T_q else 0
        dev = self.q_idx.device
        js = torch.zeros((self.BH, nQ), dtype=torch.int32, device=dev)
        je = torch.zeros((self.BH, nQ), dtype=torch.int32, device=dev)
        tiles = torch.zeros(self.BH, dtype=torch.int64, device=dev)
        qh, kh = self._hash_ptrs()
        _lib.call(
            "scfa_ref_schedule",
            _lib.ptr(self.q_idx), qh, _lib.ptr(self.k_idx), kh,
            self.BH, self.T_q, self.T_kv, self.Tq_pad, self.Tkv_pad,
            int(blocks.B_m), int(blocks.B_n), self.flags,
            _lib.ptr(js), _lib.ptr(je), _lib.ptr(tiles), _lib.stream_ptr(),
        )
        return js, je, tiles

    def ref_tiles(self, blocks=BlockSpec()):
        if self.BH == 0 or self.T_q == 0:
            return 0
        return int(self.ref_schedule(blocks)[2].sum().item())

    def validate(self, kind):
        err = torch.zeros(1, dtype=torch.int32, device=self.q_idx.device)
        if kind == "qk":
            _lib.call("scfa_validate_qk", _lib.ptr(self.q_idx), _lib.ptr(self.k_idx), self.BH,
                      self.T_q, self.T_kv, self.Tq_pad, self.Tkv_pad, _lib.ptr(err), _lib.stream_ptr())
        else:
            for idx, hsh, T, Tp in ((self.q_idx, self.q_hash, self.T_q, self.Tq_pad),
                                    (self.k_idx, self.k_hash, self.T_kv, self.Tkv_pad)):
                _lib.call("scfa_validate_sorted", _lib.ptr(idx), _lib.ptr(hsh), self.BH, T, Tp,
                          _lib.ptr(err), _lib.stream_ptr())
        code = int(err.item())
        if code:
            what = ("indices must be strictly increasing with pads forming the tail"
                    if kind == "qk" else "bucket ids must be non-decreasing and positions increase within a bucket")
            _lib.raise_for(code, what)


def pack_index(x, BH, T, oob, device):
    """Caller index tensor (B, H, T) of any int dtype -> padded int32 (BH, T_pad)."""
    x = torch.as_tensor(x, device=device)
    if x.dim() != 3 or x.shape[0] * x.shape[1] != BH or x.shape[2] != T:
        raise ShapeError(f"index tensor of shape {tuple(x.shape)} does not match ({BH} heads, T={T})")
    x2 = x.reshape(BH, T)
    out = torch.empty((BH, pad128(T)), dtype=torch.int32, device=device)
    _lib.call("scfa_pack_index", _lib.ptr(x2), _lib.dtype_code(x2), BH, T, x2.stride(0), x2.stride(1),
              pad128(T), int(oob), _lib.ptr(out), _lib.stream_ptr())
    return out


def as_operand(x, device=None):
    """Engine operand: CUDA bf16, contiguous (numpy arrays are uploaded)."""
    if not isinstance(x, torch.Tensor):
        x = torch.as_tensor(x)
    if device is None:
        device = x.device if x.is_cuda else torch.device("cuda")
    if x.device != torch.device(device) or x.dtype != torch.bfloat16:
        x = x.to(device=device, dtype=torch.bfloat16)
    return x.contiguous()


def check_forward_operands(q, k, v):
    if q.dim() != 4 or k.dim() != 4 or v.dim() != 4:
        raise ShapeError("attention operands must be 4-D (B, H, T, D)")
    if q.shape[:2] != k.shape[:2] or k.shape != v.shape or q.shape[3] != k.shape[3]:
        raise ShapeError(f"operand shapes disagree: {tuple(q.shape)}, {tuple(k.shape)}, {tuple(v.shape)}")


def _scale(scale, D):
    return float(default_scale(D) if scale is None else scale)


def _zeros_or_empty(shape, dtype, dev, zero):
    return torch.zeros(shape, dtype=dtype, device=dev) if zero else torch.empty(shape, dtype=dtype, device=dev)


class RowTables:
    """Gather-mode addressing (scfa_row_map): slot s of slice bh lives at row q_rows[bh, s]
    of the caller's (B, T_Q, H, D) tensor viewed as [B*T_Q*H, D] (k_rows likewise)."""

    def __init__(self, q_rows, k_rows, R_q, R_kv):
        self.q_rows, self.k_rows, self.R_q, self.R_kv = q_rows, k_rows, int(R_q), int(R_kv)

    def args(self):
        return [_lib.ptr(self.q_rows), _lib.ptr(self.k_rows), self.R_q, self.R_kv]


_NO_ROWS = [None, None, 0, 0]


def check_status(err, what="attention"):
    """Raise the reference error class for a device status word (int32, 0 = ok).

    The engine's kernels report data-dependent failures through one device word instead
    of aborting: SCFA_ERR_SHAPE for bad bucket ids / keep entries (hash_sparse.py:112-113,
    qk_sparse.py:54-55), SCFA_ERR_NUMERIC for a non-finite output (softmax.py:63-64).
    Reading it synchronises with the stream, so the public calls read it once, after
    every launch of the call is queued."""
    if err is None:
        return
    code = int(err.item())
    if code:
        msgs = {_lib.ERR_SHAPE: "bucket ids must be non-negative (and < 2**31)",
                _lib.ERR_NUMERIC: "non-finite values in attention output (update_stats, softmax.py:63-64)"}
        if what != "attention" and code == _lib.ERR_SHAPE:
            msgs[code] = what
        _lib.raise_for_status(code, msgs.get(code, what))


def attention_forward(problem, q, k, v, scale=None, blocks=None, boundary=None, rows=None, q_out=None, err=None,
                      check=False):
    """Launch the forward kernel over the exact tile list; returns FlashOutputs.

    boundary=None: O is engine layout (B, H, T_q, D) in kernel (sorted/compacted) order.
    boundary=(T_out, zero_fill): the epilogue writes each row straight to its original
    position of a (B, T_out, H, D) tensor (fused inverse scatter); positions no row maps
    to are zero-filled first when zero_fill (QK drops).  M, L stay in kernel order.
    rows=RowTables: q, k, v are the caller's (B, T, H, D) tensors, read by TMA gather4
    through the row tables (no sorted copies); requires boundary.  With rows.k_rows None
    the keys / values are kernel-order copies (tiled loads) and only Q is gathered;
    q_out (B, H, T_q, D) bf16 then receives the gathered Q in kernel order.
    err: int32 device status word the kernel flags SCFA_ERR_NUMERIC in; check=True reads
    it after the launch and raises NumericError (reference update_stats, softmax.py:63-64).
    """
    if rows is not None:
        B, T_in, H, D = q.shape
        T_q, T_kv = problem.T_q, problem.T_kv
    else:
        B, H, T_q, D = q.shape
        T_kv = k.shape[2]
    dev = q.device
    if boundary is None:
        O = torch.empty((B, H, T_q, D), dtype=torch.bfloat16, device=dev)
        T_out, out_b = T_q, 0
    else:
        T_out, zero = boundary
        O = _zeros_or_empty((B, T_out, H, D), torch.bfloat16, dev, zero)
        out_b = 1
    M = torch.empty((B, H, T_q), dtype=torch.float32, device=dev)
    L = torch.empty((B, H, T_q), dtype=torch.float32, device=dev)
    lse2 = torch.empty((B * H, pad128(T_q)), dtype=torch.float32, device=dev)
    if check and err is None:
        err = torch.zeros(1, dtype=torch.int32, device=dev)
    if B * H > 0 and T_q > 0:
        sched = problem.schedule("fwd")
        lst, cnt, stride = sched["fwd"]
        _lib.call(
            "scfa_attn_fwd",
            _lib.ptr(q), _lib.ptr(k), _lib.ptr(v), B * H, T_q, T_kv, D,
            _lib.ptr(problem.q_idx), _lib.ptr(sched["q_runs"]), problem.Tq_pad, problem.Tkv_pad,
            _lib.ptr(lst), _lib.ptr(cnt), stride, _scale(scale, D), H, T_out, out_b,
            _lib.ptr(O), _lib.ptr(M), _lib.ptr(L), _lib.ptr(lse2),
            *(rows.args() if rows is not None else _NO_ROWS), _lib.ptr(q_out), _lib.ptr(err), _lib.stream_ptr(),
        )
    out = FlashOutputs(O, M, L, problem=problem, blocks=blocks, lse2=lse2)
    out._boundary = boundary
    if check:
        check_status(err)
    return out


def attention_backward(problem, q, k, v, outputs, d_out, scale=None, boundary=None, rows=None, q_rank=None):
    """dQ, dK, dV (fp32) recomputing P from the saved statistics.

    boundary=None: d_out and outputs.O are engine layout in kernel order and the
    gradients come back the same way.  boundary=(T_q_out, T_kv_out, zero_fill):
    outputs.O and d_out are (B, T_q_out, H, D); dO is gathered into kernel order
    inside the delta pass, and dQ / dK / dV are written straight to their original
    positions of (B, T_*_out, H, D) fp32 tensors.  rows=RowTables: as attention_forward
    (q, k, v, d_out, outputs.O all (B, T, H, D)); the delta pass is fused into the dQ
    kernel and nothing is gathered or copied.
    """
    if rows is not None:
        B, _, H, D = q.shape
        T_q, T_kv = problem.T_q, problem.T_kv
    else:
        B, H, T_q, D = q.shape
        T_kv = k.shape[2]
    dev = q.device
    BH = B * H
    Tq_pad = pad128(T_q)
    O = as_operand(outputs.O, dev)
    d_out = as_operand(d_out, dev)
    if boundary is None:
        if tuple(d_out.shape) != tuple(q.shape):
            raise ShapeError(f"dO shape {tuple(d_out.shape)} != {tuple(q.shape)}")
        dq = torch.empty((B, H, T_q, D), dtype=torch.float32, device=dev)
        dk = torch.empty((B, H, T_kv, D), dtype=torch.float32, device=dev)
        dv = torch.empty((B, H, T_kv, D), dtype=torch.float32, device=dev)
        Tq_out, Tkv_out, out_b = T_q, T_kv, 0
        d_sorted = d_out
    else:
        Tq_out, Tkv_out, zero = boundary
        dq = _zeros_or_empty((B, Tq_out, H, D), torch.float32, dev, zero)
        dk = _zeros_or_empty((B, Tkv_out, H, D), torch.float32, dev, zero)
        dv = _zeros_or_empty((B, Tkv_out, H, D), torch.float32, dev, zero)
        out_b = 1
        d_sorted = d_out if rows is not None else torch.empty((B, H, T_q, D), dtype=torch.bfloat16, device=dev)
    if BH == 0:
        return dq, dk, dv
    delta = torch.empty((BH, Tq_pad), dtype=torch.float32, device=dev)
    lse_in = getattr(outputs, "_lse2", None)
    rargs = rows.args() if rows is not None else _NO_ROWS
    if lse_in is not None and (rows is not None or boundary is None):
        lse2 = lse_in  # from our forward; delta is fused into the dQ kernel
        fuse = True
    elif lse_in is not None and q_rank is not None and T_q == Tq_out:
        # shared hash ids (every position has a slot): the delta pass reads O / dO in
        # memory order and writes dO / delta at each position's slot
        lse2, fuse = lse_in, False
        _lib.call("scfa_bwd_prep_rank", _lib.ptr(O), _lib.ptr(d_out), B, T_q, H, D, Tq_pad, _lib.ptr(q_rank),
                  _lib.ptr(d_sorted), _lib.ptr(delta), _lib.stream_ptr())
    else:
        fuse = False
        lse2 = torch.empty((BH, Tq_pad), dtype=torch.float32, device=dev)
        M = outputs.M if lse_in is None else None
        Lv = outputs.L if lse_in is None else None
        if M is not None:
            M = torch.as_tensor(M, device=dev).to(torch.float32).contiguous()
            Lv = torch.as_tensor(Lv, device=dev).to(torch.float32).contiguous()
        if rows is not None:
            raise ShapeError("row-table backward needs the forward's saved log-sum-exp")
        _lib.call("scfa_bwd_prep", _lib.ptr(O), _lib.ptr(d_out), _lib.ptr(lse_in), _lib.ptr(M), _lib.ptr(Lv),
                  BH, T_q, D, Tq_pad, _lib.ptr(problem.q_idx) if out_b else None, H, Tq_out,
                  _lib.ptr(d_sorted) if out_b else None, _lib.ptr(delta), _lib.ptr(lse2), _lib.stream_ptr())
    sched = problem.schedule("dq", "dkdv")
    if T_q > 0:
        lst, cnt, stride = sched["dq"]
        _lib.call(
            "scfa_attn_bwd_dq",
            _lib.ptr(q), _lib.ptr(k), _lib.ptr(v), _lib.ptr(d_sorted), BH, T_q, T_kv, D,
            _lib.ptr(problem.q_idx), _lib.ptr(sched["q_runs"]), problem.Tq_pad, problem.Tkv_pad,
            _lib.ptr(lse2), _lib.ptr(delta), _lib.ptr(lst), _lib.ptr(cnt), stride,
            _scale(scale, D), H, Tq_out, out_b, _lib.ptr(dq), *rargs,
            _lib.ptr(O) if fuse else None, _lib.ptr(delta) if fuse else None, None, None, _lib.stream_ptr(),
        )
    if T_kv > 0:
        lst, cnt, stride = sched["dkdv"]
        _lib.call(
            "scfa_attn_bwd_dkdv",
            _lib.ptr(q), _lib.ptr(k), _lib.ptr(v), _lib.ptr(d_sorted), BH, T_q, T_kv, D,
            _lib.ptr(problem.k_idx), _lib.ptr(sched["k_runs"]), problem.Tq_pad, problem.Tkv_pad,
            _lib.ptr(lse2), _lib.ptr(delta), _lib.ptr(lst), _lib.ptr(cnt), stride,
            _scale(scale, D), H, Tkv_out, out_b, _lib.ptr(dk), _lib.ptr(dv), *rargs, None, _lib.stream_ptr(),
        )
    return dq, dk, dv


def dq_backward_gathered(problem, q, k_sorted, v_sorted, outputs, d_out, rows, scale, T_out, do_out,
                         q_sorted=None):
    """dQ with the stationary Q / dO read through rows.q_rows from the caller's (B, T, H, D)
    tensors (gather4, once per item) and streamed K / V from bucket-order copies; delta =
    rowsum(dO * O) fused in (O read where the forward wrote it) and the gathered dO written
    back in kernel order to do_out (B, H, T_q, D) for the dK/dV pass.
    Returns (dQ (B, T_out, H, D) fp32, delta (BH, Tq_pad))."""
    B, H, D = problem.B, problem.H, problem.D
    T_q, T_kv = problem.T_q, problem.T_kv
    dev = q.device
    BH = B * H
    dq = torch.empty((B, T_out, H, D), dtype=torch.float32, device=dev)
    delta = torch.empty((BH, pad128(T_q)), dtype=torch.float32, device=dev)
    if BH == 0 or T_q == 0:
        return dq, delta
    sched = problem.schedule("dq")
    lst, cnt, stride = sched["dq"]
    _lib.call(
        "scfa_attn_bwd_dq",
        _lib.ptr(q), _lib.ptr(k_sorted), _lib.ptr(v_sorted), _lib.ptr(d_out), BH, T_q, T_kv, D,
        _lib.ptr(problem.q_idx), _lib.ptr(sched["q_runs"]), problem.Tq_pad, problem.Tkv_pad,
        _lib.ptr(outputs._lse2), _lib.ptr(delta), _lib.ptr(lst), _lib.ptr(cnt), stride,
        _scale(scale, D), H, T_out, 1, _lib.ptr(dq), *rows.args(),
        _lib.ptr(as_operand(outputs.O, dev)), _lib.ptr(delta), _lib.ptr(do_out), _lib.ptr(q_sorted),
        _lib.stream_ptr(),
    )
    return dq, delta


def dkdv_backward_sorted(problem, q_sorted, k_sorted, v_sorted, do_sorted, lse2, delta, scale, T_out, out_rows=None):
    """dK / dV from bucket-order (B, H, T, D) copies, written to their original positions of
    (B, T_out, H, D) fp32 tensors.  out_rows (BH, Tkv_pad) int32: route every key slot, pads
    included, through this row table (each row of dK / dV is then written)."""
    B, H, D = problem.B, problem.H, problem.D
    T_q, T_kv = problem.T_q, problem.T_kv
    dev = k_sorted.device
    BH = B * H
    dk = torch.empty((B, T_out, H, D), dtype=torch.float32, device=dev)
    dv = torch.empty((B, T_out, H, D), dtype=torch.float32, device=dev)
    if BH == 0 or T_kv == 0:
        return dk, dv
    sched = problem.schedule("dkdv")
    lst, cnt, stride = sched["dkdv"]
    _lib.call(
        "scfa_attn_bwd_dkdv",
        _lib.ptr(q_sorted), _lib.ptr(k_sorted), _lib.ptr(v_sorted), _lib.ptr(do_sorted), BH, T_q, T_kv, D,
        _lib.ptr(problem.k_idx), _lib.ptr(sched["k_runs"]), problem.Tq_pad, problem.Tkv_pad,
        _lib.ptr(lse2), _lib.ptr(delta), _lib.ptr(lst), _lib.ptr(cnt), stride,
        _scale(scale, D), H, T_out, 1, _lib.ptr(dk), _lib.ptr(dv), *_NO_ROWS, _lib.ptr(out_rows), _lib.stream_ptr(),
    )
    return dk, dv


def backward_single_pass(problem, q_sorted, k_sorted, v_sorted, do_sorted, lse2, delta, scale, Tq_out, Tkv_out,
                         boundary=True):
    """dQ, dK, dV in one key-stationary sweep (scfa_attn_bwd, D = 64): kernel-order operands,
    the dK/dV schedule; dQ is reduced per tile pair into a zero-filled fp32 tensor.

    boundary=True: gradients at their original positions of (B, T_*_out, H, D) fp32 tensors
    (the inverse scatter fused); else engine layout (B, H, T, D) in kernel order.
    Not bitwise reproducible in dQ (fp32 reduction order); attention_backward is."""
    B, H, D = problem.B, problem.H, problem.D
    T_q, T_kv = problem.T_q, problem.T_kv
    dev = k_sorted.device
    BH = B * H
    if boundary:
        dq = torch.zeros((B, Tq_out, H, D), dtype=torch.float32, device=dev)
        dk = torch.empty((B, Tkv_out, H, D), dtype=torch.float32, device=dev)
        dv = torch.empty((B, Tkv_out, H, D), dtype=torch.float32, device=dev)
    else:
        dq = torch.zeros((B, H, T_q, D), dtype=torch.float32, device=dev)
        dk = torch.empty((B, H, T_kv, D), dtype=torch.float32, device=dev)
        dv = torch.empty((B, H, T_kv, D), dtype=torch.float32, device=dev)
    if BH == 0 or T_kv == 0 or T_q == 0:
        if T_kv and BH:
            dk.zero_()
            dv.zero_()
        return dq, dk, dv
    sched = problem.schedule("dkdv")
    lst, cnt, stride = sched["dkdv"]
    _lib.call(
        "scfa_attn_bwd",
        _lib.ptr(q_sorted), _lib.ptr(k_sorted), _lib.ptr(v_sorted), _lib.ptr(do_sorted), BH, T_q, T_kv, D,
        _lib.ptr(problem.q_idx), _lib.ptr(problem.k_idx), _lib.ptr(sched["k_runs"]), problem.Tq_pad, problem.Tkv_pad,
        _lib.ptr(lse2), _lib.ptr(delta), _lib.ptr(lst), _lib.ptr(cnt), stride, _scale(scale, D), H,
        Tq_out if boundary else T_q, Tkv_out if boundary else T_kv, 1 if boundary else 0,
        _lib.ptr(dq), _lib.ptr(dk), _lib.ptr(dv), _lib.stream_ptr(),
    )
    return dq, dk, dv


def make_row_tables(q_perm, k_perm, B, H, T_q_slots, T_kv_slots, T_Q, T_KV, Tq_pad, Tkv_pad, shared=False):
    """scfa_row_map for both sides (shared=True reuses the query table for keys)."""
    dev = q_perm.device

    def one(perm, n_slots, T_src, T_pad):
        rows = torch.empty((B * H, T_pad), dtype=torch.int32, device=dev)
        if B * H and n_slots:
            _lib.call("scfa_row_map", _lib.ptr(perm), B, H, perm.shape[1], n_slots, T_pad, T_src, _lib.ptr(rows),
                      _lib.stream_ptr())
        return rows

    qr = one(q_perm, T_q_slots, T_Q, Tq_pad)
    kr = qr if shared else one(k_perm, T_kv_slots, T_KV, Tkv_pad)
    return RowTables(qr, kr, B * T_Q * H, B * T_KV * H)


def causal_j_stops(q_idx, k_idx, blocks=BlockSpec()):
    """Reference ``causal_j_stops`` for one head's 1-D index vectors (computed on the GPU)."""
    q = torch.as_tensor(q_idx)
    k = torch.as_tensor(k_idx)
    dev = q.device if q.is_cuda else torch.device("cuda")
    Tq, Tk = int(q.numel()), int(k.numel())
    pq = pack_index(q.reshape(1, 1, Tq), 1, Tq, -1, dev)
    pk = pack_index(k.reshape(1, 1, Tk), 1, Tk, 0x7FFFFFFF, dev)
    prob = Problem(1, 1, Tq, Tk, 64, pq, pk)
    return prob.ref_schedule(blocks)[1][0]


def hash_tile_ranges(q_hash, q_idx, k_hash, k_idx, blocks=BlockSpec()):
    """Reference ``hash_tile_ranges`` (_kernel.py:56-79) for one head, on the GPU."""
    tens = [torch.as_tensor(x) for x in (q_hash, q_idx, k_hash, k_idx)]
    dev = next((t.device for t in tens if t.is_cuda), torch.device("cuda"))
    Tq, Tk = int(tens[1].numel()), int(tens[3].numel())
    qh = pack_index(tens[0].reshape(1, 1, Tq), 1, Tq, -3, dev)
    qi = pack_index(tens[1].reshape(1, 1, Tq), 1, Tq, -1, dev)
    kh = pack_index(tens[2].reshape(1, 1, Tk), 1, Tk, -2, dev)
    ki = pack_index(tens[3].reshape(1, 1, Tk), 1, Tk, 0x7FFFFFFF, dev)
    prob = Problem(1, 1, Tq, Tk, 64, qi, ki, qh, kh, flags=_lib.FLAG_HASH)
    js, je, _ = prob.ref_schedule(blocks)
    return js[0], je[0]
