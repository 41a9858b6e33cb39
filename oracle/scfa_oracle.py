"""NumPy restatement of the reference attention path (TEST INFRASTRUCTURE ONLY).

Each function names the reference lines it restates (paths under
/root/reference/pkg/src/scfa/).  Written for clarity at test sizes, in
float64 by default; never imported by the product package.
"""

import numpy as np

KEY_PAD = 10**9  # tensors.py:22-24
QUERY_PAD = -1


# ---------------------------------------------------------------- visibility / attention

def visibility(q_idx, k_idx, q_hash=None, k_hash=None, exclude_self=False):
    """(..., T_Q, T_KV) bool: causal on original positions, AND same bucket (oracle.py:14-40)."""
    qi = np.asarray(q_idx)[..., :, None]
    ki = np.asarray(k_idx)[..., None, :]
    vis = (qi > ki) if exclude_self else (qi >= ki)
    if q_hash is not None:
        vis = vis & (np.asarray(q_hash)[..., :, None] == np.asarray(k_hash)[..., None, :])
    return vis


def _probs(q, k, vis, scale):
    s = scale * np.einsum("...td,...sd->...ts", q, k)
    s = np.where(vis, s, -np.inf)
    m = s.max(axis=-1, keepdims=True)
    m_hat = np.where(np.isneginf(m), 0.0, m)
    e = np.exp(s - m_hat)
    den = e.sum(axis=-1, keepdims=True)
    p = e / np.where(den == 0.0, 1.0, den)
    return p, m[..., 0], den[..., 0]


def attention(q, k, v, vis, scale=None):
    """softmax(scale QK^T | vis) V with stranded rows 0 (oracle.py:49-68).

    Returns (O, M, L): M = row max of visible scaled logits (-inf if none),
    L = sum exp(s - M) (0 if none) — FlashOutputs.M/L semantics (_kernel.py:18-30).
    """
    q, k, v = (np.asarray(x, dtype=np.float64) for x in (q, k, v))
    if scale is None:
        scale = 1.0 / np.sqrt(q.shape[-1])
    p, m, den = _probs(q, k, vis, scale)
    return p @ v, m, den


def attention_grads(q, k, v, vis, d_out, scale=None):
    """Closed-form gradients of <attention(Q,K,V), dO> (what backward_head computes,
    _kernel.py:139-193): dS = P (dP - rowsum(dO*O)), dQ = s dS K, dK = s dS^T Q, dV = P^T dO."""
    q, k, v, d_out = (np.asarray(x, dtype=np.float64) for x in (q, k, v, d_out))
    if scale is None:
        scale = 1.0 / np.sqrt(q.shape[-1])
    p, _, _ = _probs(q, k, vis, scale)
    o = p @ v
    dp = d_out @ np.swapaxes(v, -1, -2)
    delta = (d_out * o).sum(axis=-1, keepdims=True)
    ds = p * (dp - delta)
    dq = scale * ds @ k
    dk = scale * np.swapaxes(ds, -1, -2) @ q
    dv = np.swapaxes(p, -1, -2) @ d_out
    return dq, dk, dv


# ---------------------------------------------------------------- index preparation

def compact_order(keep):
    """Per (b, h): kept positions ascending, then dropped ascending == stable
    argsort(~kept) along T (qk_sparse.py:57-60).  keep (B, T, H) -> order (B, T, H), counts (B, H)."""
    kept = np.asarray(keep).astype(bool)
    B, T, H = kept.shape
    order = np.empty((B, T, H), dtype=np.int64)
    counts = kept.sum(axis=1)
    for b in range(B):
        for h in range(H):
            col = kept[b, :, h]
            order[b, :, h] = np.concatenate([np.flatnonzero(col), np.flatnonzero(~col)])
    return order, counts


def padded(index, counts, pad):
    """Slots >= count -> pad (qk_sparse.py:74-83)."""
    out = np.array(index, dtype=np.int64, copy=True)
    slot = np.arange(out.shape[1])[None, :, None]
    out[slot >= np.asarray(counts)[:, None, :]] = pad
    return out


def bucket_order(hashes, idx=None):
    """Stable order by (bucket, position) along the last axis (hash_sparse.py:89-94)."""
    hashes = np.asarray(hashes, dtype=np.int64)
    if idx is None:
        idx = np.broadcast_to(np.arange(hashes.shape[-1]), hashes.shape)
    return np.lexsort((np.asarray(idx), hashes), axis=-1)


# ---------------------------------------------------------------- reference schedules

def _blk(x, size, fn):
    x = np.asarray(x)
    return np.array([fn(x[i:i + size]) for i in range(0, x.size, size)], dtype=np.int64)


def causal_j_stops(q_idx, k_idx, B_m=64, B_n=64):
    """j_stop[i] = #{j : min k_idx of key block j <= max q_idx of query block i} (_kernel.py:45-53)."""
    max_q = _blk(q_idx, B_m, np.max)
    min_k = _blk(k_idx, B_n, np.min)
    return np.array([int(np.sum(min_k <= mq)) for mq in max_q], dtype=np.int64)


def hash_tile_ranges(q_hash, q_idx, k_hash, k_idx, B_m=64, B_n=64):
    """Banded [j_start, j_stop) per query block for sorted inputs (_kernel.py:56-79)."""
    mnqh, mxqh = _blk(q_hash, B_m, np.min), _blk(q_hash, B_m, np.max)
    mnkh, mxkh = _blk(k_hash, B_n, np.min), _blk(k_hash, B_n, np.max)
    mnki, mxqi = _blk(k_idx, B_n, np.min), _blk(q_idx, B_m, np.max)
    starts, stops = [], []
    for i in range(mnqh.size):
        a = int(np.sum(mxkh < mnqh[i]))
        b = int(np.sum(mnkh <= mxqh[i]))
        stop = a
        for j in range(b - 1, a - 1, -1):
            if mnki[j] <= mxqi[i]:
                stop = j + 1
                break
        starts.append(a)
        stops.append(stop)
    return np.array(starts, dtype=np.int64), np.array(stops, dtype=np.int64)


def live_pairs_qk(q_keep, k_keep):
    """P_live for QK: sum over heads of #{(q kept, k kept) : k <= q}."""
    qk = np.asarray(q_keep).astype(bool)
    kk = np.asarray(k_keep).astype(bool)
    ck = np.cumsum(kk, axis=1)  # kept keys at positions <= t
    return int(np.sum(np.where(qk, ck, 0)))


def live_pairs_hash(q_hash, k_hash, exclude_self=True):
    """P_live for hash with shared ids: sum_g c_g(c_g - 1)/2 (+ c_g if self allowed), per head."""
    q_hash = np.asarray(q_hash)
    total = 0
    B, T, H = q_hash.shape
    for b in range(B):
        for h in range(H):
            c = np.bincount(q_hash[b, :, h])
            total += int(np.sum(c * (c - 1) // 2 + (0 if exclude_self else c)))
    return total


# ---------------------------------------------------------------- bucket producer

def philox_stream(seed, domain, index=0):
    """numpy Generator for one (seed, domain, index) Philox key (tensors.py:86-93)."""
    key = ((seed & ((1 << 64) - 1)) << 64) | ((domain & 0xFF) << 56) | (index & ((1 << 56) - 1))
    return np.random.Generator(np.random.Philox(key=key))


def lsh_buckets(x, nb, seed, domain_projections=1):
    """Angular LSH ids (hash_sparse.py:34-52): per (b, h) R = D x nb/2 normal from the
    (seed, DOMAIN_PROJECTIONS=1, b*H + h) stream, id = argmax([xR, -xR]) (first max)."""
    x = np.asarray(x)
    B, T, H, D = x.shape
    out = np.empty((B, T, H), dtype=np.int64)
    for b in range(B):
        for h in range(H):
            r = philox_stream(seed, domain_projections, b * H + h).standard_normal((D, nb // 2))
            rot = x[b, :, h, :] @ r
            out[b, :, h] = np.argmax(np.concatenate([rot, -rot], axis=1), axis=1)
    return out

