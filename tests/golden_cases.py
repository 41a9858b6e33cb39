"""Loader for the golden vectors in tests/golden/ (written by tests/golden/make_golden.py
from the reference package) plus the oracle restatement of each case.

Inputs are regenerated here from the seeds with this package's copies of the
reference generators; the stored checksums prove they are the same values the
reference saw.  Only tests import this module.
"""

import json
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def case_names(kind=None):
    with open(os.path.join(GOLDEN, "cases.json")) as f:
        meta = json.load(f)
    return [n for n, m in sorted(meta.items()) if kind is None or m["kind"] == kind]


def load(name):
    with open(os.path.join(GOLDEN, "cases.json")) as f:
        meta = json.load(f)[name]
    with np.load(os.path.join(GOLDEN, f"{name}.npz")) as z:
        arrays = {k: z[k] for k in z.files}
    return meta, arrays


def bf16(x):
    import torch

    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).to(torch.bfloat16).to(torch.float64).numpy()


def checksum(x):
    """Same reduction as make_golden.checksum."""
    x = np.asarray(x, dtype=np.float64)
    return np.array([x.sum(), np.abs(x).sum(), (x * np.arange(x.size).reshape(x.shape) % 7).sum()])


def _drop_head(q_keep, k_keep):
    q_keep[0, :, 1] = 0.0
    k_keep[0, :, 1] = 0.0
    k_keep[0, 5, 1] = 1.0


def _late_keys(q_keep, k_keep):
    k_keep[:, :100, :] = 0.0


OVERRIDES = {"_drop_head": _drop_head, "_late_keys": _late_keys}


def inputs(meta):
    """Boundary-layout (B, T, H, D) float64 bf16-representable q, k, v, dO."""
    from paper_2306_01160_b200.tensors import random_tensor_np

    B, H, D, s = meta["B"], meta["H"], meta["D"], meta["seed"]
    TQ, TK = meta["T_Q"], meta["T_KV"]
    if meta["kind"] == "dense":  # engine layout in the reference case
        return tuple(bf16(random_tensor_np((B, H, TQ, D), s + i)) for i in range(4))
    shapes = [(B, H, TQ, D), (B, H, TK, D), (B, H, TK, D), (B, H, TQ, D)]
    return tuple(bf16(np.swapaxes(random_tensor_np(sh, s + i), 1, 2)) for i, sh in enumerate(shapes))


def sparsity(meta):
    """QK: (q_keep, k_keep) float64 (B, T, H).  Hash: (q_hash, k_hash) int64 (B, T, H)."""
    from paper_2306_01160_b200.hash_sparse import random_buckets
    from paper_2306_01160_b200.qk_sparse import random_keep

    B, H, s = meta["B"], meta["H"], meta["seed"]
    TQ, TK = meta["T_Q"], meta["T_KV"]
    if meta["kind"] == "qk":
        qk = random_keep(B, TQ, H, meta["drop"], s + 6)
        kk = random_keep(B, TK, H, meta["drop"], s + 7)
        if meta.get("overrides"):
            OVERRIDES[meta["overrides"]](qk, kk)
        return qk, kk
    if meta["kind"] == "hash":
        qh = random_buckets(B, TQ, H, meta["nb"], s + 5)
        kh = qh if meta["shared"] else random_buckets(B, TK, H, meta["nb"], s + 4)
        return qh, kh
    return None, None


def visibility(meta, a=None, b=None):
    """(B, H, T_Q, T_KV) visible pairs on original positions (oracle.build_mask semantics)."""
    from oracle import scfa_oracle as orc

    TQ, TK = meta["T_Q"], meta["T_KV"]
    pq, pk = np.arange(TQ), np.arange(TK)
    if meta["kind"] == "dense":
        return orc.visibility(pq, pk)[None, None]
    if meta["kind"] == "qk":
        vis = orc.visibility(pq, pk)[None, None]
        qk = np.swapaxes(a, 1, 2) > 0
        kk = np.swapaxes(b, 1, 2) > 0
        return vis & qk[..., :, None] & kk[..., None, :]
    qh, kh = np.swapaxes(a, 1, 2), np.swapaxes(b, 1, 2)
    return orc.visibility(pq, pk, qh, kh, exclude_self=meta["exclude_self"])


def oracle_outputs(meta):
    """O, dQ, dK, dV in the golden layout (boundary for qk/hash, engine for dense)."""
    from oracle import scfa_oracle as orc

    q, k, v, dO = inputs(meta)
    a, b = sparsity(meta)
    vis = visibility(meta, a, b)
    eng = (lambda x: x) if meta["kind"] == "dense" else (lambda x: np.swapaxes(x, 1, 2))
    O, M, L = orc.attention(eng(q), eng(k), eng(v), vis)
    dq, dk, dv = orc.attention_grads(eng(q), eng(k), eng(v), vis, eng(dO))
    if meta["kind"] == "qk":  # dropped rows carry zeros (qk_postprocess scatters into zeros)
        qm = (np.swapaxes(a, 1, 2) > 0)[..., None]
        km = (np.swapaxes(b, 1, 2) > 0)[..., None]
        O, dq, dk, dv = O * qm, dq * qm, dk * km, dv * km
    return tuple(eng(x) for x in (O, dq, dk, dv)), (M, L)
