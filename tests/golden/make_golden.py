"""Generate the golden vectors under tests/golden/ by running the REFERENCE package.

Run in the build container (where /root/reference exists), from the repo root:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Every case draws its inputs from the reference's own seeded generators
(random_tensor tensors.py:96-107, random_keep qk_sparse.py:242-247,
random_buckets hash_sparse.py:55-60), rounds Q/K/V/dO to bf16 (so the GPU
engine and the reference see identical values) and runs the
reference's public functions in float64:

  qk:    qk_preprocess (qk_sparse.py:196-211) -> qk_forward_kernel (:120-148)
         -> qk_postprocess (:214-225); backward composed as SURVEY.md §8c:
         qk_backward_kernel (:151-183) on dO gathered by scatter_index, grads
         scattered back with the q / k compaction indices (dropped rows 0).
  hash:  sort_by_bucket (hash_sparse.py:97-133) -> hash_forward_kernel
         (:145-179) -> hash_scatter (:216-220); backward via
         hash_backward_kernel (:182-213) on dO sorted by q_idx.
  dense: flash_forward / flash_backward (dense.py:33-93).
  lsh:   lsh_buckets (hash_sparse.py:34-52) at several bucket counts (lsh_small.npz;
         `--lsh-only` regenerates just that file).
  files: tensor_f32.scfa / tensor_f64.scfa written by the reference's save_tensor
         (tensors.py:110-125) with their arrays in tensor_files.npz.

Stored per case (one .npz): the integer provenance (compaction indices,
counts, sorted positions / buckets, reference schedules at BlockSpec(64,64)),
tiles_computed, O (boundary layout), M/L (kernel order), dQ/dK/dV (boundary
layout), and input checksums so the tests can confirm they regenerate the
same inputs.  Nothing on the GPU box reads /root/reference: the tests only
read these files.
"""

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))


def _bf16(x):
    import torch

    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).to(torch.bfloat16).to(torch.float64).numpy()


def _boundary(shape_bhtd, seed):
    import scfa

    return _bf16(scfa.from_heads(scfa.random_tensor(shape_bhtd, seed)))


def checksum(x):
    x = np.asarray(x, dtype=np.float64)
    return np.array([x.sum(), np.abs(x).sum(), (x * np.arange(x.size).reshape(x.shape) % 7).sum()])


def qk_case(name, B, H, T_Q, T_KV, D, drop, seed=0, keep_overrides=None):
    import scfa
    from scfa import qk_sparse as qs

    q = _boundary((B, H, T_Q, D), seed)
    k = _boundary((B, H, T_KV, D), seed + 1)
    v = _boundary((B, H, T_KV, D), seed + 2)
    dO = _boundary((B, H, T_Q, D), seed + 3)
    q_keep = scfa.random_keep(B, T_Q, H, drop, seed + 6)
    k_keep = scfa.random_keep(B, T_KV, H, drop, seed + 7)
    if keep_overrides:
        keep_overrides(q_keep, k_keep)
    prep = scfa.qk_preprocess(q, k, v, q_keep, k_keep)
    out = scfa.qk_forward_kernel(prep.q_c, prep.k_c, prep.v_c, prep.q_idx, prep.k_idx)
    O = scfa.qk_postprocess(out.O, prep.scatter_index, T_Q)
    # backward composition (the reference has no autograd)
    dO_c = scfa.to_heads(qs.compact(None, dO, index=prep.scatter_index).compact)
    dq_c, dk_c, dv_c = scfa.qk_backward_kernel(prep.q_c, prep.k_c, prep.v_c, out, dO_c, prep.q_idx, prep.k_idx)
    _, k_index, k_counts = qs.compact(k_keep, k)
    _, q_index, q_counts = qs.compact(q_keep, q)
    dq = scfa.qk_postprocess(dq_c, prep.scatter_index, T_Q)
    dk = scfa.qk_postprocess(dk_c, k_index, T_KV)
    dv = scfa.qk_postprocess(dv_c, k_index, T_KV)
    nq = prep.q_idx.shape[2]
    j_stop = np.stack([np.stack([scfa.qk_tile_schedule(prep.q_idx[b, h], prep.k_idx[b, h], scfa.BlockSpec())
                                 for h in range(H)]) for b in range(B)]) if nq else np.zeros((B, H, 0), np.int64)
    tiles_128 = scfa.qk_forward_kernel(prep.q_c, prep.k_c, prep.v_c, prep.q_idx, prep.k_idx,
                                       blocks=scfa.BlockSpec(128, 128)).tiles_computed
    arrays = dict(
        q_keep=q_keep.astype(np.uint8), k_keep=k_keep.astype(np.uint8),
        q_index=q_index.astype(np.int32), q_counts=q_counts.astype(np.int32),
        k_index=k_index.astype(np.int32), k_counts=k_counts.astype(np.int32),
        q_idx=prep.q_idx.astype(np.int32), k_idx=prep.k_idx.astype(np.int32),
        scatter_index=prep.scatter_index.astype(np.int32), j_stop=j_stop.astype(np.int32),
        O=O, M=out.M, L=out.L, dq=dq, dk=dk, dv=dv,
        checksum_q=checksum(q), checksum_k=checksum(k), checksum_v=checksum(v), checksum_dO=checksum(dO),
    )
    meta = dict(kind="qk", B=B, H=H, T_Q=T_Q, T_KV=T_KV, D=D, drop=drop, seed=seed,
                tiles_computed=int(out.tiles_computed), tiles_computed_128=int(tiles_128),
                overrides=keep_overrides.__name__ if keep_overrides else None)
    return arrays, meta


def hash_case(name, B, H, T_Q, T_KV, D, nb, seed=0, shared=True, exclude_self=True):
    import scfa

    q = _boundary((B, H, T_Q, D), seed)
    k = _boundary((B, H, T_KV, D), seed + 1)
    v = _boundary((B, H, T_KV, D), seed + 2)
    dO = _boundary((B, H, T_Q, D), seed + 3)
    q_hash = scfa.random_buckets(B, T_Q, H, nb, seed + 5)
    k_hash = q_hash if shared else scfa.random_buckets(B, T_KV, H, nb, seed + 4)
    sb = scfa.sort_by_bucket(scfa.to_heads(q), scfa.to_heads(k), scfa.to_heads(v), scfa.to_heads(q_hash),
                             scfa.to_heads(k_hash))
    out = scfa.hash_forward_kernel(sb, exclude_self=exclude_self)
    O = scfa.from_heads(scfa.hash_scatter(out.O, sb.q_idx))
    O_api = scfa.hash_sparse_attention(q, k, v, q_hash, k_hash, exclude_self=exclude_self)
    assert np.array_equal(O, O_api)
    dO_s = np.take_along_axis(scfa.to_heads(dO), sb.q_idx[..., None], axis=2)
    dq_s, dk_s, dv_s = scfa.hash_backward_kernel(sb, out, dO_s, exclude_self=exclude_self)
    dq = scfa.from_heads(scfa.hash_scatter(dq_s, sb.q_idx))
    dk = scfa.from_heads(scfa.hash_scatter(dk_s, sb.k_idx))
    dv = scfa.from_heads(scfa.hash_scatter(dv_s, sb.k_idx))
    js, je = [], []
    for b in range(B):
        for h in range(H):
            a, e = scfa.hash_tile_ranges(sb.q_hash[b, h], sb.q_idx[b, h], sb.k_hash[b, h], sb.k_idx[b, h],
                                         scfa.BlockSpec())
            js.append(a)
            je.append(e)
    nqb = len(js[0])
    tiles_128 = scfa.hash_forward_kernel(sb, blocks=scfa.BlockSpec(128, 128), exclude_self=exclude_self)
    arrays = dict(
        q_hash=q_hash.astype(np.int32), k_hash=k_hash.astype(np.int32),
        q_idx=sb.q_idx.astype(np.int32), k_idx=sb.k_idx.astype(np.int32),
        q_hash_sorted=sb.q_hash.astype(np.int32), k_hash_sorted=sb.k_hash.astype(np.int32),
        j_start=np.array(js, np.int32).reshape(B, H, nqb), j_stop=np.array(je, np.int32).reshape(B, H, nqb),
        O=O, M=out.M, L=out.L, dq=dq, dk=dk, dv=dv,
        checksum_q=checksum(q), checksum_k=checksum(k), checksum_v=checksum(v), checksum_dO=checksum(dO),
    )
    meta = dict(kind="hash", B=B, H=H, T_Q=T_Q, T_KV=T_KV, D=D, nb=nb, seed=seed, shared=shared,
                exclude_self=exclude_self, tiles_computed=int(out.tiles_computed),
                tiles_computed_128=int(tiles_128.tiles_computed))
    return arrays, meta


def dense_case(name, B, H, T, D, seed=0):
    import scfa

    q, k, v, dO = (_bf16(scfa.random_tensor((B, H, T, D), seed + i)) for i in range(4))
    out = scfa.flash_forward(q, k, v)
    dq, dk, dv = scfa.flash_backward(q, k, v, out, dO)
    arrays = dict(O=out.O, M=out.M, L=out.L, dq=dq, dk=dk, dv=dv,
                  checksum_q=checksum(q), checksum_k=checksum(k), checksum_v=checksum(v), checksum_dO=checksum(dO))
    meta = dict(kind="dense", B=B, H=H, T_Q=T, T_KV=T, D=D, seed=seed, tiles_computed=int(out.tiles_computed),
                tiles_computed_128=int(scfa.flash_forward(q, k, v, blocks=scfa.BlockSpec(128, 128)).tiles_computed))
    return arrays, meta


def _drop_head(q_keep, k_keep):
    """Head (0, 1) keeps nothing on the query side and a single key (stranded rows, empty heads)."""
    q_keep[0, :, 1] = 0.0
    k_keep[0, :, 1] = 0.0
    k_keep[0, 5, 1] = 1.0


def _late_keys(q_keep, k_keep):
    """All keys before position 100 dropped: early queries are stranded (rows exactly zero)."""
    k_keep[:, :100, :] = 0.0


CASES = [
    # name, builder, kwargs, float storage dtype
    ("qk_cfg1", qk_case, dict(B=2, H=4, T_Q=1024, T_KV=1024, D=64, drop=0.5), np.float32),
    ("qk_small", qk_case, dict(B=1, H=2, T_Q=200, T_KV=200, D=64, drop=0.3, seed=10), np.float32),
    ("qk_rect", qk_case, dict(B=1, H=2, T_Q=160, T_KV=300, D=64, drop=0.5, seed=20), np.float32),
    ("qk_nodrop", qk_case, dict(B=1, H=1, T_Q=256, T_KV=256, D=64, drop=0.0, seed=30), np.float32),
    ("qk_heavy", qk_case, dict(B=1, H=2, T_Q=384, T_KV=384, D=64, drop=0.9, seed=40), np.float32),
    ("qk_empty_head", qk_case, dict(B=1, H=2, T_Q=256, T_KV=256, D=64, drop=0.5, seed=50,
                                    keep_overrides=_drop_head), np.float32),
    ("qk_stranded", qk_case, dict(B=1, H=2, T_Q=256, T_KV=256, D=64, drop=0.3, seed=60,
                                  keep_overrides=_late_keys), np.float32),
    ("qk_d128", qk_case, dict(B=1, H=2, T_Q=256, T_KV=256, D=128, drop=0.5, seed=70), np.float32),
    ("hash_small", hash_case, dict(B=1, H=2, T_Q=256, T_KV=256, D=64, nb=4, seed=100), np.float32),
    ("hash_rect", hash_case, dict(B=1, H=2, T_Q=192, T_KV=320, D=64, nb=8, seed=110, shared=False), np.float32),
    ("hash_single", hash_case, dict(B=1, H=1, T_Q=256, T_KV=256, D=64, nb=1, seed=120), np.float32),
    ("hash_self", hash_case, dict(B=1, H=2, T_Q=256, T_KV=256, D=64, nb=4, seed=130, exclude_self=False),
     np.float32),
    ("hash_t2048", hash_case, dict(B=1, H=1, T_Q=2048, T_KV=2048, D=64, nb=16, seed=140), np.float32),
    ("hash_d128", hash_case, dict(B=1, H=1, T_Q=320, T_KV=320, D=128, nb=4, seed=150), np.float32),
    ("dense_small", dense_case, dict(B=1, H=2, T=192, D=64, seed=200), np.float32),
    ("dense_d128", dense_case, dict(B=1, H=1, T=256, D=128, seed=210), np.float32),
]


def lsh_case():
    """lsh_buckets (hash_sparse.py:34-52) of the reference on float32 boundary-layout
    vectors, several bucket counts (incl. nb/2 not a power of two)."""
    from scfa.hash_sparse import lsh_buckets

    rng = np.random.default_rng(300)
    x = rng.standard_normal((2, 200, 3, 32)).astype(np.float32)
    x[0, :4] = 0.0  # zero vectors: every projection ties at 0 -> id 0
    arrays = {"x": x}
    for nb in (2, 6, 16, 64):
        arrays[f"ids_nb{nb}"] = lsh_buckets(x, nb, 31)
    return arrays, {"seed": 31, "nbs": [2, 6, 16, 64]}


def tensor_files():
    """Two files written by the reference's save_tensor (tensors.py:110-125), and the arrays."""
    from scfa import save_tensor

    x = np.random.default_rng(7).standard_normal((2, 3, 5, 4)).astype(np.float32)
    y = np.random.default_rng(8).standard_normal((1, 2, 3, 8))
    save_tensor(os.path.join(HERE, "tensor_f32.scfa"), x)
    save_tensor(os.path.join(HERE, "tensor_f64.scfa"), y)
    np.savez_compressed(os.path.join(HERE, "tensor_files.npz"), f32=x, f64=y)


def main():
    try:
        import scfa  # noqa: F401
    except ImportError:
        sys.exit("run with PYTHONPATH=/root/reference/pkg/src (the reference package)")
    if "--tensor-files-only" in sys.argv:
        tensor_files()
        return
    if "--lsh-only" in sys.argv:
        arrays, meta = lsh_case()
        np.savez_compressed(os.path.join(HERE, "lsh_small.npz"), **arrays)
        print("lsh_small", meta)
        return
    index = {}
    for name, fn, kw, fdt in CASES:
        arrays, meta = fn(name, **kw)
        arrays = {k: (a.astype(fdt) if np.asarray(a).dtype.kind == "f" and not k.startswith("checksum") else a)
                  for k, a in arrays.items()}
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **arrays)
        meta["float_storage"] = np.dtype(fdt).name
        index[name] = meta
        print(name, meta)
    with open(os.path.join(HERE, "cases.json"), "w") as f:
        json.dump(index, f, indent=1, sort_keys=True)
    arrays, meta = lsh_case()
    np.savez_compressed(os.path.join(HERE, "lsh_small.npz"), **arrays)
    print("lsh_small", meta)
    tensor_files()


if __name__ == "__main__":
    main()
