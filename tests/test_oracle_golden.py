"""Pin the oracle (CPU, no GPU): the NumPy and C restatements under oracle/ must reproduce
the golden vectors the REFERENCE package produced (tests/golden/make_golden.py), and
the reference's own known-answer tests (pkg/tests/test_qk.py, test_hash.py).

Tolerances: integer provenance (indices, counts, schedules, tile counts) bit-exact;
floats against the float64 reference stored as float32: 2e-6 relative to max|ref|
for the float64 NumPy oracle, 2e-4 for the float32 C tile loop.
"""

import numpy as np
import pytest

import golden_cases as gc
from oracle import scfa_oracle as orc

ALL = gc.case_names()


def _rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    den = max(float(np.max(np.abs(b))), 1e-30) if b.size else 1.0
    return float(np.max(np.abs(a - b))) / den if b.size else 0.0


# ---------------------------------------------------------------- inputs regenerate exactly

@pytest.mark.parametrize("name", ALL)
def test_generators_reproduce_reference_inputs(name):
    meta, g = gc.load(name)
    for label, x in zip("q k v dO".split(), gc.inputs(meta)):
        np.testing.assert_array_equal(gc.checksum(x), g[f"checksum_{label}"], err_msg=label)
    a, b = gc.sparsity(meta)
    if meta["kind"] == "qk":
        np.testing.assert_array_equal(a.astype(np.uint8), g["q_keep"])
        np.testing.assert_array_equal(b.astype(np.uint8), g["k_keep"])
    elif meta["kind"] == "hash":
        np.testing.assert_array_equal(a, g["q_hash"])
        np.testing.assert_array_equal(b, g["k_hash"])


# ---------------------------------------------------------------- index provenance, bit-exact

@pytest.mark.parametrize("name", gc.case_names("qk"))
def test_compaction_order_matches_reference(name):
    meta, g = gc.load(name)
    qk, kk = gc.sparsity(meta)
    for keep, index, counts, idx, pad in ((qk, g["q_index"], g["q_counts"], g["q_idx"], orc.QUERY_PAD),
                                          (kk, g["k_index"], g["k_counts"], g["k_idx"], orc.KEY_PAD)):
        order, cnt = orc.compact_order(keep)
        buf = index.shape[1]
        np.testing.assert_array_equal(cnt, counts)
        assert buf == (int(cnt.max()) if cnt.size else 0)
        np.testing.assert_array_equal(order[:, :buf], index)
        np.testing.assert_array_equal(np.swapaxes(orc.padded(order[:, :buf], cnt, pad), 1, 2), idx)
    np.testing.assert_array_equal(g["scatter_index"], g["q_index"])


@pytest.mark.parametrize("name", gc.case_names("hash"))
def test_bucket_order_matches_reference(name):
    meta, g = gc.load(name)
    qh, kh = gc.sparsity(meta)
    for h, idx, hs in ((qh, g["q_idx"], g["q_hash_sorted"]), (kh, g["k_idx"], g["k_hash_sorted"])):
        he = np.swapaxes(h, 1, 2)
        order = orc.bucket_order(he)
        np.testing.assert_array_equal(order, idx)
        np.testing.assert_array_equal(np.take_along_axis(he, order, -1), hs)


@pytest.mark.parametrize("name", gc.case_names("qk") + gc.case_names("hash"))
def test_reference_schedule_and_tile_count(name):
    meta, g = gc.load(name)
    B, H = meta["B"], meta["H"]
    total = 0
    for b in range(B):
        for h in range(H):
            if meta["kind"] == "qk":
                stop = orc.causal_j_stops(g["q_idx"][b, h], g["k_idx"][b, h]) if g["q_idx"].shape[2] else []
                np.testing.assert_array_equal(stop, g["j_stop"][b, h])
                total += int(np.sum(stop))
            else:
                a, e = orc.hash_tile_ranges(g["q_hash_sorted"][b, h], g["q_idx"][b, h], g["k_hash_sorted"][b, h],
                                            g["k_idx"][b, h])
                np.testing.assert_array_equal(a, g["j_start"][b, h])
                np.testing.assert_array_equal(e, g["j_stop"][b, h])
                total += int(np.sum(e - a))
    assert total == meta["tiles_computed"]


# ---------------------------------------------------------------- numerics

@pytest.mark.parametrize("name", ALL)
def test_numpy_oracle_matches_reference_outputs(name):
    meta, g = gc.load(name)
    (O, dq, dk, dv), (M, L) = gc.oracle_outputs(meta)
    for label, got in (("O", O), ("dq", dq), ("dk", dk), ("dv", dv)):
        assert _rel(got, g[label]) < 2e-6, f"{label}: rel {_rel(got, g[label]):.2e}"
    # M / L are stored in kernel order: row s of (b, h) is original query position q_idx[b, h, s]
    if meta["kind"] == "dense":
        Mg, Lg = M, L
    else:
        qi = g["q_idx"].astype(np.int64)
        Mg = np.where(qi >= 0, np.take_along_axis(M, np.clip(qi, 0, None), -1), -np.inf)
        Lg = np.where(qi >= 0, np.take_along_axis(L, np.clip(qi, 0, None), -1), 0.0)
    fin = np.isfinite(g["M"])
    np.testing.assert_array_equal(fin, np.isfinite(Mg))
    assert _rel(Mg[fin], g["M"][fin]) < 2e-6
    assert _rel(Lg, g["L"]) < 2e-6


@pytest.mark.parametrize("name", ALL)
def test_c_tile_loop_matches_reference(name):
    """oracle/scfa_oracle.c (the CPU baseline) on kernel-order operands: outputs and the
    reference's tiles_computed at BlockSpec(64, 64) and (128, 128)."""
    from oracle import c_oracle

    meta, g = gc.load(name)
    q, k, v, dO = gc.inputs(meta)
    B, H, D = meta["B"], meta["H"], meta["D"]
    kind = meta["kind"]
    if kind == "dense":
        eq, ek, ev, edo = (x.reshape(B * H, -1, D) for x in (q, k, v, dO))
        qi = ki = np.arange(meta["T_Q"])
        qi, ki = np.broadcast_to(qi, (B * H, qi.size)), np.broadcast_to(ki, (B * H, ki.size))
        qh = kh = None
        qord = kord = None
        excl = False
    else:
        qi = g["q_idx"].reshape(B * H, -1).astype(np.int64)
        ki = g["k_idx"].reshape(B * H, -1).astype(np.int64)
        if kind == "qk":
            qord = np.swapaxes(g["q_index"], 1, 2).reshape(B * H, -1)
            kord = np.swapaxes(g["k_index"], 1, 2).reshape(B * H, -1)
            qh = kh = None
            excl = False
        else:
            qord, kord = qi, ki
            qh = g["q_hash_sorted"].reshape(B * H, -1).astype(np.int64)
            kh = g["k_hash_sorted"].reshape(B * H, -1).astype(np.int64)
            excl = meta["exclude_self"]
        heads = lambda x: np.swapaxes(x, 1, 2).reshape(B * H, x.shape[1], D)
        take = lambda x, o: np.take_along_axis(heads(x), o[..., None].astype(np.int64), 1)
        eq, ek, ev, edo = take(q, qord), take(k, kord), take(v, kord), take(dO, qord)
    o, m, l, tiles = c_oracle.forward(eq, ek, ev, qi, ki, qh, kh, exclude_self=excl, threads=4)
    assert tiles == meta["tiles_computed"]
    t128 = c_oracle.forward(eq, ek, ev, qi, ki, qh, kh, B_m=128, B_n=128, exclude_self=excl, threads=4)[3]
    assert t128 == meta["tiles_computed_128"]
    dq, dk, dv = c_oracle.backward(eq, ek, ev, o, m, l, edo, qi, ki, qh, kh, exclude_self=excl, threads=4)
    np.testing.assert_allclose(m.reshape(g["M"].shape)[np.isfinite(g["M"])], g["M"][np.isfinite(g["M"])],
                               rtol=1e-5, atol=1e-5)
    if kind == "dense":
        outs = [x.reshape(B, H, -1, D) for x in (o, dq, dk, dv)]
    else:
        def back(x, order, valid, T):  # kernel order -> boundary (B, T, H, D); pad slots dropped
            out = np.zeros((B * H, T, D))
            for bh in range(B * H):
                out[bh, order[bh][valid[bh]].astype(np.int64)] = x[bh][valid[bh]]
            return np.swapaxes(out.reshape(B, H, T, D), 1, 2)
        qv, kv = qi >= 0, ki < orc.KEY_PAD
        TQ, TK = meta["T_Q"], meta["T_KV"]
        outs = [back(o, qord, qv, TQ), back(dq, qord, qv, TQ), back(dk, kord, kv, TK), back(dv, kord, kv, TK)]
    for label, got in zip(("O", "dq", "dk", "dv"), outs):
        assert _rel(got, g[label]) < 2e-4, f"{label}: rel {_rel(got, g[label]):.2e}"


# ---------------------------------------------------------------- reference known answers

def test_kat_compaction():
    """test_qk.py:62-79: drop {4,5} -> [0,1,2,3,6,7]; unequal heads -> padded [1,4,6,-1,-1]."""
    keep = np.ones((1, 8, 1))
    keep[0, [4, 5], 0] = 0
    order, cnt = orc.compact_order(keep)
    assert list(order[0, :6, 0]) == [0, 1, 2, 3, 6, 7] and cnt[0, 0] == 6
    keep = np.zeros((1, 8, 2))
    keep[0, [1, 4, 6], 0] = 1
    keep[0, [0, 2, 3, 5, 7], 1] = 1
    order, cnt = orc.compact_order(keep)
    buf = int(cnt.max())
    assert buf == 5
    assert list(order[0, :, 1][:5]) == [0, 2, 3, 5, 7]
    assert list(orc.padded(order[:, :buf], cnt, orc.QUERY_PAD)[0, :, 0]) == [1, 4, 6, -1, -1]


def test_kat_schedules():
    """test_qk.py:114-120, test_hash.py:160-178."""
    idx = np.arange(64)
    assert list(orc.causal_j_stops(idx, idx, 16, 16)) == [1, 2, 3, 4]
    assert list(orc.causal_j_stops([0, 1, 2, 3, 6, 7], [0, 2, 3, 5, 6, 7], 2, 2)) == [1, 2, 3]
    z = np.zeros(64, np.int64)
    a, e = orc.hash_tile_ranges(z, idx, z, idx, 16, 16)
    assert not a.any() and list(e) == [1, 2, 3, 4]
    a, e = orc.hash_tile_ranges([0, 0, 1, 1], [0, 1, 2, 3], [0, 0, 1, 1], [0, 1, 6, 7], 2, 2)
    assert list(a) == [0, 1] and list(e) == [1, 1]


def test_kat_colour_grouping():
    """test_hash.py:127-140 (Fig. 1 colours)."""
    kb = np.array([1, 1, 0, 2, 2, 1, 0, 1])
    qb = np.array([1, 1, 0, 2, 2, 0, 1, 2])
    assert list(orc.bucket_order(kb)) == [2, 6, 0, 1, 5, 7, 3, 4]
    assert list(orc.bucket_order(qb)) == [2, 5, 0, 1, 6, 3, 4, 7]


def test_kat_visible_counts():
    """test_qk.py:148-162: queries [0,1,2,3,6,7] over keys [0,2,3,5,6,7] see [1,1,2,3,5,6] keys."""
    vis = orc.visibility(np.array([0, 1, 2, 3, 6, 7]), np.array([0, 2, 3, 5, 6, 7]))
    assert list(vis.sum(-1)) == [1, 1, 2, 3, 5, 6]
    q = np.zeros((6, 4))
    k = np.zeros((6, 4))
    v = np.arange(24, dtype=np.float64).reshape(6, 4)
    O, _, _ = orc.attention(q, k, v, vis)
    for r, n in enumerate([1, 1, 2, 3, 5, 6]):
        np.testing.assert_allclose(O[r], v[:n].mean(0))


def test_kat_exclude_self_earliest_zero():
    """test_hash.py:221-230: the earliest member of each bucket sees nothing under exclude_self."""
    b = np.array([0, 0, 0, 1, 1, 1])
    vis = orc.visibility(np.arange(6), np.arange(6), b, b, exclude_self=True)
    rng = np.random.default_rng(67)
    q, k, v = (rng.standard_normal((6, 3)) for _ in range(3))
    O, M, L = orc.attention(q, k, v, vis)
    assert not O[0].any() and not O[3].any() and O[1].any()
    assert np.isneginf(M[0]) and L[0] == 0


def test_live_pairs_formulas():
    """P_live for hash = sum_g c_g(c_g-1)/2; for QK = kept causal pairs."""
    rng = np.random.default_rng(0)
    h = rng.integers(0, 5, (1, 64, 2))
    vis = orc.visibility(np.arange(64), np.arange(64), h.transpose(0, 2, 1), h.transpose(0, 2, 1), True)
    assert orc.live_pairs_hash(h, h) == int(vis.sum())
    qk = rng.random((1, 64, 2)) > 0.4
    kk = rng.random((1, 64, 2)) > 0.4
    vis = orc.visibility(np.arange(64), np.arange(64))[None, None] & qk.transpose(0, 2, 1)[..., :, None] & \
        kk.transpose(0, 2, 1)[..., None, :]
    assert orc.live_pairs_qk(qk, kk) == int(vis.sum())
