"""LSH bucket producer (hash_sparse.py:34-52): oracle pinned to the reference's golden ids
(CPU), and the scfa_lsh_buckets kernel against the same ids (GPU)."""

import os

import numpy as np
import pytest
import torch

from oracle import scfa_oracle as orc

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "lsh_small.npz")
NBS = (2, 6, 16, 64)


@pytest.fixture(scope="module")
def gold():
    return np.load(GOLD)


@pytest.mark.parametrize("nb", NBS)
def test_oracle_matches_reference_ids(gold, nb):
    assert np.array_equal(orc.lsh_buckets(gold["x"], nb, 31), gold[f"ids_nb{nb}"])


def test_zero_vectors_take_bucket_zero(gold):
    assert (gold["ids_nb16"][0, :4] == 0).all()


@pytest.mark.gpu
@pytest.mark.parametrize("nb", NBS)
@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
def test_gpu_lsh_matches_reference_ids(gold, nb, dtype):
    import paper_2306_01160_b200 as scfa

    x = torch.from_numpy(gold["x"]).to("cuda", dtype)
    got = scfa.lsh_buckets(x, nb, 31)
    assert got.dtype == torch.int64 and got.is_cuda
    assert torch.equal(got.cpu(), torch.from_numpy(gold[f"ids_nb{nb}"]))


@pytest.mark.gpu
def test_gpu_lsh_strided_bf16_and_scale_invariance():
    import paper_2306_01160_b200 as scfa

    g = torch.Generator().manual_seed(3)
    base = torch.randn(2, 300, 4, 64, generator=g, dtype=torch.float64)
    want = orc.lsh_buckets(base.numpy(), 16, 7)
    # a strided view (heads of a wider tensor) and a positive rescale give the same ids
    wide = torch.zeros(2, 300, 8, 64, dtype=torch.float64)
    wide[:, :, ::2] = base * 3.5
    got = scfa.lsh_buckets(wide[:, :, ::2].cuda(), 16, 7)
    assert torch.equal(got.cpu(), torch.from_numpy(want))
    # bf16 input: ids of the bf16-rounded vectors
    xb = base.to(torch.bfloat16)
    want_b = orc.lsh_buckets(xb.double().numpy(), 16, 7)
    assert torch.equal(scfa.lsh_buckets(xb.cuda(), 16, 7).cpu(), torch.from_numpy(want_b))


@pytest.mark.gpu
def test_gpu_lsh_rejects_bad_bucket_counts():
    import paper_2306_01160_b200 as scfa
    from paper_2306_01160_b200.errors import ParameterError

    x = torch.randn(1, 8, 1, 16, device="cuda")
    for nb in (0, 3, 66):
        with pytest.raises(ParameterError):
            scfa.lsh_buckets(x, nb, 0)
