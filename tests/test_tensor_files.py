"""SCFA tensor container (tensors.py:110-154): files written by the reference's
save_tensor load to the same arrays, ours are byte-identical, and every defect raises
FormatError with the reference's byte offset."""

import os
import struct

import numpy as np
import pytest

from paper_2306_01160_b200 import FormatError, ShapeError, load_tensor, save_tensor

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.mark.parametrize("name", ["f32", "f64"])
def test_reads_reference_files_and_writes_identical_bytes(name, tmp_path):
    want = np.load(os.path.join(GOLD, "tensor_files.npz"))[name]
    ref_path = os.path.join(GOLD, f"tensor_{name}.scfa")
    got = load_tensor(ref_path)
    assert got.dtype == want.dtype and np.array_equal(got, want)
    ours = tmp_path / "x.scfa"
    save_tensor(ours, want)
    assert ours.read_bytes() == open(ref_path, "rb").read()


def test_torch_round_trip(tmp_path):
    import torch

    x = torch.randn(1, 2, 7, 3, dtype=torch.float64)
    save_tensor(tmp_path / "t.scfa", x)
    assert np.array_equal(load_tensor(tmp_path / "t.scfa"), x.numpy())


def _corrupt(tmp_path, mutate):
    x = np.arange(2 * 1 * 3 * 2, dtype=np.float32).reshape(2, 1, 3, 2)
    p = tmp_path / "c.scfa"
    save_tensor(p, x)
    raw = bytearray(p.read_bytes())
    raw = mutate(raw)
    p.write_bytes(bytes(raw))
    with pytest.raises(FormatError) as e:
        load_tensor(p)
    return e.value.offset


def test_format_errors_carry_offsets(tmp_path):
    assert _corrupt(tmp_path, lambda r: r[:10]) == 10                                  # truncated header
    assert _corrupt(tmp_path, lambda r: b"XCFA" + r[4:]) == 0                          # magic
    assert _corrupt(tmp_path, lambda r: r[:4] + struct.pack("<I", 2) + r[8:]) == 4     # version
    assert _corrupt(tmp_path, lambda r: r[:8] + b"\x02" + r[9:]) == 8                  # precision byte
    assert _corrupt(tmp_path, lambda r: r[:17] + struct.pack("<Q", 0) + r[25:]) == 17  # extent 1 = 0
    full = 41 + 12 * 4
    assert _corrupt(tmp_path, lambda r: r[:-4]) == full - 4                            # short payload
    assert _corrupt(tmp_path, lambda r: r + b"\0") == full                             # long payload


def test_save_rejects_bad_tensors(tmp_path):
    with pytest.raises(ShapeError):
        save_tensor(tmp_path / "a", np.zeros((2, 3)))
    with pytest.raises(ShapeError):
        save_tensor(tmp_path / "b", np.zeros((1, 1, 1, 1), dtype=np.int32))
    with pytest.raises(ShapeError):
        save_tensor(tmp_path / "c", np.full((1, 1, 1, 1), np.nan))
