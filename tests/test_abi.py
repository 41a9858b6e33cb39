"""CPU checks of the drop-in boundary: the C-ABI library builds for sm_100a, loads,
and exports every entry point include/scfa_b200.h declares (no GPU needed)."""

import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "scfa_b200.h")


def _declared():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(scfa_\w+)\s*\(", text, flags=re.M)))


def test_header_declares_entry_points():
    names = _declared()
    assert "scfa_attn_fwd" in names and "scfa_attn_bwd_dkdv" in names and "scfa_hash_sort" in names
    assert len(names) >= 17


def test_library_exports_every_declared_symbol():
    from paper_2306_01160_b200 import _lib
    from paper_2306_01160_b200.build import build

    build()
    lib = ctypes.CDLL(_lib.LIB_PATH)
    missing = [n for n in _declared() if not hasattr(lib, n)]
    assert not missing, f"symbols declared in the header but not exported: {missing}"
    # the Python binding covers exactly the declared surface
    assert sorted(_lib.exported_symbols()) == _declared()


def test_library_is_sm100a():
    from paper_2306_01160_b200 import _lib

    out = os.popen(f"cuobjdump -lelf {_lib.LIB_PATH} 2>/dev/null").read()
    if not out:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out


def test_error_codes_map_to_reference_taxonomy():
    from paper_2306_01160_b200 import _lib
    from paper_2306_01160_b200.errors import ContractError, ShapeError

    with pytest.raises(ShapeError):
        _lib.raise_for(_lib.ERR_SHAPE, "x")
    with pytest.raises(ContractError):
        _lib.raise_for(_lib.ERR_CONTRACT, "x")


def test_abi_version_matches_the_package():
    from paper_2306_01160_b200 import _lib

    assert _lib.load().scfa_abi_version() == _lib.ABI_VERSION
