"""ctypes binding of the C-ABI engine (include/scfa_b200.h).

The product path has exactly one implementation: the sm_100a kernels in
``lib/libscfa_b200.so``.  If the library or a CUDA device is missing every
entry point raises; there is no CPU fallback.
"""

import ctypes
import os

import torch

from .errors import (
    ContractError,
    FormatError,
    NumericError,
    ParameterError,
    ScfaError,
    ShapeError,
)

_HERE = os.path.dirname(os.path.abspath(__file__))
# SCFA_LIB overrides the path (A/B timing of two builds); the default is the in-tree build
LIB_PATH = os.environ.get("SCFA_LIB") or os.path.join(_HERE, "lib", "libscfa_b200.so")

ABI_VERSION = 6  # include/scfa_b200.h / scfa_abi_version()
OK = 0
ERR_SHAPE, ERR_FORMAT, ERR_PARAM, ERR_NUMERIC, ERR_CONTRACT, ERR_CUDA = 1, 2, 3, 4, 5, 6
DT_F32, DT_F64, DT_U8, DT_I32, DT_I64, DT_BF16 = 0, 1, 2, 3, 4, 5
FLAG_EXCLUDE_SELF, FLAG_HASH = 1, 2

_ERRORS = {
    ERR_SHAPE: ShapeError,
    ERR_FORMAT: lambda m: FormatError(m, -1),
    ERR_PARAM: ParameterError,
    ERR_NUMERIC: NumericError,
    ERR_CONTRACT: ContractError,
}

_P, _I, _L, _F = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_float

# name -> argtypes (all return int status, except the two introspection calls)
_SIGS = {
    "scfa_qk_compact": [_P, _I, _L, _L, _L, _L, _L, _L, _P, _P, _P, _P, _P],
    "scfa_qk_prepare": [_P, _I, _L, _L, _L, _P, _I, _L, _L, _L, _L, _L, _L, _L, _P, _P, _P, _P, _P, _P, _P, _P,
                        _P, _P, _P, _P, _P],
    "scfa_hash_sort": [_P, _I, _L, _L, _L, _L, _L, _L, _P, _I, _L, _L, _P, _P, _P, _P, _P],
    "scfa_gather_rows": [_P, _I, _L, _L, _L, _L, _L, _L, _P, _L, _L, _P, _P],
    "scfa_gather_rows3": [_I, _P, _P, _P, _P, _I, _L, _L, _L, _P, _P, _P],
    "scfa_permute_rows3": [_I, _P, _P, _P, _P, _I, _L, _L, _L, _L, _P, _P],
    "scfa_hash_prepare": [_P, _I, _L, _L, _L, _L, _L, _L, _I, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P],
    "scfa_row_map": [_P, _L, _L, _L, _L, _L, _L, _P, _P],
    "scfa_scatter_rows": [_P, _I, _L, _L, _L, _L, _P, _L, _P, _I, _L, _L, _L, _P],
    "scfa_build_aux": [_P, _P, _L, _L, _L, _L, _L, ctypes.c_int32, ctypes.c_int32, _P, _I, _L, _L, _L,
                       ctypes.c_int32, _P, _I, _L, _L, _P, _P, _P],
    "scfa_invert_index": [_P, _I, _L, _L, _L, _L, _L, _L, _L, _P, _P, _P],
    "scfa_pack_index": [_P, _I, _L, _L, _L, _L, _L, ctypes.c_int32, _P, _P],
    "scfa_validate_qk": [_P, _P, _L, _L, _L, _L, _L, _P, _P],
    "scfa_validate_sorted": [_P, _P, _L, _L, _L, _P, _P],
    "scfa_build_schedule": [_P, _P, _P, _P, _L, _L, _L, _L, _L, _I, _P, _P, _I, _P, _P, _L, _P, _P, _L, _P, _P,
                            _L, _P, _P],
    "scfa_ref_schedule": [_P, _P, _P, _P, _L, _L, _L, _L, _L, _L, _L, _I, _P, _P, _P, _P],
    "scfa_lsh_buckets": [_P, _I, _L, _L, _L, _L, _L, _L, _L, _L, _P, _I, _P, _L, _L, _L, _P],
    "scfa_attn_fwd": [_P, _P, _P, _L, _L, _L, _L, _P, _P, _L, _L, _P, _P, _L, _F, _L, _L, _I, _P, _P, _P, _P,
                      _P, _P, _L, _L, _P, _P, _P],
    "scfa_zero_dropped": [_P, _I, _L, _L, _L, _L, _L, _L, _P, _L, _P, _L, _P],
    "scfa_bwd_prep_rank": [_P, _P, _L, _L, _L, _L, _L, _P, _P, _P, _P],
    "scfa_bwd_prep": [_P, _P, _P, _P, _P, _L, _L, _L, _L, _P, _L, _L, _P, _P, _P, _P],
    "scfa_attn_bwd_dq": [_P, _P, _P, _P, _L, _L, _L, _L, _P, _P, _L, _L, _P, _P, _P, _P, _L, _F, _L, _L, _I,
                         _P, _P, _P, _L, _L, _P, _P, _P, _P, _P],
    "scfa_attn_bwd": [_P, _P, _P, _P, _L, _L, _L, _L, _P, _P, _P, _L, _L, _P, _P, _P, _P, _L, _F, _L, _L, _L, _I,
                      _P, _P, _P, _P],
    "scfa_debug_timing": [_P, _L],
    "scfa_debug_ctas_per_sm": [_I, _L],
    "scfa_attn_bwd_dkdv": [_P, _P, _P, _P, _L, _L, _L, _L, _P, _P, _L, _L, _P, _P, _P, _P, _L, _F, _L, _L,
                           _I, _P, _P, _P, _P, _L, _L, _P, _P],
}

_lib = None


def load():
    """Load (once) and return the engine library; raise if it is unavailable."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ScfaError(
            f"CUDA engine not built: {LIB_PATH} is missing "
            "(run `python -m paper_2306_01160_b200.build`)"
        )
    lib = ctypes.CDLL(LIB_PATH)
    for name, argtypes in _SIGS.items():
        fn = getattr(lib, name)
        fn.argtypes = argtypes
        fn.restype = ctypes.c_int
    lib.scfa_last_error.restype = ctypes.c_char_p
    lib.scfa_last_error.argtypes = []
    lib.scfa_abi_version.restype = ctypes.c_int
    lib.scfa_abi_version.argtypes = []
    if lib.scfa_abi_version() != ABI_VERSION:  # a stale build: fail loudly, not with bad arguments
        raise ScfaError(f"{LIB_PATH}: ABI {lib.scfa_abi_version()}, this package needs {ABI_VERSION} (rebuild it)")
    _lib = lib
    return lib


def exported_symbols():
    return list(_SIGS) + ["scfa_last_error", "scfa_abi_version"]


def raise_for(code, what=""):
    if code == OK:
        return
    msg = load().scfa_last_error().decode(errors="replace") or what
    cls = _ERRORS.get(code)
    if cls is None:
        raise ScfaError(f"{what}: CUDA engine failure: {msg}")
    raise cls(f"{what}: {msg}" if what else msg)


def raise_for_status(code, msg):
    """A device status word (SCFA_ERR_*) -> the reference exception class."""
    cls = _ERRORS.get(code)
    if cls is None:
        raise ScfaError(f"engine status {code}: {msg}")
    raise cls(msg)


# kernels launched per successful call (for launch accounting in bench.py)
KERNELS_PER_CALL = {"scfa_build_schedule": 2, "scfa_invert_index": 2, "scfa_hash_prepare": 2}
launches = 0
EVENT_HOOK = None  # optional callable(name, phase) used by bench.py to time each entry point


def call(name, *args, kernels=None):
    global launches
    if EVENT_HOOK is not None:
        EVENT_HOOK(name, 0)
    rc = getattr(load(), name)(*args)
    if EVENT_HOOK is not None:
        EVENT_HOOK(name, 1)
    raise_for(rc, name)
    launches += KERNELS_PER_CALL.get(name, 1) if kernels is None else kernels


def ptr_array(tensors):
    """Host array of device pointers (void*[n]) for the multi-tensor entry points."""
    return (ctypes.c_void_p * len(tensors))(*[t.data_ptr() for t in tensors])


def i64_array(values):
    return (ctypes.c_int64 * len(values))(*[int(v) for v in values])


def ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def stream_ptr(device=None):
    return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)


def dtype_code(t):
    m = {
        torch.float32: DT_F32,
        torch.float64: DT_F64,
        torch.uint8: DT_U8,
        torch.bool: DT_U8,
        torch.int32: DT_I32,
        torch.int64: DT_I64,
    }
    if t.dtype not in m:
        raise ShapeError(f"unsupported index dtype {t.dtype}")
    return m[t.dtype]


def require_cuda():
    if not torch.cuda.is_available():
        raise ScfaError("the SCFA engine needs a CUDA device (sm_100a); none is visible")
    load()
