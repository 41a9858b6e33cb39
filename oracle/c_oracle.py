"""ctypes wrapper of oracle/scfa_oracle.c (TEST INFRASTRUCTURE ONLY).

Float32 restatement of the reference's tiled forward/backward with the
reference's BlockSpec schedule; used as the CPU baseline ("kind": "port")
and as a fast oracle for larger parity cases.
"""

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "lib", "liboracle.so")
_lib = None


def build():
    src = os.path.join(HERE, "scfa_oracle.c")
    if not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(src):
        subprocess.run(["make", "-s", "-C", HERE], check=True)
    return LIB


def load():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            build()
        _lib = ctypes.CDLL(LIB)
        P, L, I, Dd = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_double
        _lib.oracle_forward.argtypes = [L, L, L, L, P, P, P, P, P, P, P, L, L, I, Dd, I, P, P, P]
        _lib.oracle_forward.restype = L
        _lib.oracle_backward.argtypes = [L, L, L, L, P, P, P, P, P, P, P, P, P, P, P, L, L, I, Dd, I, P, P, P]
        _lib.oracle_backward.restype = None
        _lib.oracle_max_threads.restype = I
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _f32(x):
    return np.ascontiguousarray(x, dtype=np.float32)


def _i64(x):
    return None if x is None else np.ascontiguousarray(x, dtype=np.int64)


def forward(q, k, v, q_idx, k_idx, q_hash=None, k_hash=None, B_m=64, B_n=64, exclude_self=False, scale=None,
            threads=0):
    """q (BH, Tq, D), k/v (BH, Tkv, D) -> (o, m, l, tiles), float32."""
    lib = load()
    q, k, v = _f32(q), _f32(k), _f32(v)
    BH, Tq, D = q.shape
    Tkv = k.shape[1]
    qi, ki = _i64(np.broadcast_to(q_idx, (BH, Tq))), _i64(np.broadcast_to(k_idx, (BH, Tkv)))
    qh, kh = _i64(q_hash), _i64(k_hash)
    if scale is None:
        scale = 1.0 / np.sqrt(D)
    o = np.empty_like(q)
    m = np.empty((BH, Tq), np.float32)
    l = np.empty((BH, Tq), np.float32)
    tiles = lib.oracle_forward(BH, Tq, Tkv, D, _p(q), _p(k), _p(v), _p(qi), _p(ki), _p(qh), _p(kh), B_m, B_n,
                               int(exclude_self), float(scale), int(threads), _p(o), _p(m), _p(l))
    return o, m, l, int(tiles)


def backward(q, k, v, o, m, l, d_out, q_idx, k_idx, q_hash=None, k_hash=None, B_m=64, B_n=64, exclude_self=False,
             scale=None, threads=0):
    lib = load()
    q, k, v, o, m, l, d_out = (_f32(x) for x in (q, k, v, o, m, l, d_out))
    BH, Tq, D = q.shape
    Tkv = k.shape[1]
    qi, ki = _i64(np.broadcast_to(q_idx, (BH, Tq))), _i64(np.broadcast_to(k_idx, (BH, Tkv)))
    qh, kh = _i64(q_hash), _i64(k_hash)
    if scale is None:
        scale = 1.0 / np.sqrt(D)
    dq, dk, dv = np.empty_like(q), np.empty_like(k), np.empty_like(v)
    lib.oracle_backward(BH, Tq, Tkv, D, _p(q), _p(k), _p(v), _p(o), _p(m), _p(l), _p(d_out), _p(qi), _p(ki),
                        _p(qh), _p(kh), B_m, B_n, int(exclude_self), float(scale), int(threads), _p(dq), _p(dk),
                        _p(dv))
    return dq, dk, dv


def max_threads():
    return int(load().oracle_max_threads())
