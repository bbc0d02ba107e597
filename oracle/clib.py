"""ctypes loader of the oracle's C helpers (oracle/c/oracle_nn.c).
TEST INFRASTRUCTURE ONLY."""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None
_dp = ctypes.POINTER(ctypes.c_double)
_fp = ctypes.POINTER(ctypes.c_float)


def lib():
    """Load (building on first use) the oracle's C helper library."""
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "_build", "liboracle.so")
        src = os.path.join(_HERE, "c", "oracle_nn.c")
        if not os.path.exists(path) or os.path.getmtime(path) < os.path.getmtime(src):
            subprocess.check_call(["make", "-s", "-C", _HERE])
        h = ctypes.CDLL(path)
        h.oracle_nn_parents.argtypes = [_dp, ctypes.c_int64, _dp, ctypes.c_int64, ctypes.c_int,
                                        ctypes.POINTER(ctypes.c_int32)]
        h.oracle_project.argtypes = [_dp, ctypes.c_int, _dp, ctypes.c_int64, ctypes.c_int, _dp]
        h.oracle_d2_fp32.argtypes = [_fp, _fp, ctypes.c_int64, _fp, ctypes.c_float, _fp]
        _LIB = h
    return _LIB


def d2_fp32(rows, tail, q, q_tail=0.0) -> np.ndarray:
    rows = np.ascontiguousarray(np.asarray(rows, dtype=np.float32).reshape(-1, 128))
    tail = np.ascontiguousarray(np.asarray(tail, dtype=np.float32).reshape(-1))
    q = np.ascontiguousarray(np.asarray(q, dtype=np.float32).reshape(128))
    out = np.empty(rows.shape[0], dtype=np.float32)
    lib().oracle_d2_fp32(rows.ctypes.data_as(_fp), tail.ctypes.data_as(_fp), rows.shape[0],
                         q.ctypes.data_as(_fp), ctypes.c_float(float(np.float32(q_tail))),
                         out.ctypes.data_as(_fp))
    return out
