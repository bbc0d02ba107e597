"""Bit-level numerics shared by the oracle and (by construction) the device.

Every function names the reference line it restates and the exact operation
order the CUDA kernels use, so the oracle and the device agree bit for bit.
"""

from __future__ import annotations

import numpy as np

SCALE_HEADROOM = 1.05          # geometry.py:31
DPAD = 128                      # device row width (keys zero-padded to 128 dims)


def pairwise_sum(a: np.ndarray) -> np.ndarray:
    """Row sums of a 2-D fp64 array in NumPy's pairwise order.

    NumPy's `add.reduce` over a contiguous axis (used by
    `np.linalg.norm(mat, axis=1)` in `dci.py:517` and `(keys*keys).sum(-1)`
    in `geometry.py:53`) sums blocks of <=128 elements with eight interleaved
    accumulators and splits longer rows recursively.  The device kernel
    `lift_rows` uses the same order, so norms agree bit for bit.
    """
    a = np.asarray(a, dtype=np.float64)
    n = a.shape[1]
    if n < 8:
        r = a[:, 0].copy() if n else np.zeros(a.shape[0])
        for i in range(1, n):
            r = r + a[:, i]
        return r
    if n <= 128:
        r = [a[:, j].copy() for j in range(8)]
        i = 8
        lim = n - (n % 8)
        while i < lim:
            for j in range(8):
                r[j] = r[j] + a[:, i + j]
            i += 8
        res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]))
        for i in range(lim, n):
            res = res + a[:, i]
        return res
    n2 = n // 2
    n2 -= n2 % 8
    return pairwise_sum(a[:, :n2]) + pairwise_sum(a[:, n2:])


def sq_norms(keys: np.ndarray) -> np.ndarray:
    keys = np.atleast_2d(np.asarray(keys, dtype=np.float64))
    return pairwise_sum(keys * keys)


def key_scale(keys: np.ndarray, headroom: float = SCALE_HEADROOM) -> float:
    """`KeyScale.from_keys` (geometry.py:47-56): c = 1.05 * sqrt(max |k|^2)."""
    keys = np.atleast_2d(np.asarray(keys, dtype=np.float64))
    if keys.size == 0:
        raise ValueError("empty key set")
    max_norm = float(np.sqrt(sq_norms(keys).max()))
    if max_norm == 0.0:
        max_norm = 1.0
    return headroom * max_norm


def lift_keys64(keys: np.ndarray, c: float):
    """Batch lifting of `dci.py:517-523` in fp64.

    Returns (rows[n,d] fp64, tail[n] fp64, over[n] bool).  Over-scale keys are
    clamped to [k/|k|, 0] (counted in scale_clamps).
    """
    keys = np.atleast_2d(np.asarray(keys, dtype=np.float64))
    norms = np.sqrt(sq_norms(keys))
    over = norms > c
    safe = np.where(over, norms, c)
    rows = keys / safe[:, None]
    tail = np.sqrt(np.maximum(0.0, 1.0 - (norms / safe) ** 2))
    return rows, tail, over


def lift_keys32(keys: np.ndarray, c: float):
    """fp32 storage image of the lifted keys: (rows[n,DPAD] f32, tail[n] f32, over)."""
    rows, tail, over = lift_keys64(keys, c)
    n, d = rows.shape
    out = np.zeros((n, DPAD), dtype=np.float32)
    out[:, :d] = rows.astype(np.float32)
    return out, tail.astype(np.float32), over


def lift_query32(q: np.ndarray) -> np.ndarray:
    """`transform_query` (geometry.py:89-98) rounded to fp32, padded to DPAD.

    The norm uses the pairwise order (the reference's 1-D `np.linalg.norm`
    goes through BLAS ddot; the two agree except in the last fp64 ulp).
    """
    q = np.asarray(q, dtype=np.float64).reshape(1, -1)
    norm = float(np.sqrt(sq_norms(q)[0]))
    if norm == 0.0:
        raise ZeroDivisionError("zero query")
    out = np.zeros(DPAD, dtype=np.float32)
    out[: q.shape[1]] = (q[0] / norm).astype(np.float32)
    return out


def d2_fp32(rows: np.ndarray, tail: np.ndarray, q: np.ndarray, q_tail=0.0) -> np.ndarray:
    """Squared lifted distance `sum (p - q)^2` (dci.py:311-312) in fp32.

    Fixed order (mirrors lane_sq4 / warp_sum_butterfly / d2_finish in
    csrc/icb.cuh): lane l of a warp owns dims 4l..4l+3 and forms
    fma(d3,d3, fma(d2,d2, fma(d1,d1, d0*d0))) of the differences; lanes are
    combined by an xor butterfly 16, 8, 4, 2, 1 (commutative adds, so every
    lane holds the same value); the tail term enters last as
    fma(dt, dt, f), dt = p_d - q_d (q_d = 0 for decode queries, the lifted
    key's tail for insert-time parent searches).  Fused multiply-adds cannot
    be expressed exactly in NumPy, so this calls the C restatement
    (oracle/c/oracle_nn.c:oracle_d2_fp32, compiled with explicit fmaf).
    """
    from .clib import d2_fp32 as _c_d2
    return _c_d2(rows, tail, q, q_tail)


def pack_keys(d2: np.ndarray, ids: np.ndarray) -> np.ndarray:
    """64-bit ranking keys (d2 bits << 32 | id): ascending == (d2, id) order."""
    bits = np.asarray(d2, dtype=np.float32).view(np.uint32).astype(np.uint64)
    return (bits << np.uint64(32)) | np.asarray(ids, dtype=np.uint64)


def key_ids(keys: np.ndarray) -> np.ndarray:
    return (np.asarray(keys, dtype=np.uint64) & np.uint64(0xFFFFFFFF)).astype(np.int64)
