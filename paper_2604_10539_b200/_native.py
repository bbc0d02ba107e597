"""ctypes binding of libicecache_b200.so (the C ABI in include/icecache_b200.h).

There is no fallback: if the library is missing or a CUDA device is not
available the first call raises.
"""

from __future__ import annotations

import ctypes
import os

from .errors import (ConfigError, ConsistencyError, DegenerateQueryError, IceCacheError, InputError,
                     PolicyError)

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("ICB_LIB") or os.path.join(
    _HERE, "libicecache_b200_debug.so" if os.environ.get("ICB_DEBUG_LIB") == "1" else "libicecache_b200.so")

ICB_OK, ICB_E_INPUT, ICB_E_CONFIG, ICB_E_CONSISTENCY, ICB_E_CUDA, ICB_E_CAPACITY, ICB_E_POLICY, \
    ICB_E_DEGENERATE = range(8)
KV_F32, KV_BF16 = 0, 1
ROLE_SINK, ROLE_WINDOW, ROLE_INDEXED = 1, 2, 3
SENTINEL_LEVEL = -1

# device error bits (csrc/icb.cuh)
ERR_BITS = {
    1 << 0: (ConfigError, "node capacity exceeded"),
    1 << 1: (ConfigError, "member-pool capacity exceeded"),
    1 << 2: (ConfigError, "page capacity exceeded"),
    1 << 3: (ConfigError, "owned-node list capacity exceeded"),
    1 << 4: (InputError, "token id outside [0, tok_cap)"),
    1 << 5: (InputError, "point id already indexed"),
    1 << 6: (InputError, "query on an empty tree"),
    1 << 7: (DegenerateQueryError, "zero query cannot be normalized"),
    1 << 8: (ConsistencyError, "token is not mapped to any page"),
    1 << 9: (ConfigError, "search scratch exceeded (k or candidate count too large)"),
    1 << 10: (ConfigError, "P-DCI node too large"),
    1 << 11: (InputError, "window ring inconsistent"),
}


class icb_forest_config(ctypes.Structure):
    _fields_ = [("n_trees", ctypes.c_int32), ("dim", ctypes.c_int32), ("dim_v", ctypes.c_int32),
                ("page_size", ctypes.c_int32), ("kv_dtype", ctypes.c_int32),
                ("tok_cap", ctypes.c_int32), ("node_cap", ctypes.c_int32),
                ("page_cap", ctypes.c_int32), ("member_cap", ctypes.c_int32),
                ("own_cap", ctypes.c_int32), ("dirs_cap", ctypes.c_int32),
                ("promotion_ratio", ctypes.c_double), ("kv_host", ctypes.c_int32),
                ("pool_pages", ctypes.c_int32)]


_lib = None
P = ctypes.c_void_p
I32 = ctypes.c_int32
I64 = ctypes.c_int64

EXPORTS = {
    "icb_last_error": ([], ctypes.c_char_p),
    "icb_version": ([], ctypes.c_int),
    "icb_forest_create": ([ctypes.POINTER(icb_forest_config), ctypes.POINTER(P)], ctypes.c_int),
    "icb_forest_destroy": ([P], ctypes.c_int),
    "icb_seed_trees": ([P, P, I32, P, I32, P], ctypes.c_int),
    "icb_alloc_resident_pages": ([P, P, I32, I32, I32, I32, P, P, P, P], ctypes.c_int),
    "icb_build": ([P, P, I32, I32, P, P, P, P, P], ctypes.c_int),
    "icb_query": ([P, P, I32, I32, P, I32, I32, I64, I64, I32, P, I32, P, P, I32, P, P], ctypes.c_int),
    "icb_insert": ([P, P, I32, I32, P, P, P, P, P, P], ctypes.c_int),
    "icb_rotate_window": ([P, P, I32, I32, P, P], ctypes.c_int),
    "icb_append_window": ([P, P, I32, I32, P, P, P], ctypes.c_int),
    "icb_append_window_dev": ([P, P, I32, P, P, P, P], ctypes.c_int),
    "icb_dense_attention_dev": ([I32, I32, I32, I32, I32, P, P, P, I64, P, P, I32, P], ctypes.c_int),
    "icb_dense_append": ([I32, I32, I32, I32, P, P, P, P, I64, P, P], ctypes.c_int),
    "icb_pages_from_tokens": ([P, P, I32, P, P, P, I32, I32, P, I32, P, P], ctypes.c_int),
    "icb_node_query": ([P, I32, I32, P, I32, I64, P, P, P], ctypes.c_int),
    "icb_attended_mask": ([P, P, I32, P, I32, P, P, P], ctypes.c_int),
    "icb_query_attend": ([P, P, I32, I32, P, I32, I64, I64, P, I32, P, P, I32, P, P, P, I32, P], ctypes.c_int),
    "icb_step_attend": ([P, P, I32, I32, P, I32, I64, I64, P, I32, P, P, I32, P, P, P, I32, I32, P, P, P, P, P],
                        ctypes.c_int),
    "icb_sparse_attention": ([P, P, I32, I32, P, P, I32, P, P, P, I32, I32, P], ctypes.c_int),
    "icb_dense_attention": ([I32, I32, I32, I32, I32, P, P, P, I64, I32, P, I32, P], ctypes.c_int),
    "icb_exact_attention": ([I32, I32, I32, P, P, P, P, P, P], ctypes.c_int),
    "icb_attention_weights": ([P, P, I32, I32, P, P, I32, P, P, P, I32, P, P], ctypes.c_int),
    "icb_dense_weights": ([I32, I32, I32, I32, P, P, I64, I32, P, P], ctypes.c_int),
    "icb_tree_info": ([P, I32, P], ctypes.c_int),
    "icb_export_tree": ([P, I32] + [P] * 18, ctypes.c_int),
    "icb_read_pages": ([P, I32, P, I32, P, P], ctypes.c_int),
    "icb_clear_errors": ([P, I32], ctypes.c_int),
    "icb_errors": ([P, P, I32], ctypes.c_int),
    "icb_read_meta_c": ([P, I32, P], ctypes.c_int),
    "icb_set_scale": ([P, I32, ctypes.c_double], ctypes.c_int),
    "icb_host_pcg_doubles": ([P, I32, P, I32, I32, P], ctypes.c_int),
    "icb_pool_stats": ([P, P], ctypes.c_int),
    "icb_host_pcg_jump_doubles": ([P, I32, P, I32, ctypes.c_int64, I32, P], ctypes.c_int),
}


def lib():
    """Load the extension (raises loudly when it is missing)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: build it with `python -c 'import "
                              f"__graft_entry__; __graft_entry__.build()'` (no CPU fallback exists)")
        h = ctypes.CDLL(LIB_PATH)
        for name, (args, res) in EXPORTS.items():
            fn = getattr(h, name)
            fn.argtypes = args
            fn.restype = res
        _lib = h
    return _lib


_EXC = {ICB_E_INPUT: InputError, ICB_E_CONFIG: ConfigError, ICB_E_CONSISTENCY: ConsistencyError,
        ICB_E_POLICY: PolicyError, ICB_E_DEGENERATE: DegenerateQueryError}


def check(rc: int) -> None:
    if rc != ICB_OK:
        msg = lib().icb_last_error().decode(errors="replace")
        raise _EXC.get(rc, IceCacheError)(msg or f"icecache_b200 error {rc}")


def raise_device_error(err: int) -> None:
    """Map sticky device error bits to the reference's exception types."""
    for bit, (exc, msg) in ERR_BITS.items():
        if err & bit:
            raise exc(msg)
    raise IceCacheError(f"device error bits {err:#x}")
