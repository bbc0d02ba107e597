"""ICET workload traces: the reference's binary q/k/v trace format
(workload.py:18-24 of the reference package, save_trace :175-192,
load_trace :195-224), so recorded streams drive the device engine.

Layout, all little-endian: b"ICET", u32 version (1), u32 {layers, kv_heads,
query heads per group, d, d_prime, n_tokens}, then an f32 payload ordered
token, layer, kv head with (key[d], value[d_prime], group query[d]) per
entry.  A group stores its first head's query; loading shares it across the
group's heads.  Malformed files raise TraceFormatError naming the byte offset
where the file stops making sense, as the reference does.
"""

from __future__ import annotations

import struct
from dataclasses import dataclass

import numpy as np

from .errors import TraceFormatError

TRACE_MAGIC = b"ICET"
TRACE_VERSION = 1
HEADER = struct.Struct("<4sIIIIIII")


@dataclass
class Trace:
    layers: int
    kv_heads: int
    query_heads_per_group: int
    d: int
    d_prime: int
    n_tokens: int
    keys: np.ndarray      # [n, L, H, d] float32
    values: np.ndarray    # [n, L, H, d'] float32
    queries: np.ndarray   # [n, L, H*G, d] float32 (group query shared by its heads)


def save_trace(keys, values, queries, query_heads_per_group: int, path: str) -> None:
    """keys [n,L,H,d], values [n,L,H,d'], queries [n,L,H*G,d] (any float
    dtype; stored as f32).  Writes each group's first-head query."""
    keys, values, queries = np.asarray(keys), np.asarray(values), np.asarray(queries)
    n, L, H, d = keys.shape
    dv = values.shape[-1]
    G = int(query_heads_per_group)
    if values.shape[:3] != (n, L, H) or queries.shape != (n, L, H * G, d):
        raise TraceFormatError("inconsistent key / value / query shapes for a trace")
    body = np.empty((n, L, H, 2 * d + dv), dtype="<f4")
    body[..., :d] = keys
    body[..., d:d + dv] = values
    body[..., d + dv:] = queries[:, :, ::G, :]
    with open(path, "wb") as fh:
        fh.write(HEADER.pack(TRACE_MAGIC, TRACE_VERSION, L, H, G, d, dv, n))
        fh.write(body.tobytes())


def load_trace(path: str) -> Trace:
    with open(path, "rb") as fh:
        raw = fh.read()
    if len(raw) < HEADER.size:
        raise TraceFormatError(f"truncated header: file ends at byte offset {len(raw)}")
    magic, version, L, H, G, d, dv, n = HEADER.unpack_from(raw, 0)
    if magic != TRACE_MAGIC:
        raise TraceFormatError(f"bad magic {magic!r} at byte offset 0")
    if version != TRACE_VERSION:
        raise TraceFormatError(f"unsupported trace version {version} at byte offset 4")
    if min(L, H, G, d, dv, n) < 1:
        raise TraceFormatError("non-positive shape field in header at byte offset 8")
    want = n * L * H * (2 * d + dv) * 4
    if len(raw) - HEADER.size != want:
        raise TraceFormatError(f"payload is {len(raw) - HEADER.size} bytes, expected {want}: "
                               f"file ends at byte offset {len(raw)}")
    body = np.frombuffer(raw, dtype="<f4", offset=HEADER.size).reshape(n, L, H, 2 * d + dv)
    keys = np.ascontiguousarray(body[..., :d], dtype=np.float32)
    values = np.ascontiguousarray(body[..., d:d + dv], dtype=np.float32)
    queries = np.ascontiguousarray(np.repeat(body[..., d + dv:], G, axis=2), dtype=np.float32)
    return Trace(L, H, G, d, dv, n, keys, values, queries)


def to_stream(trace: Trace, n_prefill: int, device="cuda"):
    """The trace as engine inputs: a workload.DeviceStream whose first
    n_prefill tokens are the prompt and whose queries are the decode steps'."""
    import torch

    from .workload import DeviceStream
    if not 0 < n_prefill < trace.n_tokens:
        raise TraceFormatError(f"n_prefill must lie in (0, {trace.n_tokens})")
    dev = torch.device(device)
    return DeviceStream(torch.as_tensor(trace.keys, device=dev), torch.as_tensor(trace.values, device=dev),
                        torch.as_tensor(trace.queries[n_prefill:], device=dev), n_prefill)
