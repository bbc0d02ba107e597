"""Synthetic q/k/v streams generated on the device.

Same distributions as the reference generator (workload.py:119-167 of the
reference package): clustered keys around per-head unit centers with a small
per-layer jitter, queries aimed at a cluster center and scaled by sqrt(d),
values N(0, 1/d').  Drawn with torch's CUDA RNG (not NumPy's streams), so
they are statistically -- not bitwise -- equal to the reference's; parity
tests use the oracle's bit-identical NumPy generator instead.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import torch


@dataclass
class DeviceStream:
    keys: torch.Tensor      # [n, L, H, d]
    values: torch.Tensor    # [n, L, H, d']
    queries: torch.Tensor   # [steps, L, H*G, d]  (decode tokens only)
    n_prefill: int


def _unit(x):
    return x / x.norm(dim=-1, keepdim=True)


def clustered_stream(n_prefill: int, steps: int, layers: int, kv_heads: int, G: int, d: int, d_prime: int, *,
                     clusters: int = 32, spread: float = 0.1, jitter: float = 0.1, seed: int = 0,
                     device="cuda") -> DeviceStream:
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    n = n_prefill + steps
    H, L = kv_heads, layers
    kw = dict(device=device, generator=g)
    centers = _unit(torch.randn(H, clusters, d, **kw))
    cluster_of = torch.randint(0, clusters, (n,), **kw)
    qcluster = torch.randint(0, clusters, (steps,), **kw)
    sigma = spread / math.sqrt(d)
    jit = jitter * sigma
    hidx = torch.arange(H, device=device)
    base = centers[hidx[None, :], cluster_of[:, None]]                       # [n, H, d]
    base = base + torch.randn(n, H, d, **kw) * sigma
    keys = torch.empty((n, L, H, d), dtype=torch.float32, device=device)
    for layer in range(L):
        keys[:, layer] = base + torch.randn(n, H, d, **kw) * jit
    values = torch.randn(n, L, H, d_prime, **kw) / math.sqrt(d_prime)
    qbase = centers[hidx[None, :], qcluster[:, None]]                        # [steps, H, d]
    qbase = qbase[:, :, None, :].expand(steps, H, G, d) + torch.randn(steps, H, G, d, **kw) * sigma
    queries = torch.empty((steps, L, H * G, d), dtype=torch.float32, device=device)
    for layer in range(L):
        queries[:, layer] = ((qbase + torch.randn(steps, H, G, d, **kw) * jit) * math.sqrt(d)).reshape(steps, H * G, d)
    return DeviceStream(keys, values, queries, n_prefill)
