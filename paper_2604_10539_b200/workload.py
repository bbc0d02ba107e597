"""Workloads: the reference's q/k/v stream types and generator, plus a
device-side generator for the bench.

* `WorkloadSpec`, `DecodeStep`, `Workload`, `generate_workload` mirror the
  reference package's (workload.py:42-167): same fields, validation and
  errors, and the generator makes the same NumPy draws in the same order, so a
  spec and seed give the same bits as the reference's `generate_workload`.
  `Engine.prefill(workload, n)` and `Engine.decode_step(step)` take these (or
  the reference's own objects: they are duck-typed on `spec`,
  `prefill_view` and `token_id/queries/keys/values`).
* `clustered_stream` draws the same distributions with torch's CUDA RNG
  (statistically -- not bitwise -- equal; too large a stream for NumPy at
  the bench's 32k x 32-layer shape).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import torch

from .errors import ConfigError

KINDS = ("clustered", "planted_needle", "uniform", "trace_file")


@dataclass
class WorkloadSpec:
    """workload.py:42-75: parameters of a synthetic workload."""

    kind: str = "clustered"
    n_tokens: int = 4096
    d: int = 64
    d_prime: int = 64
    clusters: int = 32
    cluster_spread: float = 0.1
    needle_gain: float = 2.0
    seed: int = 0
    layers: int = 4
    kv_heads: int = 2
    query_heads_per_group: int = 1
    layer_jitter: float = 0.1

    def __post_init__(self) -> None:
        if self.kind not in KINDS:
            raise ConfigError(f"unknown workload kind {self.kind!r}")
        if self.n_tokens < 1:
            raise ConfigError("n_tokens must be positive")
        if self.kind == "clustered" and self.clusters < 1:
            raise ConfigError("clustered workloads need clusters >= 1")
        if min(self.d, self.d_prime, self.layers, self.kv_heads, self.query_heads_per_group) < 1:
            raise ConfigError("dims, layers and head counts must be >= 1")

    @property
    def n_query_heads(self) -> int:
        return self.kv_heads * self.query_heads_per_group


@dataclass
class DecodeStep:
    """workload.py:78-85: one decode token's per-layer queries and own K/V."""

    token_id: int
    queries: np.ndarray   # (layers, n_query_heads, d)
    keys: np.ndarray      # (layers, kv_heads, d)
    values: np.ndarray    # (layers, kv_heads, d_prime)


@dataclass
class Workload:
    """workload.py:88-112: full q/k/v streams, sliced into a prefill region
    and decode steps."""

    spec: WorkloadSpec
    keys: np.ndarray      # (n_tokens, layers, kv_heads, d)
    values: np.ndarray    # (n_tokens, layers, kv_heads, d_prime)
    queries: np.ndarray   # (n_tokens, layers, n_query_heads, d)
    needle_token: int | None = None
    cluster_of: np.ndarray | None = field(default=None, repr=False)
    query_cluster: np.ndarray | None = field(default=None, repr=False)

    @property
    def n_tokens(self) -> int:
        return self.keys.shape[0]

    def prefill_view(self, n_prefill: int):
        if not 0 < n_prefill <= self.n_tokens:
            raise ConfigError(f"prefill length {n_prefill} outside 1..{self.n_tokens}")
        return self.keys[:n_prefill], self.values[:n_prefill]

    def decode_step(self, n_prefill: int, step: int) -> DecodeStep:
        token = n_prefill + step
        if token >= self.n_tokens:
            raise ConfigError(f"step {step} runs past the {self.n_tokens}-token stream")
        return DecodeStep(token, self.queries[token], self.keys[token], self.values[token])


def _unit_np(v: np.ndarray) -> np.ndarray:
    return v / np.linalg.norm(v, axis=-1, keepdims=True)


def generate_workload(spec: WorkloadSpec) -> Workload:
    """workload.py:119-167: the reference's draws, in its order, vectorised
    over heads (each element sees the same float operations, so the bits are
    identical).  Draw order: values; then per kind (clustered: centers,
    token clusters, query clusters, key noise, query noise, then per layer the
    key and query jitter)."""
    if spec.kind == "trace_file":
        raise ConfigError("trace_file workloads are loaded with load_trace()")
    rng = np.random.default_rng(spec.seed)
    n, L, H, G = spec.n_tokens, spec.layers, spec.kv_heads, spec.query_heads_per_group
    d, dv = spec.d, spec.d_prime
    values = rng.normal(size=(n, L, H, dv)) / np.sqrt(dv)
    keys = np.empty((n, L, H, d))
    queries = np.empty((n, L, H * G, d))
    needle = cluster_of = query_cluster = None
    if spec.kind == "uniform":
        keys[:] = rng.normal(size=(n, L, H, d)) / np.sqrt(d)
        queries[:] = _unit_np(rng.normal(size=(n, L, H * G, d))) * np.sqrt(d)
    elif spec.kind == "clustered":
        centers = _unit_np(rng.normal(size=(H, spec.clusters, d)))
        cluster_of = rng.integers(0, spec.clusters, size=n)
        query_cluster = rng.integers(0, spec.clusters, size=n)
        sigma = spec.cluster_spread / np.sqrt(d)
        jitter = spec.layer_jitter * sigma
        key_noise = rng.normal(size=(n, H, d)) * sigma
        query_noise = rng.normal(size=(n, H * G, d)) * sigma
        heads = np.arange(H)
        kctr = centers[heads[None, :], cluster_of[:, None]]                    # (n, H, d)
        qctr = centers[(np.arange(H * G) // G)[None, :], query_cluster[:, None]]   # (n, H*G, d)
        for layer in range(L):
            layer_key = rng.normal(size=(n, H, d)) * jitter
            layer_query = rng.normal(size=(n, H * G, d)) * jitter
            keys[:, layer] = kctr + key_noise + layer_key
            queries[:, layer] = (qctr + query_noise + layer_query) * np.sqrt(d)
    elif spec.kind == "planted_needle":
        target = _unit_np(rng.normal(size=(H, d)))
        base = rng.normal(size=(n, L, H, d)) * (spec.cluster_spread / np.sqrt(d))
        keys[:] = _unit_np(target[None, None, :, :] + base)
        needle = int(rng.integers(n // 4, 3 * n // 4))
        keys[needle] = spec.needle_gain * target[None, :, :]
        queries[:] = np.repeat(target, G, axis=0)[None, None] * np.sqrt(d)
    return Workload(spec, keys, values, queries, needle_token=needle, cluster_of=cluster_of,
                    query_cluster=query_cluster)


def workload_from_trace(trace) -> Workload:
    """A loaded ICET trace (trace.load_trace) as a Workload (kind trace_file)."""
    spec = WorkloadSpec(kind="trace_file", n_tokens=trace.n_tokens, d=trace.d, d_prime=trace.d_prime,
                        layers=trace.layers, kv_heads=trace.kv_heads,
                        query_heads_per_group=trace.query_heads_per_group)
    return Workload(spec, trace.keys.astype(np.float64), trace.values.astype(np.float64),
                    trace.queries.astype(np.float64))


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
                     device="cuda", dtype=torch.float32) -> DeviceStream:
    """Keys / values [n, L, H, d] in `dtype` (bf16 halves a multi-sequence
    prompt's footprint: its values are then bf16-representable fp32 inputs),
    queries [steps, L, H*G, d] fp32.  Generated layer by layer."""
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
    keys = torch.empty((n, L, H, d), dtype=dtype, device=device)
    values = torch.empty((n, L, H, d_prime), dtype=dtype, device=device)
    for layer in range(L):
        keys[:, layer] = base + torch.randn(n, H, d, **kw) * jit
    for layer in range(L):
        values[:, layer] = torch.randn(n, H, d_prime, **kw) / math.sqrt(d_prime)
    qbase = centers[hidx[None, :], qcluster[:, None]]                        # [steps, H, d]
    qbase = qbase[:, :, None, :].expand(steps, H, G, d) + torch.randn(steps, H, G, d, **kw) * sigma
    queries = torch.empty((steps, L, H * G, d), dtype=torch.float32, device=device)
    for layer in range(L):
        queries[:, layer] = ((qbase + torch.randn(steps, H, G, d, **kw) * jit) * math.sqrt(d)).reshape(steps, H * G, d)
    return DeviceStream(keys, values, queries, n_prefill)
