"""Synthetic q/k/v streams, restating workload.py:119-167 (generate_workload)
draw for draw, so the oracle and the reference see the same bits.
TEST INFRASTRUCTURE ONLY."""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass
class Spec:
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


def _unit(v):
    return v / np.linalg.norm(v, axis=-1, keepdims=True)


def generate(spec: Spec, fp32: bool = True):
    """(keys [n,L,H,d], values [n,L,H,d'], queries [n,L,H*G,d]) fp64 arrays.

    With fp32=True every array is rounded to fp32-representable values (the
    parity contract feeds both sides identical fp32 inputs).
    """
    rng = np.random.default_rng(spec.seed)
    n, L, H, G = spec.n_tokens, spec.layers, spec.kv_heads, spec.query_heads_per_group
    d, dv = spec.d, spec.d_prime
    values = rng.normal(size=(n, L, H, dv)) / np.sqrt(dv)
    keys = np.empty((n, L, H, d))
    queries = np.empty((n, L, H * G, d))
    needle = None
    if spec.kind == "uniform":
        keys[:] = rng.normal(size=(n, L, H, d)) / np.sqrt(d)
        queries[:] = _unit(rng.normal(size=(n, L, H * G, d))) * np.sqrt(d)
    elif spec.kind == "clustered":
        centers = _unit(rng.normal(size=(H, spec.clusters, d)))
        cluster_of = rng.integers(0, spec.clusters, size=n)
        query_cluster = rng.integers(0, spec.clusters, size=n)
        sigma = spec.cluster_spread / np.sqrt(d)
        jitter = spec.layer_jitter * sigma
        key_noise = rng.normal(size=(n, H, d)) * sigma
        query_noise = rng.normal(size=(n, H * G, d)) * sigma
        for layer in range(L):
            lk = rng.normal(size=(n, H, d)) * jitter
            lq = rng.normal(size=(n, H * G, d)) * jitter
            for h in range(H):
                keys[:, layer, h] = centers[h, cluster_of] + key_noise[:, h] + lk[:, h]
                ctr = centers[h, query_cluster]
                for g in range(G):
                    qh = h * G + g
                    queries[:, layer, qh] = (ctr + query_noise[:, qh] + lq[:, qh]) * np.sqrt(d)
    elif spec.kind == "planted_needle":
        target = _unit(rng.normal(size=(H, d)))
        base = rng.normal(size=(n, L, H, d)) * (spec.cluster_spread / np.sqrt(d))
        keys[:] = _unit(target[None, None, :, :] + base)
        needle = int(rng.integers(n // 4, 3 * n // 4))
        for h in range(H):
            keys[needle, :, h] = spec.needle_gain * target[h]
            for g in range(G):
                queries[:, :, h * G + g, :] = target[h] * np.sqrt(d)
    else:
        raise ValueError(spec.kind)
    if fp32:
        keys = keys.astype(np.float32).astype(np.float64)
        values = values.astype(np.float32).astype(np.float64)
        queries = queries.astype(np.float32).astype(np.float64)
    return keys, values, queries, needle
