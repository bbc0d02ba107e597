"""Generate golden vectors by running the UNMODIFIED reference package.

Runs only in the build container (it imports /root/reference/pkg/src read
only); the resulting .npz fixtures are committed and travel to the GPU box.
Usage:  python tests/golden/make_golden.py
Every input is rounded to fp32-representable values first (the parity
contract feeds both sides identical fp32 inputs).
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
import icecache as ic  # noqa: E402
from icecache.dci import SENTINEL_LEVEL  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def f32(x):
    return np.asarray(x, dtype=np.float64).astype(np.float32).astype(np.float64)


def clustered(seed, n, d, clusters, spread=0.1):
    rng = np.random.default_rng(seed)
    centers = rng.normal(size=(clusters, d))
    centers /= np.linalg.norm(centers, axis=1, keepdims=True)
    labels = rng.integers(0, clusters, size=n)
    keys = centers[labels] + rng.normal(size=(n, d)) * spread / np.sqrt(d)
    return f32(keys), f32(centers)


def export_tree(tree, store):
    nodes = []
    for n in sorted(tree.nodes.values(), key=lambda x: x.node_id):
        nodes.append([n.node_id, n.level, -1 if n.parent_id is None else n.parent_id,
                      n.owner_id, list(map(int, n.member_ids)), list(map(int, n.page_ids))])
    out = dict(levels=tree.levels, top=tree.top_node_id,
               point_level={str(k): v for k, v in tree.point_level.items()},
               nodes=nodes, scale=tree.scale.c, scale_clamps=tree.scale_clamps,
               distance_evals=tree.distance_evals, query_count=tree.query_count)
    if store is not None:
        out["pages"] = {str(pid): [p.role, list(map(int, p.token_ids))]
                        for pid, p in store.pages.items()}
    return out


def tree_cases():
    """(name, n, d, r, seed, page_size, k, n_queries, n_inserts)."""
    return [
        ("clu_d16", 1500, 16, 0.15, 5, 8, 16, 40, 200),
        ("clu_d128", 4000, 128, 0.1, (0, 1, 2), 16, 256, 24, 96),
        ("flat_d8", 700, 8, 0.02, 9, 16, 8, 20, 300),      # big nodes: P-DCI paths
        ("clu_d64_r3", 3000, 64, 0.3, 11, 16, 32, 30, 120),
    ]


def make_tree_goldens():
    for name, n, d, r, seed, s, k, nq, nins in tree_cases():
        keys, centers = clustered(7 * len(name) + n, n + nins, d, 16)
        vals = f32(np.random.default_rng(n).normal(size=(n + nins, 4)))
        store = ic.TierStore(d, 4)
        pairs = [(i, keys[i]) for i in range(n)]
        tree = ic.dci_indexing(pairs, r, seed=seed, values=[vals[i] for i in range(n)],
                               store=store, page_size=s)
        build = export_tree(tree, store)
        lifted = np.stack([tree.lifted(i) for i in range(n)])
        rng = np.random.default_rng(1000 + n)
        qs = f32(centers[rng.integers(0, len(centers), size=nq)] +
                 rng.normal(size=(nq, d)) * 0.1 / np.sqrt(d))
        budget = ic.SearchBudget.for_k(k)
        topk, evals = [], []
        for q in qs:
            before = tree.distance_evals
            topk.append(tree.query(ic.transform_query(q), SENTINEL_LEVEL, k, budget))
            evals.append(tree.distance_evals - before)
        exh = [tree.query(ic.transform_query(q), SENTINEL_LEVEL, k, ic.SearchBudget.exhaustive(k))
               for q in qs[:5]]
        levels = []
        for i in range(n, n + nins):
            levels.append(tree.insert(i, keys[i], vals[i]))
        tree.check_invariants()
        after = export_tree(tree, store)
        topk2 = [tree.query(ic.transform_query(q), SENTINEL_LEVEL, k, budget) for q in qs]
        meta = dict(name=name, n=n, d=d, r=r, seed=seed if isinstance(seed, int) else list(seed),
                    page_size=s, k=k, build=build, after=after, topk=topk, evals=evals,
                    exhaustive=exh, insert_levels=levels, topk_after=topk2)
        np.savez_compressed(os.path.join(OUT, f"tree_{name}.npz"), keys=keys.astype(np.float32),
                            values=vals.astype(np.float32), queries=qs.astype(np.float32),
                            lifted=lifted[:300], meta=json.dumps(meta))
        print("tree", name, "levels", tree.levels, "nodes", len(tree.nodes))


def engine_cases():
    return [
        # name, spec kwargs, cfg kwargs, n_prefill, steps
        ("mini", dict(n_tokens=700, d=32, d_prime=16, clusters=8, layers=3, kv_heads=2,
                      query_heads_per_group=2, seed=3),
         dict(token_budget=24, skip_layers=1), 512, 40),
        ("c1", dict(n_tokens=4096 + 16, d=128, d_prime=128, clusters=32, layers=1, kv_heads=8,
                    query_heads_per_group=4, seed=0),
         dict(token_budget=256, skip_layers=0), 4096, 16),
        # selection reuse (engine.py:321-363): anchors every 3rd indexed layer
        ("reuse", dict(n_tokens=1024 + 40, d=32, d_prime=16, clusters=8, layers=8, kv_heads=2,
                       query_heads_per_group=2, seed=11),
         dict(token_budget=24, skip_layers=2, reuse_stride=3), 1024, 40),
        # evaluation metrics (engine.py:536-566): recall / hit rate / mass / error
        ("eval", dict(n_tokens=700, d=32, d_prime=16, clusters=8, layers=3, kv_heads=2,
                      query_heads_per_group=2, seed=3),
         dict(token_budget=24, skip_layers=1, evaluate=True), 512, 20),
        ("eval_reuse", dict(n_tokens=1024 + 40, d=32, d_prime=16, clusters=8, layers=8, kv_heads=2,
                            query_heads_per_group=2, seed=11),
         dict(token_budget=24, skip_layers=2, reuse_stride=3, evaluate=True), 1024, 20),
        # acceptance 06 (tests/test_acceptance.py:135-153): TokenOrderBaseline hit rates
        ("baseline", dict(n_tokens=10_100, d=64, d_prime=32, clusters=32, layers=3, kv_heads=1,
                          query_heads_per_group=1, seed=106),
         dict(token_budget=64, evaluate=True, compare_baseline=True), 10_000, 100),
    ]


def make_engine_goldens(only=None):
    for name, sk, ck, n_prefill, steps in engine_cases():
        if only and name not in only:
            continue
        spec = ic.WorkloadSpec(kind="clustered", **sk)
        wl = ic.generate_workload(spec)
        wl.keys[:] = f32(wl.keys)
        wl.values[:] = f32(wl.values)
        wl.queries[:] = f32(wl.queries)
        cfg = ic.EngineConfig(layers=sk["layers"], kv_heads=sk["kv_heads"],
                              query_heads_per_group=sk["query_heads_per_group"], d=sk["d"],
                              d_prime=sk["d_prime"], seed=sk["seed"], **ck)
        eng = ic.Engine(cfg).prefill(wl, n_prefill)
        tok_log = []
        orig = eng._select_tokens

        def spy(q, layer, kv_head, budget=None):
            res = orig(q, layer, kv_head, budget)
            tok_log[-1].append([layer, kv_head, list(map(int, res))])
            return res
        eng._select_tokens = spy
        rows, outs = [], []
        for t in range(steps):
            tok_log.append([])
            o, m = eng.decode_step(wl.decode_step(n_prefill, t))
            rows.append(m.__dict__)
            outs.append(np.stack([[o[l][qh].value_out for qh in range(cfg.n_query_heads)]
                                  for l in range(cfg.layers)]))
        meta = dict(name=name, spec=sk, cfg=ck, n_prefill=n_prefill, steps=steps, rows=rows,
                    tokens=tok_log)
        np.savez_compressed(os.path.join(OUT, f"engine_{name}.npz"),
                            outputs=np.stack(outs).astype(np.float64), meta=json.dumps(meta))
        print("engine", name, rows[0], rows[-1])


def make_llama_golden():
    """The reference engine on q/k/v from a (random-init) Llama forward:
    tests/golden/llama_small.icet, written by tools/llama_trace.py."""
    from icecache.workload import load_trace
    wl = load_trace(os.path.join(OUT, "llama_small.icet"))
    sp = wl.spec
    cfg = ic.EngineConfig(layers=sp.layers, kv_heads=sp.kv_heads, query_heads_per_group=sp.query_heads_per_group,
                          d=sp.d, d_prime=sp.d_prime, token_budget=32, skip_layers=1, evaluate=True, seed=5)
    n_prefill, steps = 600, 100
    eng = ic.Engine(cfg).prefill(wl, n_prefill)
    tok_log = []
    orig = eng._select_tokens

    def spy(q, layer, kv_head, budget=None):
        res = orig(q, layer, kv_head, budget)
        tok_log[-1].append([layer, kv_head, list(map(int, res))])
        return res
    eng._select_tokens = spy
    rows, outs = [], []
    for t in range(steps):
        tok_log.append([])
        o, m = eng.decode_step(wl.decode_step(n_prefill, t))
        rows.append(m.__dict__)
        outs.append(np.stack([[o[l][qh].value_out for qh in range(cfg.n_query_heads)] for l in range(cfg.layers)]))
    meta = dict(name="llama", trace="llama_small.icet", cfg=dict(token_budget=32, skip_layers=1, evaluate=True,
                                                                 seed=5),
                n_prefill=n_prefill, steps=steps, rows=rows, tokens=tok_log)
    np.savez_compressed(os.path.join(OUT, "engine_llama.npz"), outputs=np.stack(outs).astype(np.float64),
                        meta=json.dumps(meta))
    print("engine llama", rows[0], rows[-1])


def make_trace_golden():
    """An ICET trace written by the reference's save_trace (workload.py:175-192)
    and the arrays its load_trace (:195-224) returns."""
    from icecache.workload import WorkloadSpec, generate_workload, load_trace, save_trace
    spec = WorkloadSpec(kind="clustered", n_tokens=40, d=12, d_prime=6, clusters=4, layers=3, kv_heads=2,
                        query_heads_per_group=2, seed=11)
    path = os.path.join(OUT, "trace_small.icet")
    save_trace(generate_workload(spec), path)
    back = load_trace(path)
    np.savez_compressed(os.path.join(OUT, "trace_small.npz"), keys=back.keys, values=back.values,
                        queries=back.queries, shape=np.array([back.spec.layers, back.spec.kv_heads,
                                                              back.spec.query_heads_per_group, back.spec.d,
                                                              back.spec.d_prime, back.spec.n_tokens]))
    print("trace", os.path.getsize(path), "bytes")


if __name__ == "__main__":
    which = sys.argv[1:] or ["tree", "engine", "trace", "llama"]
    if "llama" in which:
        make_llama_golden()
        which = [w for w in which if w != "llama"] if len(which) > 1 else []
    if "tree" in which:
        make_tree_goldens()
    if "trace" in which:
        make_trace_golden()
    if "engine" in which:
        make_engine_goldens([w for w in which if w not in ("tree", "engine", "trace", "llama")] or None)
