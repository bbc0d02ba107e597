"""Pin the CPU oracle against golden vectors produced by the unmodified
reference (tests/golden/make_golden.py).  CPU only."""

import numpy as np
import pytest

from conftest import load_golden
from oracle import numerics as nm
from oracle.dci import SENTINEL, build
from oracle.engine import OConfig, OracleEngine
from oracle.store import OStore
from oracle.workload import Spec, generate

TREES = ["clu_d16", "clu_d128", "flat_d8", "clu_d64_r3"]


def _canon_nodes(nodes):
    return [(n[0], n[1], n[2], n[3], tuple(n[4]), tuple(n[5])) for n in nodes]


def _build(z, meta):
    n, d = meta["n"], meta["d"]
    keys = z["keys"].astype(np.float64)
    vals = z["values"].astype(np.float64)
    seed = meta["seed"] if isinstance(meta["seed"], int) else tuple(meta["seed"])
    store = OStore(d, 4)
    tree = build([(i, keys[i]) for i in range(n)], meta["r"], seed=seed,
                 values=[vals[i] for i in range(n)], store=store, page_size=meta["page_size"])
    return tree, store, keys, vals


def _near_tie_ok(tree, q32, got, want, eps=2e-6):
    """Ranked lists may differ only where fp32 distances sit within eps of the
    k-th boundary (the reference ranks fp64 distances, the device fp32)."""
    if got == want:
        return True
    rows = np.stack([tree.row[p] for p in set(got) | set(want)])
    ids = list(set(got) | set(want))
    d2 = dict(zip(ids, nm.d2_fp32(rows, np.array([tree.tail[p] for p in ids]), q32).tolist()))
    boundary = max(d2[p] for p in want)
    for p in set(got) ^ set(want):
        if abs(d2[p] - boundary) > eps:
            return False
    # same set: order flips only between near-equal distances
    for a, b in zip(got, want):
        if a != b and abs(d2[a] - d2[b]) > eps:
            return False
    return True


@pytest.mark.parametrize("name", TREES)
def test_build_structure_matches_reference(name):
    z, meta = load_golden(f"tree_{name}.npz")
    tree, store, keys, _ = _build(z, meta)
    ref = meta["build"]
    assert tree.c == ref["scale"]
    assert tree.levels == ref["levels"] and tree.top == ref["top"]
    assert tree.point_level == {int(k): v for k, v in ref["point_level"].items()}
    assert tree.export()["nodes"] == _canon_nodes(ref["nodes"])
    assert {pid: p.tokens for pid, p in store.pages.items()} == \
        {int(k): v[1] for k, v in ref["pages"].items()}
    # lifted rows: fp64 build lift equals the reference's bit for bit
    rows64, tail64, _ = nm.lift_keys64(keys[: meta["n"]], tree.c)
    lifted = z["lifted"]
    m = lifted.shape[0]
    assert np.array_equal(rows64[:m], lifted[:, :-1])
    assert np.array_equal(tail64[:m], lifted[:, -1])


@pytest.mark.parametrize("name", TREES)
def test_queries_match_reference(name):
    z, meta = load_golden(f"tree_{name}.npz")
    tree, store, keys, _ = _build(z, meta)
    k = meta["k"]
    for q, want, ev in zip(z["queries"], meta["topk"], meta["evals"]):
        q32 = nm.lift_query32(q.astype(np.float64))
        before = tree.distance_evals
        got = tree.query(q32, SENTINEL, k, 2 * k, 4 * k)
        assert _near_tie_ok(tree, q32, got, want)
        if got == want:
            assert tree.distance_evals - before == ev
    for q, want in zip(z["queries"], meta["exhaustive"]):
        q32 = nm.lift_query32(q.astype(np.float64))
        got = tree.query(q32, SENTINEL, k, 2**62, 2**62)
        assert _near_tie_ok(tree, q32, got, want)


@pytest.mark.parametrize("name", TREES)
def test_inserts_match_reference(name):
    z, meta = load_golden(f"tree_{name}.npz")
    tree, store, keys, vals = _build(z, meta)
    n = meta["n"]
    levels = [tree.insert(i, keys[i], vals[i]) for i in range(n, n + len(meta["insert_levels"]))]
    assert levels == meta["insert_levels"]
    tree.check_invariants()
    ref = meta["after"]
    assert tree.levels == ref["levels"] and tree.top == ref["top"]
    assert tree.export()["nodes"] == _canon_nodes(ref["nodes"])
    assert {pid: p.tokens for pid, p in store.pages.items()} == \
        {int(k): v[1] for k, v in ref["pages"].items()}
    k = meta["k"]
    for q, want in zip(z["queries"], meta["topk_after"]):
        q32 = nm.lift_query32(q.astype(np.float64))
        assert _near_tie_ok(tree, q32, tree.query(q32, SENTINEL, k, 2 * k, 4 * k), want)


@pytest.mark.parametrize("name", ["mini", "c1", "reuse"])
def test_engine_matches_reference(name):
    z, meta = load_golden(f"engine_{name}.npz")
    sk, ck = meta["spec"], meta["cfg"]
    keys, values, queries, _ = generate(Spec(kind="clustered", **sk))
    cfg = OConfig(layers=sk["layers"], kv_heads=sk["kv_heads"],
                  query_heads_per_group=sk["query_heads_per_group"], d=sk["d"],
                  d_prime=sk["d_prime"], seed=sk["seed"], **ck)
    n0 = meta["n_prefill"]
    eng = OracleEngine(cfg).prefill(keys, values, n0)
    G = cfg.query_heads_per_group
    for t in range(meta["steps"]):
        tok = n0 + t
        out, m, trace = eng.decode_step(tok, queries[tok], keys[tok], values[tok])
        row = meta["rows"][t]
        for key in ("pages_selected", "pages_loaded", "tokens_loaded", "bytes_moved",
                    "transactions", "dci_queries"):
            assert m[key] == row[key], (t, key)
        # per query head ranked token lists, in the reference's call order
        calls = meta["tokens"][t]
        idx = 0
        stride = cfg.reuse_stride
        for layer in range(cfg.skip_layers, cfg.layers):
            if stride >= 2 and (layer - cfg.skip_layers) % stride:
                continue   # reuse layer: no query (select_with_reuse, engine.py:331-363)
            for h in range(cfg.kv_heads):
                for g in range(G):
                    rl, rh, want = calls[idx]
                    idx += 1
                    assert (rl, rh) == (layer, h)
                    got = trace["tokens"][(layer, h * G + g)]
                    assert set(got) == set(want), (t, layer, h, g)
        assert idx == len(calls)
        ref_out = z["outputs"][t]
        err = np.linalg.norm(out - ref_out, axis=-1) / np.linalg.norm(ref_out, axis=-1)
        assert err.max() < 1e-10


def test_oracle_engine_on_llama_trace_matches_reference():
    """The oracle on the Llama-forward trace (tools/llama_trace.py) against the
    reference's own run: step metrics and per-head token sets."""
    import os
    from paper_2604_10539_b200.trace import load_trace
    z, meta = load_golden("engine_llama.npz")
    tr = load_trace(os.path.join(os.path.dirname(__file__), "golden", meta["trace"]))
    keys, values, queries = (tr.keys.astype(np.float64), tr.values.astype(np.float64), tr.queries.astype(np.float64))
    ck = meta["cfg"]
    cfg = OConfig(layers=tr.layers, kv_heads=tr.kv_heads, query_heads_per_group=tr.query_heads_per_group, d=tr.d,
                  d_prime=tr.d_prime, token_budget=ck["token_budget"], skip_layers=ck["skip_layers"], seed=ck["seed"])
    n0 = meta["n_prefill"]
    eng = OracleEngine(cfg).prefill(keys, values, n0)
    G = cfg.query_heads_per_group
    for t in range(meta["steps"]):
        tok = n0 + t
        _, m, trace = eng.decode_step(tok, queries[tok], keys[tok], values[tok])
        for key in ("pages_selected", "pages_loaded", "tokens_loaded", "bytes_moved", "transactions", "dci_queries"):
            assert m[key] == meta["rows"][t][key], (t, key)
        calls = meta["tokens"][t]
        for i, (layer, h, want) in enumerate(calls):
            g = i % G
            assert set(trace["tokens"][(layer, h * G + g)]) == set(want), (t, layer, h, g)
