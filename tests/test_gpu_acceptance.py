"""Reference acceptance criteria re-run on the device path (tests/test_acceptance.py
and tests/test_engine.py of the reference), plus a long-generation insert
stress (C5-shaped, scaled down) against the oracle with structural invariants."""

import math

import numpy as np
import pytest

from oracle.engine import OConfig, OracleEngine, full_attention
from oracle.workload import Spec, generate

pytestmark = pytest.mark.gpu


def _engine(shape, **kw):
    from paper_2604_10539_b200.engine import Engine, EngineConfig
    return Engine(EngineConfig(**shape, **kw))


def test_full_budget_equals_full_attention(cuda_ok):
    """Acceptance 2 (reference tests/test_acceptance.py:45-67): unbounded
    budget, beam and visit cap attend every token -> full attention."""
    sk = dict(n_tokens=1074, d=32, d_prime=16, clusters=8, layers=4, kv_heads=4, seed=102)
    keys, values, queries, _ = generate(Spec(kind="clustered", **sk))
    shape = dict(layers=4, kv_heads=4, d=32, d_prime=16, seed=102)
    eng = _engine(shape, token_budget=10**6, beam=2**61, visit_cap=2**61, kv_dtype="fp32",
                  max_tokens=1074 + 1).prefill(keys, values, 1024)
    worst = 0.0
    for t in range(50):
        tok = 1024 + t
        out, _ = eng.decode_step(tok, queries[tok], keys[tok], values[tok], metrics=False)
        out = out.cpu().numpy()
        for layer in range(4):
            for h in range(4):
                _, ref = full_attention(queries[tok, layer, h], keys[:tok + 1, layer, h],
                                        values[:tok + 1, layer, h])
                worst = max(worst, np.linalg.norm(out[layer, h] - ref) / np.linalg.norm(ref))
    assert worst <= 1e-5, worst   # fp32 accumulation (the reference's fp64 bound is 1e-6)


def test_planted_needle_retrieved(cuda_ok):
    """Acceptance 3 (reference tests/test_acceptance.py:70-90): the needle token
    is in the attended set of every indexed layer."""
    hits = 0
    seeds = range(20)
    for seed in seeds:
        sk = dict(n_tokens=4001, d=32, d_prime=8, cluster_spread=4.0, needle_gain=2.0, layers=3,
                  kv_heads=1, seed=seed)
        keys, values, queries, needle = generate(Spec(kind="planted_needle", **sk))
        eng = _engine(dict(layers=3, kv_heads=1, d=32, d_prime=8, seed=seed), token_budget=64,
                      kv_dtype="fp32", max_tokens=4001).prefill(keys, values, 4000)
        eng.decode_step(4000, queries[4000], keys[4000], values[4000], metrics=False)
        ids, counts, pages, npages = eng.selected()
        ok = True
        for tr in range(eng.T):
            toks = set()
            ex = eng.forest.export(tr)
            for p in pages[tr, :npages[tr]]:
                toks |= set(ex["pages"][int(p)][1])
            ok &= needle in toks
        hits += ok
    assert hits == len(seeds)


def test_long_generation_inserts_match_oracle(cuda_ok):
    """C5-shaped stress, scaled: 2k prompt + 320 decode steps = 20 rotations
    x 16 device inserts per tree (P-DCI parent searches, grown nodes, new
    pages); every step's selections and metrics equal the oracle's, and the
    final trees satisfy check_invariants (dci.py:453-476)."""
    sk = dict(n_tokens=2048 + 330, d=64, d_prime=64, clusters=16, layers=2, kv_heads=2,
              query_heads_per_group=2, seed=5)
    keys, values, queries, _ = generate(Spec(kind="clustered", **sk))
    shape = dict(layers=2, kv_heads=2, query_heads_per_group=2, d=64, d_prime=64, seed=5)
    cfg = dict(token_budget=32, skip_layers=1, promotion_ratio=0.2)
    oeng = OracleEngine(OConfig(**shape, **cfg)).prefill(keys, values, 2048)
    eng = _engine(shape, **cfg, kv_dtype="fp32", max_tokens=2048 + 330).prefill(keys, values, 2048)
    for t in range(320):
        tok = 2048 + t
        _, om, trace = oeng.decode_step(tok, queries[tok], keys[tok], values[tok])
        _, m = eng.decode_step(tok, queries[tok], keys[tok], values[tok])
        for k in ("pages_selected", "pages_loaded", "tokens_loaded", "bytes_moved"):
            assert getattr(m, k) == om[k], (t, k)
        ids, counts, pages, npages = eng.selected()
        for h in range(2):
            assert list(pages[h, :npages[h]]) == trace["pages"][(1, h)], (t, h)
    for h in range(2):
        ex = eng.forest.export(h)
        ot = oeng.heads[(1, h)].tree
        ot.check_invariants()
        assert [(n[0], n[1], n[2], n[3], n[4]) for n in ex["nodes"]] == \
            [(i, lv, par, own, mem) for i, lv, par, own, mem, _ in ot.export()["nodes"]]
        _check_invariants(ex)


def _check_invariants(ex):
    """check_invariants (dci.py:453-476) on the exported device tree."""
    nodes = {n[0]: n for n in ex["nodes"]}
    levels = ex["info"]["levels"]
    top = ex["info"]["top_node"]
    assert {n[1] for n in nodes.values()} == set(range(1, levels + 1))
    leaf_members = []
    for i, lv, par, own, mem in nodes.values():
        assert mem
        if i == top:
            assert par == -1 and own == -1
        else:
            assert nodes[par][1] == lv + 1 and own in nodes[par][4]
        if lv == 1:
            leaf_members += list(mem)
            fills = sum(len(ex["pages"][p][1]) for p in ex["leaf_pages"][i])
            assert fills == len(mem)
    assert sorted(leaf_members) == sorted(ex["point_level"])
    assert len(set(leaf_members)) == len(leaf_members)


def test_short_prompt_falls_back_to_full_attention(cuda_ok):
    """reference tests/test_engine.py:50-58: a prompt shorter than sink+window+1
    pages attends exactly over everything."""
    sk = dict(n_tokens=600, d=16, d_prime=8, clusters=8, layers=3, kv_heads=2, seed=0)
    keys, values, queries, _ = generate(Spec(kind="clustered", **sk))
    eng = _engine(dict(layers=3, kv_heads=2, d=16, d_prime=8), token_budget=16,
                  kv_dtype="fp32", max_tokens=64).prefill(keys, values, 40)
    assert eng.fallback
    out, m = eng.decode_step(40, queries[40], keys[40], values[40])
    _, ref = full_attention(queries[40, 2, 0], keys[:41, 2, 0], values[:41, 2, 0])
    assert np.linalg.norm(out.cpu().numpy()[2, 0] - ref) / np.linalg.norm(ref) < 1e-5
    assert m.pages_selected == 0 and m.dci_queries == 0


@pytest.mark.parametrize("G,d", [(1, 12), (3, 40), (8, 128)])
def test_odd_shapes_match_oracle(cuda_ok, G, d):
    """GQA ratios 1, 3 (padded to 4 inside the kernel) and 8; key dims not a
    multiple of 4; rotation at step 0."""
    sk = dict(n_tokens=700, d=d, d_prime=d, clusters=8, layers=2, kv_heads=2,
              query_heads_per_group=G, seed=G)
    keys, values, queries, _ = generate(Spec(kind="clustered", **sk))
    shape = dict(layers=2, kv_heads=2, query_heads_per_group=G, d=d, d_prime=d, seed=G)
    cfg = dict(token_budget=16, skip_layers=1)
    oeng = OracleEngine(OConfig(**shape, **cfg)).prefill(keys, values, 512)
    eng = _engine(shape, **cfg, kv_dtype="fp32", max_tokens=700).prefill(keys, values, 512)
    for t in range(20):
        tok = 512 + t
        oout, om, trace = oeng.decode_step(tok, queries[tok], keys[tok], values[tok])
        out, m = eng.decode_step(tok, queries[tok], keys[tok], values[tok])
        ids, counts, pages, npages = eng.selected()
        for h in range(2):
            for g in range(G):
                assert list(ids[h, g, :counts[h, g]]) == trace["tokens"][(1, h * G + g)]
        o = out.cpu().numpy()
        assert (np.linalg.norm(o - oout, axis=-1) / np.linalg.norm(oout, axis=-1)).max() < 1e-3


def test_selection_reuse_acceptance(cuda_ok):
    """Acceptance 9 (reference tests/test_acceptance.py:210-238) on the device:
    reuse stride 3 issues ceil(6/3) = 2 DCI queries per step (6 vanilla) and
    loses at most 0.10 recall (evaluate=True metrics computed on the device)."""
    sk = dict(n_tokens=4100, d=64, d_prime=32, clusters=32, cluster_spread=0.1, layers=8, kv_heads=1, seed=109)
    keys, values, queries, _ = generate(Spec(kind="clustered", **sk))
    base = dict(layers=8, kv_heads=1, d=64, d_prime=32, token_budget=64, evaluate=True, seed=109)
    recalls, queries_per_step = {}, {}
    for label, stride in (("vanilla", 0), ("reuse", 3)):
        eng = _engine({}, reuse_stride=stride, kv_dtype="fp32", max_tokens=4100, **base).prefill(keys, values, 4000)
        r, qc = [], []
        for t in range(60):
            tok = 4000 + t
            _, m = eng.decode_step(tok, queries[tok], keys[tok], values[tok])
            r.append(m.recall_at_k)
            qc.append(m.dci_queries)
        recalls[label] = float(np.mean(r))
        queries_per_step[label] = qc
    assert all(q == 2 for q in queries_per_step["reuse"])
    assert all(q == 6 for q in queries_per_step["vanilla"])
    assert recalls["vanilla"] - recalls["reuse"] <= 0.10, recalls
