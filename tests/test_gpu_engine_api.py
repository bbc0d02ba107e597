"""The reference's engine-behaviour tests (tests/test_engine.py of the
reference package), re-run against the device Engine through its public API:
rotation timing, reload-free repeated selections, bitwise determinism,
stream validation, GQA groups sharing one page union."""

import numpy as np
import pytest

from oracle.workload import Spec, generate

pytestmark = pytest.mark.gpu


def _small(seed=0, n_tokens=700, layers=3, kv_heads=2, d=16, d_prime=8, G=1, **cfg):
    from paper_2604_10539_b200.engine import Engine, EngineConfig
    keys, values, queries, _ = generate(Spec(kind="clustered", n_tokens=n_tokens, d=d, d_prime=d_prime, clusters=8,
                                             layers=layers, kv_heads=kv_heads, query_heads_per_group=G, seed=seed))
    c = EngineConfig(layers=layers, kv_heads=kv_heads, d=d, d_prime=d_prime, query_heads_per_group=G, seed=seed,
                     max_tokens=n_tokens, **cfg)
    return Engine, c, keys, values, queries


def test_window_rotation_fires_at_capacity_minus_one(cuda_ok):
    """test_engine.py:77-100: with the prompt a multiple of the page size the
    first step rotates (one page offloaded, s tokens indexed); the fresh window
    page then takes s-1 appends before the next rotation."""
    Engine, cfg, k, v, q = _small(token_budget=8)
    n0 = 512
    eng = Engine(cfg).prefill(k, v, n0)
    s = cfg.page_size
    pts0 = eng.forest.info(0)["n_points"]
    assert eng.rotation_due()
    eng.decode_step(n0, q[n0], k[n0], v[n0])
    assert int(eng.rot_stats[0, 1]) == 1                 # one offload transaction
    assert eng.forest.info(0)["n_points"] == pts0 + s    # the page's s tokens indexed
    steps_until = 0   # counts the rotating step itself, as the reference's loop does
    for t in range(1, 2 * s):
        due = eng.rotation_due()
        eng.decode_step(n0 + t, q[n0 + t], k[n0 + t], v[n0 + t])
        steps_until += 1
        if due:
            break
    assert steps_until == s - 1
    assert int(eng.rot_stats[0, 1]) == 2
    assert eng.forest.info(0)["n_points"] == pts0 + 2 * s


def test_identical_consecutive_queries_reload_nothing(cuda_ok):
    """test_engine.py:132-140."""
    Engine, cfg, k, v, q = _small(token_budget=16)
    n0 = 520   # newest window page at fill 8: no rotation for a while
    q = q.copy()
    q[n0 + 1] = q[n0]
    eng = Engine(cfg).prefill(k, v, n0)
    _, first = eng.decode_step(n0, q[n0], k[n0], v[n0])
    _, second = eng.decode_step(n0 + 1, q[n0 + 1], k[n0 + 1], v[n0 + 1])
    assert first.pages_loaded > 0
    assert second.pages_loaded == 0 and second.transactions == 0


def test_decode_requires_prefill_and_stream_alignment(cuda_ok):
    """test_engine.py:143-150."""
    from paper_2604_10539_b200.errors import ConfigError, InputError
    Engine, cfg, k, v, q = _small()
    eng = Engine(cfg)
    with pytest.raises(ConfigError):
        eng.decode_step(500, q[500], k[500], v[500])
    eng.prefill(k, v, 500)
    with pytest.raises(InputError):
        eng.decode_step(503, q[503], k[503], v[503])   # skips ahead


def test_run_determinism_bitwise(cuda_ok):
    """test_engine.py:176-183 (evaluation metrics included)."""
    results = []
    for _ in range(2):
        Engine, cfg, k, v, q = _small(seed=33, evaluate=True, token_budget=24)
        eng = Engine(cfg).prefill(k, v, 500)
        rows = []
        for t in range(12):
            out, m = eng.decode_step(500 + t, q[500 + t], k[500 + t], v[500 + t])
            rows.append((m.__dict__.copy(), np.asarray(out.cpu()).tobytes()))
        results.append(rows)
    assert results[0] == results[1]


def test_gqa_groups_share_the_union(cuda_ok):
    """test_engine.py:153-164: the group's pages are the union of every head's
    pages, and the heads attend the same token set."""
    Engine, cfg, k, v, q = _small(G=2, token_budget=8)
    eng = Engine(cfg).prefill(k, v, 500)
    eng.decode_step(500, q[500], k[500], v[500])
    ids, counts, pages, npages = eng.selected()
    for tr in range(ids.shape[0]):
        t2p = eng.forest.export(tr)["tok2page"]
        per_head = set()
        for g in range(ids.shape[1]):
            per_head |= set(int(t2p[t]) for t in ids[tr, g, :counts[tr, g]])
        assert per_head == set(int(p) for p in pages[tr, :npages[tr]])


def test_page_bound_fuzz(cuda_ok):
    """Acceptance test 05 (test_acceptance.py:107-132): 10,000 random queries
    with random k in [1, 64] against one tree; every selection has at most k
    pages, and the tokens loaded with them fit in pages x page size.  Batched
    by k: the same tree repeated along the launch, one query per row."""
    import torch
    from paper_2604_10539_b200.dci import SearchBudget
    Engine, cfg, k, v, q = _small(seed=105, n_tokens=2049, layers=3, kv_heads=1, d=16, d_prime=8, token_budget=64)
    eng = Engine(cfg).prefill(k, v, 2048)
    f, tree = eng.forest, eng.T - 1                  # layer 2, head 0
    pages_of = {p: len(toks) for p, (role, toks) in f.export(tree)["pages"].items()}
    rng = np.random.default_rng(1055)
    qs = rng.normal(size=(10_000, 16)).astype(np.float32)
    ks = rng.integers(1, 65, size=10_000)
    s = cfg.page_size
    violations = 0
    for kk in np.unique(ks):
        rows = np.nonzero(ks == kk)[0]
        b = SearchBudget.for_k(int(kk))
        _, _, pages, npages = f.query(torch.full((len(rows),), tree, dtype=torch.int32), qs[rows][:, None, :],
                                      b.k, b.beam, b.visit_cap)
        pages, npages = pages.cpu().numpy(), npages.cpu().numpy()
        for i in range(len(rows)):
            sel = pages[i, :npages[i]]
            loaded = sum(pages_of[int(p)] for p in sel)
            if loaded > len(sel) * s or len(sel) > kk:
                violations += 1
    assert violations == 0
