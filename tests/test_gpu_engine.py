"""End-to-end decode parity: the device Engine against the oracle engine
(pinned to the reference's golden engine runs) -- ranked top-k per query
head and union pages bit-exact, step metrics equal, outputs within the
north-star tolerance.  Covers prefill layout, window rotation + device
inserts, skip layers (dense) and GQA groups."""

import numpy as np
import pytest

from conftest import load_golden
from oracle.engine import OConfig, OracleEngine
from oracle.workload import Spec, generate

pytestmark = pytest.mark.gpu

KEYS = ("pages_selected", "pages_loaded", "tokens_loaded", "bytes_moved", "transactions", "dci_queries")


def _run(name, kv="fp32", tol=1e-3, layer_serial=False, steps=None):
    from paper_2604_10539_b200.engine import Engine, EngineConfig
    z, meta = load_golden(f"engine_{name}.npz")
    sk, ck = meta["spec"], meta["cfg"]
    keys, values, queries, _ = generate(Spec(kind="clustered", **sk))
    shape = dict(layers=sk["layers"], kv_heads=sk["kv_heads"], query_heads_per_group=sk["query_heads_per_group"],
                 d=sk["d"], d_prime=sk["d_prime"], seed=sk["seed"])
    ocfg = OConfig(**shape, **ck)
    n0 = meta["n_prefill"]
    steps = steps or meta["steps"]
    oeng = OracleEngine(ocfg).prefill(keys, values, n0)
    eng = Engine(EngineConfig(**shape, **ck, kv_dtype=kv, max_tokens=n0 + steps + 1,
                              layer_serial=layer_serial)).prefill(keys, values, n0)
    G = ocfg.query_heads_per_group
    H = ocfg.kv_heads
    for t in range(steps):
        tok = n0 + t
        oout, om, trace = oeng.decode_step(tok, queries[tok], keys[tok], values[tok])
        out, m = eng.decode_step(tok, queries[tok], keys[tok], values[tok])
        for k in KEYS:
            assert getattr(m, k) == om[k], (t, k)
            assert om[k] == meta["rows"][t][k]       # oracle still on the reference's numbers
        ids, counts, pages, npages = eng.selected()
        for layer in range(ocfg.skip_layers, ocfg.layers):
            for h in range(H):
                tr = (layer - ocfg.skip_layers) * H + h
                reuse_layer = ocfg.reuse_stride >= 2 and (layer - ocfg.skip_layers) % ocfg.reuse_stride
                for g in range(G if not reuse_layer else 0):   # reuse layers run no query
                    want = trace["tokens"][(layer, h * G + g)]
                    assert list(ids[tr, g, :counts[tr, g]]) == want, (t, layer, h, g)
                assert list(pages[tr, :npages[tr]]) == trace["pages"][(layer, h)], (t, layer, h)
        o = out.cpu().numpy()
        err = np.linalg.norm(o - oout, axis=-1) / np.linalg.norm(oout, axis=-1)
        assert err.max() < tol, (t, err.max())
        ref = z["outputs"][t]
        assert (np.linalg.norm(o - ref, axis=-1) / np.linalg.norm(ref, axis=-1)).max() < tol
    return eng, oeng


def test_engine_odd_dims_vs_oracle(cuda_ok):
    """d = 30, d' = 6 (not multiples of 4): device rows are padded, but logits
    are scaled by 1/sqrt(30) (attention.py:70, d = q.size) in the dense skip
    layer and in the paged layers alike."""
    from paper_2604_10539_b200.engine import Engine, EngineConfig
    sk = dict(n_tokens=600, d=30, d_prime=6, clusters=8, layers=3, kv_heads=2, query_heads_per_group=2, seed=5)
    keys, values, queries, _ = generate(Spec(kind="clustered", **sk))
    shape = dict(layers=3, kv_heads=2, query_heads_per_group=2, d=30, d_prime=6, seed=5)
    ck = dict(token_budget=24, skip_layers=1)
    n0 = 512
    oeng = OracleEngine(OConfig(**shape, **ck)).prefill(keys, values, n0)
    eng = Engine(EngineConfig(**shape, **ck, max_tokens=600)).prefill(keys, values, n0)
    for t in range(20):
        tok = n0 + t
        oout, om, trace = oeng.decode_step(tok, queries[tok], keys[tok], values[tok])
        out, m = eng.decode_step(tok, queries[tok], keys[tok], values[tok])
        for k in KEYS:
            assert getattr(m, k) == om[k], (t, k)
        o = out.cpu().numpy()
        err = np.linalg.norm(o - oout, axis=-1) / np.linalg.norm(oout, axis=-1)
        assert err.max() < 1e-3, (t, err.max())


def test_engine_mini_fp32(cuda_ok):
    _run("mini")


def test_engine_mini_bf16(cuda_ok):
    _run("mini", kv="bf16", tol=1e-2)


def test_engine_selection_reuse(cuda_ok):
    """select_with_reuse (engine.py:321-363), reference golden 'reuse': anchors
    every 3rd indexed layer search; the others map the anchor's token union
    through their own page table (pages, metrics and dci_queries equal)."""
    eng, _ = _run("reuse")
    assert eng.anchor_layers() == [2, 5]


def test_engine_mini_layer_serial(cuda_ok):
    _run("mini", layer_serial=True, steps=18)


def test_engine_c1(cuda_ok):
    eng, oeng = _run("c1")
    # tree structure after the step-0 rotation (16 device inserts per tree)
    for h in range(8):
        ex = eng.forest.export(h)
        ot = oeng.heads[(0, h)].tree.export()
        assert [tuple(n[:4]) + (n[4],) for n in ex["nodes"]] == \
            [(i, lv, par, own, mem) for i, lv, par, own, mem, _ in ot["nodes"]]


def test_cuda_graph_replay_matches_eager(cuda_ok):
    """Captured decode steps (both variants: plain and rotating) replay to the
    same outputs and selections as eager steps, bit for bit."""
    import torch
    from paper_2604_10539_b200.engine import Engine, EngineConfig
    from oracle.workload import Spec, generate
    sk = dict(n_tokens=2048 + 60, d=64, d_prime=64, clusters=16, layers=4, kv_heads=2,
              query_heads_per_group=4, seed=9)
    keys, values, queries, _ = generate(Spec(kind="clustered", **sk))
    shape = dict(layers=4, kv_heads=2, query_heads_per_group=4, d=64, d_prime=64, seed=9)
    cfg = dict(token_budget=32, skip_layers=1, kv_dtype="bf16", max_tokens=2048 + 60)
    eager = Engine(EngineConfig(**shape, **cfg)).prefill(keys, values, 2048)
    graph = Engine(EngineConfig(**shape, **cfg, cuda_graph=True)).prefill(keys, values, 2048)
    q = torch.as_tensor(queries, device="cuda")
    k = torch.as_tensor(keys, device="cuda")
    v = torch.as_tensor(values, device="cuda")
    for t in range(50):
        tok = 2048 + t
        o1, _ = eager.decode_step(tok, q[tok], k[tok], v[tok], metrics=False)
        o2, _ = graph.decode_step(tok, q[tok], k[tok], v[tok], metrics=False)
        assert torch.equal(o1, o2), t
        (i1, c1, p1, n1), (i2, c2, p2, n2) = eager.selected(), graph.selected()
        assert (c1 == c2).all() and (n1 == n2).all(), t
        for tr in range(c1.shape[0]):
            assert list(p1[tr, :n1[tr]]) == list(p2[tr, :n2[tr]]), t
            for g in range(c1.shape[1]):
                assert list(i1[tr, g, :c1[tr, g]]) == list(i2[tr, g, :c2[tr, g]]), t
    assert set(graph._graphs) == {False, True}   # both variants captured and replayed


def test_fused_rotation_step_matches_separate_launches(cuda_ok):
    """icb_step_attend (rotation + window append + search + attention in one
    CTA per tree) gives the outputs, selections, step metrics and final tree
    structure of the separate rotate / append / query_attend launches."""
    import torch
    from paper_2604_10539_b200.engine import Engine, EngineConfig
    from oracle.workload import Spec, generate
    sk = dict(n_tokens=2048 + 70, d=64, d_prime=64, clusters=16, layers=4, kv_heads=2,
              query_heads_per_group=4, seed=5)
    keys, values, queries, _ = generate(Spec(kind="clustered", **sk))
    shape = dict(layers=4, kv_heads=2, query_heads_per_group=4, d=64, d_prime=64, seed=5)
    cfg = dict(token_budget=32, skip_layers=1, kv_dtype="bf16", max_tokens=2048 + 70)
    sep = Engine(EngineConfig(**shape, **cfg, fuse_rotation=False)).prefill(keys, values, 2048)
    fus = Engine(EngineConfig(**shape, **cfg, fuse_rotation=True)).prefill(keys, values, 2048)
    q = torch.as_tensor(queries, device="cuda")
    k = torch.as_tensor(keys, device="cuda")
    v = torch.as_tensor(values, device="cuda")
    for t in range(64):
        tok = 2048 + t
        o1, m1 = sep.decode_step(tok, q[tok], k[tok], v[tok])
        o2, m2 = fus.decode_step(tok, q[tok], k[tok], v[tok])
        assert torch.equal(o1, o2), t
        assert m1 == m2, t
        (i1, c1, p1, n1), (i2, c2, p2, n2) = sep.selected(), fus.selected()
        assert (c1 == c2).all() and (n1 == n2).all(), t
        for tr in range(c1.shape[0]):
            assert list(p1[tr, :n1[tr]]) == list(p2[tr, :n2[tr]]), t
    for tr in range(sep.T):
        e1, e2 = sep.forest.export(tr), fus.forest.export(tr)
        assert e1["nodes"] == e2["nodes"] and e1["pages"] == e2["pages"], tr
        assert e1["info"] == e2["info"], tr


@pytest.mark.parametrize("name", ["eval", "eval_reuse", "baseline"])
def test_engine_evaluation_metrics(cuda_ok, name):
    """evaluate=True (engine.py:536-566) on the device: recall@k, page hit rate,
    covered attention mass and relative error against the reference's golden
    step metrics (set metrics exact up to fp64 near-ties; mass / error within
    fp32-output tolerance)."""
    from paper_2604_10539_b200.engine import Engine, EngineConfig
    z, meta = load_golden(f"engine_{name}.npz")
    sk, ck = meta["spec"], meta["cfg"]
    keys, values, queries, _ = generate(Spec(kind="clustered", **sk))
    shape = dict(layers=sk["layers"], kv_heads=sk["kv_heads"], query_heads_per_group=sk["query_heads_per_group"],
                 d=sk["d"], d_prime=sk["d_prime"], seed=sk["seed"])
    n0 = meta["n_prefill"]
    eng = Engine(EngineConfig(**shape, **ck, kv_dtype="fp32", max_tokens=n0 + meta["steps"] + 1)).prefill(
        keys, values, n0)
    k = ck["token_budget"]
    sem, base = [], []
    for t in range(meta["steps"]):
        tok = n0 + t
        out, m = eng.decode_step(tok, queries[tok], keys[tok], values[tok])
        row = meta["rows"][t]
        for key in KEYS:
            assert getattr(m, key) == row[key], (t, key)
        # recall: every layer (anchors too under reuse) scores the same token sets as the reference
        assert abs(m.recall_at_k - row["recall_at_k"]) <= 1e-9, (t, m.recall_at_k, row["recall_at_k"])
        assert abs(m.page_hit_rate - row["page_hit_rate"]) <= 1.0 / k + 1e-9, (t, m.page_hit_rate)
        assert abs(m.covered_attention_mass - row["covered_attention_mass"]) < 1e-6, t
        assert abs(m.approx_rel_error - row["approx_rel_error"]) < 1e-4 * max(1.0, row["approx_rel_error"]), t
        if row.get("baseline_hit_rate") is not None:
            # TokenOrderBaseline (engine.py:148-182) on the device: same pages, same hits
            assert abs(m.baseline_hit_rate - row["baseline_hit_rate"]) <= 1e-9, (t, m.baseline_hit_rate)
            sem.append(m.page_hit_rate)
            base.append(m.baseline_hit_rate)
        else:
            assert m.baseline_hit_rate is None
        ref = z["outputs"][t]
        o = out.cpu().numpy()
        assert (np.linalg.norm(o - ref, axis=-1) / np.linalg.norm(ref, axis=-1)).max() < 1e-3
    if sem:
        # acceptance 06 (tests/test_acceptance.py:135-153): semantic paging hits at least as often
        assert np.mean(sem) >= np.mean(base)


@pytest.mark.parametrize("kv,reuse", [("bf16", 0), ("fp32", 0), ("bf16", 3)])
def test_kv_offload_matches_resident(cuda_ok, kv, reuse):
    """BASELINE config 3: page K/V in pinned host memory, each step's sink,
    window and selected pages gathered into the HBM pool (TierStore backload /
    evict, pagestore.py:169-215).  Outputs, selections and step metrics equal
    the all-resident engine bit for bit; the pool holds exactly the last step's
    pages; the gathered bytes cover the reference's backload."""
    import torch
    from paper_2604_10539_b200.engine import Engine, EngineConfig
    from oracle.workload import Spec, generate
    sk = dict(n_tokens=2048 + 70, d=64, d_prime=64, clusters=16, layers=4, kv_heads=2,
              query_heads_per_group=4, seed=3)
    keys, values, queries, _ = generate(Spec(kind="clustered", **sk))
    shape = dict(layers=4, kv_heads=2, query_heads_per_group=4, d=64, d_prime=64, seed=3)
    cfg = dict(token_budget=32, skip_layers=1, kv_dtype=kv, max_tokens=2048 + 70, reuse_stride=reuse)
    res = Engine(EngineConfig(**shape, **cfg)).prefill(keys, values, 2048)
    off = Engine(EngineConfig(**shape, **cfg, kv_offload=True)).prefill(keys, values, 2048)
    assert off.forest.kv_host and not res.forest.kv_host
    q = torch.as_tensor(queries, device="cuda")
    k = torch.as_tensor(keys, device="cuda")
    v = torch.as_tensor(values, device="cuda")
    moved = 0
    for t in range(64):
        tok = 2048 + t
        o1, m1 = res.decode_step(tok, q[tok], k[tok], v[tok])
        o2, m2 = off.decode_step(tok, q[tok], k[tok], v[tok])
        assert torch.equal(o1, o2), t
        assert m1 == m2, t
        moved += m2.bytes_moved
        (i1, c1, p1, n1), (i2, c2, p2, n2) = res.selected(), off.selected()
        assert (n1 == n2).all(), t
        if not reuse:   # reuse layers run no query: their id rows are not written
            assert (c1 == c2).all(), t
        for tr in range(n1.shape[0]):
            assert list(p1[tr, :n1[tr]]) == list(p2[tr, :n2[tr]]), t
    if reuse:
        return   # reuse layers attend through icb_sparse_attention, which reads the host store in place
    ps = off.forest.pool_stats()
    n_sel = np.asarray(n2)
    fixed = off.cfg.sink_pages + off.cfg.window_pages
    assert (ps[:, 1] == n_sel + fixed).all()
    assert ps[:, 0].sum() > 0


def test_layer_streaming_prefill_matches_batched(cuda_ok):
    """Engine.prefill_layers (each layer's trees built on the engine's stream as
    its K/V arrive) builds the same trees as prefill(keys, values, n): equal
    exports, bit-identical decode outputs and selections."""
    import torch
    from paper_2604_10539_b200.engine import Engine, EngineConfig
    sk = dict(n_tokens=2048 + 40, d=64, d_prime=32, clusters=16, layers=5, kv_heads=2, query_heads_per_group=2,
              seed=21)
    keys, values, queries, _ = generate(Spec(kind="clustered", **sk))
    shape = dict(layers=5, kv_heads=2, query_heads_per_group=2, d=64, d_prime=32, seed=21)
    cfg = dict(token_budget=32, skip_layers=2, kv_dtype="bf16", max_tokens=2048 + 40)
    a = Engine(EngineConfig(**shape, **cfg)).prefill(keys, values, 2048)
    b = Engine(EngineConfig(**shape, **cfg))
    k = torch.as_tensor(keys, dtype=torch.float32, device="cuda")
    v = torch.as_tensor(values, dtype=torch.float32, device="cuda")
    pf = b.prefill_layers(2048)
    for layer in range(5):
        pf.layer(layer, k[:, layer] * 1.0, v[:, layer] * 1.0)   # fresh tensors, as a model would hand over
    pf.finish()
    for tr in range(a.T):
        ea, eb = a.forest.export(tr), b.forest.export(tr)
        assert ea["nodes"] == eb["nodes"] and ea["pages"] == eb["pages"], tr
    for t in range(40):
        tok = 2048 + t
        oa, _ = a.decode_step(tok, queries[tok], keys[tok], values[tok])
        ob, _ = b.decode_step(tok, queries[tok], keys[tok], values[tok])
        assert torch.equal(oa, ob), t


def test_engine_on_llama_qkv_matches_reference(cuda_ok):
    """q/k/v from a Llama forward (tools/llama_trace.py: transformers'
    LlamaForCausalLM, random init, post-RoPE q/k/v captured by an attention
    hook, stored in the reference's ICET trace format): the device engine
    against the oracle (ranked lists and pages bit-exact) and the reference's
    own run on the same trace (step metrics, evaluation metrics, outputs)."""
    import os
    from paper_2604_10539_b200.engine import Engine, EngineConfig
    from paper_2604_10539_b200.trace import load_trace
    z, meta = load_golden("engine_llama.npz")
    tr = load_trace(os.path.join(os.path.dirname(__file__), "golden", meta["trace"]))
    keys, values, queries = (tr.keys.astype(np.float64), tr.values.astype(np.float64), tr.queries.astype(np.float64))
    shape = dict(layers=tr.layers, kv_heads=tr.kv_heads, query_heads_per_group=tr.query_heads_per_group, d=tr.d,
                 d_prime=tr.d_prime)
    ck = meta["cfg"]
    n0 = meta["n_prefill"]
    oeng = OracleEngine(OConfig(**shape, token_budget=ck["token_budget"], skip_layers=ck["skip_layers"],
                                seed=ck["seed"])).prefill(keys, values, n0)
    eng = Engine(EngineConfig(**shape, **ck, kv_dtype="fp32", max_tokens=tr.n_tokens)).prefill(keys, values, n0)
    G, H = tr.query_heads_per_group, tr.kv_heads
    for t in range(meta["steps"]):
        tok = n0 + t
        oout, om, trace = oeng.decode_step(tok, queries[tok], keys[tok], values[tok])
        out, m = eng.decode_step(tok, queries[tok], keys[tok], values[tok])
        row = meta["rows"][t]
        for k in KEYS:
            assert getattr(m, k) == om[k] == row[k], (t, k)
        assert abs(m.recall_at_k - row["recall_at_k"]) <= 1e-9, t
        assert abs(m.page_hit_rate - row["page_hit_rate"]) <= 1e-9, t
        assert abs(m.covered_attention_mass - row["covered_attention_mass"]) < 1e-6, t
        ids, counts, pages, npages = eng.selected()
        for layer in range(ck["skip_layers"], tr.layers):
            for h in range(H):
                trx = (layer - ck["skip_layers"]) * H + h
                for g in range(G):
                    assert list(ids[trx, g, :counts[trx, g]]) == trace["tokens"][(layer, h * G + g)], (t, layer, h, g)
                assert list(pages[trx, :npages[trx]]) == trace["pages"][(layer, h)], (t, layer, h)
        ref = z["outputs"][t]
        o = out.cpu().numpy()
        assert (np.linalg.norm(o - ref, axis=-1) / np.linalg.norm(ref, axis=-1)).max() < 1e-3, t
