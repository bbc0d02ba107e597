"""The device Engine through the reference's own call shapes:
prefill(Workload, n) and decode_step(DecodeStep) -> (outputs[layer][query
head] AttentionOutput, StepMetrics), page_select, select_with_reuse, the
per-(layer, kv head) `heads` view and the module-level prefill -- the
behaviours the reference's tests/test_engine.py and acceptance test 03 pin,
restated, plus the AttentionOutput weights checked against an fp64 softmax
over the attended tokens in entry order."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def f32(x):
    return np.asarray(x, dtype=np.float64).astype(np.float32).astype(np.float64)


def small(seed=0, n_tokens=600, layers=3, kv_heads=2, d=16, d_prime=8, G=1, round32=False, **cfg):
    from paper_2604_10539_b200 import EngineConfig, WorkloadSpec, generate_workload
    wl = generate_workload(WorkloadSpec(kind="clustered", n_tokens=n_tokens, d=d, d_prime=d_prime, clusters=8,
                                        layers=layers, kv_heads=kv_heads, query_heads_per_group=G, seed=seed))
    if round32:
        for a in (wl.keys, wl.values, wl.queries):
            a[:] = f32(a)
    return wl, EngineConfig(layers=layers, kv_heads=kv_heads, d=d, d_prime=d_prime, query_heads_per_group=G,
                            seed=seed, max_tokens=n_tokens, **cfg)


def test_prefill_layout_and_heads_view(cuda_ok):
    from paper_2604_10539_b200 import Engine
    from paper_2604_10539_b200.pagestore import INDEXED, SINK, WINDOW
    wl, cfg = small(token_budget=16)
    eng = Engine(cfg).prefill(wl, 500)
    heads = eng.heads
    assert (0, 0) not in heads and (1, 0) not in heads and (2, 0) in heads and (2, 1) in heads
    st = heads[(2, 0)]
    assert [p.role for p in st.sink] == [SINK] * cfg.sink_pages
    assert all(p.role == WINDOW for p in st.window)
    indexed = sorted(t for p in st.store.pages.values() if p.role == INDEXED for t in p.token_ids)
    assert indexed == eng.indexed_tokens
    assert len(st.tree) == len(eng.indexed_tokens)
    assert eng.sink_tokens == list(range(cfg.sink_pages * cfg.page_size))
    assert eng.token_census(2, 0) == 500


def test_short_prompt_falls_back_to_dense(cuda_ok):
    from paper_2604_10539_b200 import Engine, full_attention
    wl, cfg = small(token_budget=16, evaluate=True, round32=True)
    eng = Engine(cfg).prefill(wl, 40)
    assert eng.fallback and not eng.heads
    outs, m = eng.decode_step(wl.decode_step(40, 0))
    ref = full_attention(wl.queries[40, 2, 0], wl.keys[:41, 2, 0], wl.values[:41, 2, 0])
    # value_out: fp32 accumulation (north-star 1e-3); weights: fp64 logits of the stored (fp32) keys
    assert np.linalg.norm(outs[2][0].value_out - ref.value_out) / np.linalg.norm(ref.value_out) < 1e-5
    assert list(outs[2][0].weights) == list(range(41))
    assert max(abs(outs[2][0].weights[t] - ref.weights[t]) for t in range(41)) < 1e-12
    assert m.approx_rel_error == 0.0


def test_rotation_cadence_and_offload_counter(cuda_ok):
    from paper_2604_10539_b200 import Engine
    wl, cfg = small(n_tokens=700, token_budget=8)
    n0, s = 512, cfg.page_size
    eng = Engine(cfg).prefill(wl, n0)
    size0 = len(eng.heads[(2, 0)].tree)
    eng.decode_step(wl.decode_step(n0, 0))                 # full newest window page: rotates now
    assert eng.heads[(2, 0)].store.stats.pages_offloaded == 1
    assert len(eng.heads[(2, 0)].tree) == size0 + s
    steps = 0
    for t in range(1, 2 * s):
        eng.decode_step(wl.decode_step(n0, t))
        steps += 1
        if eng.heads[(2, 0)].store.stats.pages_offloaded > 1:
            break
    assert steps == s - 1 and len(eng.heads[(2, 0)].tree) == size0 + 2 * s


def test_unlimited_budget_attends_every_token(cuda_ok):
    from paper_2604_10539_b200 import Engine
    wl, cfg = small(n_tokens=700, token_budget=10**6, beam=2**61, visit_cap=2**61)
    eng = Engine(cfg).prefill(wl, 512)
    outs, _ = eng.decode_step(wl.decode_step(512, 0))     # the rotation step
    assert set(outs[2][0].weights) == set(range(513))


def test_token_census_after_steps(cuda_ok):
    from paper_2604_10539_b200 import Engine
    wl, cfg = small(n_tokens=700)
    eng = Engine(cfg).prefill(wl, 512)
    for t in range(40):
        eng.decode_step(wl.decode_step(512, t))
    assert all(eng.token_census(layer, h) == 552 for layer, h in eng.heads)


def test_repeated_query_reloads_nothing(cuda_ok):
    from paper_2604_10539_b200 import Engine
    wl, cfg = small(n_tokens=700, token_budget=16)
    wl.queries[521] = wl.queries[520]
    eng = Engine(cfg).prefill(wl, 520)
    _, a = eng.decode_step(wl.decode_step(520, 0))
    _, b = eng.decode_step(wl.decode_step(520, 1))
    assert a.pages_loaded > 0 and (b.pages_loaded, b.transactions) == (0, 0)
    st = eng.heads[(2, 0)].store.stats
    assert st.pages_backloaded > 0 and st.pages_filtered_resident > 0


def test_stream_checks(cuda_ok):
    from paper_2604_10539_b200 import ConfigError, Engine, EngineConfig, InputError
    wl, cfg = small()
    eng = Engine(cfg)
    with pytest.raises(ConfigError):
        eng.decode_step(wl.decode_step(500, 0))
    with pytest.raises(ConfigError):
        Engine(cfg).prefill(wl, 0)
    with pytest.raises(ConfigError):
        Engine(EngineConfig(layers=3, kv_heads=2, d=8, d_prime=8)).prefill(wl, 100)
    eng.prefill(wl, 500)
    with pytest.raises(ConfigError):
        eng.prefill(wl, 500)
    with pytest.raises(InputError):
        eng.decode_step(wl.decode_step(500, 3))


def test_group_heads_share_one_union(cuda_ok):
    from paper_2604_10539_b200 import Engine
    wl, cfg = small(G=2, token_budget=8)
    eng = Engine(cfg).prefill(wl, 500)
    step = wl.decode_step(500, 0)
    pa = set(eng.page_select(step.queries[2, 0], 2, 0))
    pb = set(eng.page_select(step.queries[2, 1], 2, 0))
    outs, _ = eng.decode_step(step)
    attended = set(outs[2][0].weights)
    assert set(eng.heads[(2, 0)].store.tokens_in(sorted(pa | pb))) <= attended
    assert set(outs[2][1].weights) == attended


def test_page_select_bound_and_skipped_layer(cuda_ok):
    from paper_2604_10539_b200 import ConfigError, Engine
    wl, cfg = small(token_budget=12)
    eng = Engine(cfg).prefill(wl, 500)
    pages = eng.page_select(wl.queries[500, 2, 0], 2, 0)
    assert 0 < len(pages) <= 12 and pages == sorted(set(pages))
    with pytest.raises(ConfigError):
        eng.page_select(wl.queries[500, 2, 0], 0, 0)


def test_selection_reuse_api(cuda_ok):
    from paper_2604_10539_b200 import ConfigError, Engine
    wl, cfg = small(layers=8, kv_heads=1, reuse_stride=2, token_budget=8)
    assert Engine(cfg).prefill(wl, 500).anchor_layers() == [2, 4, 6]
    wl, cfg = small(token_budget=8)
    eng = Engine(cfg).prefill(wl, 500)
    with pytest.raises(ConfigError):
        eng.select_with_reuse(2, wl.queries[500, 2])
    with pytest.raises(ConfigError):
        eng.is_anchor_layer(2)
    wl, van = small(seed=12, layers=5, kv_heads=1, token_budget=16)
    wl2, reu = small(seed=12, layers=5, kv_heads=1, token_budget=16, reuse_stride=3)
    vanilla, reused = Engine(van).prefill(wl, 500), Engine(reu).prefill(wl2, 500)
    step = wl.decode_step(500, 0)
    pages_by_head, toks = reused.select_with_reuse(2, step.queries[2])
    assert pages_by_head[0] == vanilla.page_select(step.queries[2, 0], 2, 0)
    p3, t3 = reused.select_with_reuse(3, step.queries[3])      # reuse layer: the anchor's tokens
    assert t3[0] == toks[0]
    wl, cfg = small(layers=8, kv_heads=1, reuse_stride=3, token_budget=8)
    eng = Engine(cfg).prefill(wl, 500)
    assert eng.decode_step(wl.decode_step(500, 0))[1].dci_queries == 2


def test_module_prefill(cuda_ok):
    from paper_2604_10539_b200 import prefill
    wl, cfg = small()
    eng = prefill(wl, cfg, 500)
    assert eng.prefilled and eng.n_prefill == 500


def test_step_weights_are_the_softmax_over_the_attended_set(cuda_ok):
    """Every indexed head's weights: keys = sink, window and selected-page
    tokens in entry order; values = the fp64 softmax of k.q / sqrt(d) over
    exactly those tokens (fp32-representable inputs: exact up to summation
    order).  value_out within the fp32 tolerance of that softmax's output."""
    from paper_2604_10539_b200 import Engine
    wl, cfg = small(seed=4, n_tokens=800, layers=4, kv_heads=2, G=2, d=32, d_prime=16, token_budget=24,
                    round32=True)
    eng = Engine(cfg).prefill(wl, 700)
    for t in range(20):
        step = wl.decode_step(700, t)
        outs, _ = eng.decode_step(step)
        ids, counts, pages, npages = eng.selected()
        for layer in range(cfg.skip_layers, cfg.layers):
            for h in range(cfg.kv_heads):
                tr = (layer - cfg.skip_layers) * cfg.kv_heads + h
                ex = eng.forest.export(tr)
                order = ex["sink"] + ex["win"] + [int(p) for p in pages[tr, :npages[tr]]]
                toks = [tok for p in order for tok in ex["pages"][p][1]]
                keys = wl.keys[toks, layer, h]
                vals = wl.values[toks, layer, h]
                for g in range(cfg.query_heads_per_group):
                    qh = h * cfg.query_heads_per_group + g
                    q = step.queries[layer, qh]
                    lg = keys @ q / np.sqrt(q.size)
                    w = np.exp(lg - lg.max())
                    w /= w.sum()
                    o = outs[layer][qh]
                    assert list(o.weights) == toks
                    assert np.abs(np.array(list(o.weights.values())) - w).max() < 1e-12
                    ref = w @ vals
                    assert np.linalg.norm(o.value_out - ref) / np.linalg.norm(ref) < 1e-5


@pytest.mark.parametrize("seed", range(20))
def test_planted_needle_is_selected_and_weighted_highest(cuda_ok, seed):
    """Acceptance 03 (reference tests/test_acceptance.py:70-90), per seed."""
    from paper_2604_10539_b200 import Engine, EngineConfig, WorkloadSpec, generate_workload
    wl = generate_workload(WorkloadSpec(kind="planted_needle", n_tokens=10_001, d=32, d_prime=8,
                                        cluster_spread=4.0, needle_gain=2.0, layers=3, kv_heads=1, seed=seed))
    eng = Engine(EngineConfig(layers=3, kv_heads=1, d=32, d_prime=8, token_budget=64, seed=seed,
                              max_tokens=10_001)).prefill(wl, 10_000)
    pages = eng.page_select(wl.queries[10_000, 2, 0], 2, 0)
    from paper_2604_10539_b200 import find_page_index
    assert find_page_index([wl.needle_token], eng.heads[(2, 0)].table)[0] in pages
    outs, _ = eng.decode_step(wl.decode_step(10_000, 0))
    w = outs[2][0].weights
    assert max(w.items(), key=lambda kv: kv[1])[0] == wl.needle_token
