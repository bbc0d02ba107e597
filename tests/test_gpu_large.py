"""Parity at the sizes the bench reports, against golden vectors made by the
UNMODIFIED reference (tests/golden/make_golden_large.py):

* one C2 tree (32,720 points, d = 128) and one C3 tree (131,024 points: the
  device's exact-parent build path above 98,304 points): structure and pages
  identical, ranked top-256 lists identical up to documented fp32/fp64
  near-ties, distance-eval counters identical, 16 inserts (levels,
  structure), queries after the inserts; the 32k tree also bit-exact against
  the fp32 oracle;
* the C2-shaped engine (2 dense skip layers + 1 indexed layer of 8 kv heads,
  G = 4, d = 128, 32k prefill) for seeds 0-4, 16 decode steps each (two
  rotations): every step metric, every query head's token set, outputs;
* the C5-shaped long generation (8k prompt, 2 kv heads, G = 4, d = 128):
  2,048 decode steps = 128 rotations x 16 device inserts per tree, every
  step's metrics and every head's token-set digest, full ranked lists every
  16th step.

Inputs are regenerated from the recorded WorkloadSpec with the package's
NumPy generator (bit-identical to the reference's; tests/test_workload_cpu.py)
and rounded to fp32, as the goldens' were.  Near-ties: a ranked list may
differ from the reference's only between ids whose fp64 lifted distances are
within NEAR of each other (the device ranks fp32 distances, the reference
fp64), and a step whose token sets differ that way is exempt from
the exact metric comparison.
"""

import zlib

import numpy as np
import pytest

from conftest import load_golden

pytestmark = pytest.mark.gpu

NEAR = 2e-6
ROW_FIELDS = ["pages_selected", "pages_loaded", "tokens_loaded", "bytes_moved", "transactions", "dci_queries"]


def f32(x):
    return np.asarray(x, dtype=np.float64).astype(np.float32).astype(np.float64)


def workload(spec):
    from paper_2604_10539_b200 import WorkloadSpec, generate_workload
    wl = generate_workload(WorkloadSpec(kind="clustered", **spec))
    for a in (wl.keys, wl.values, wl.queries):
        a[:] = f32(a)
    return wl


def lift64(keys, c):
    n = np.linalg.norm(keys, axis=-1)
    out = np.empty(keys.shape[:-1] + (keys.shape[-1] + 1,))
    safe = np.where(n > c, n, c)
    out[..., :-1] = keys / safe[..., None]
    out[..., -1] = np.sqrt(np.maximum(0.0, 1.0 - (n / safe) ** 2))
    return out


def ranked_ok(got, want, d2):
    """got == want, or they differ only between near-tied fp64 distances."""
    if list(got) == list(want):
        return True
    if len(got) != len(want):
        return False
    bound = max(d2(p) for p in want)
    if any(abs(d2(p) - bound) > NEAR for p in set(got) ^ set(want)):
        return False
    return all(a == b or abs(d2(a) - d2(b)) <= NEAR for a, b in zip(got, want))


def digest(tokens):
    return zlib.crc32(np.asarray(sorted(int(t) for t in tokens), dtype="<i4").tobytes())


# ----------------------------------------------------------------------------- trees
def _tree_case(name):
    from paper_2604_10539_b200 import TierStore, dci_indexing
    from paper_2604_10539_b200.pagestore import SINK, WINDOW
    z, meta = load_golden(f"{name}.npz")
    wl = workload(meta["spec"])
    layer, h = meta["layer"], meta["h"]
    idx = list(range(meta["sink_end"], meta["win_start"]))
    store = TierStore(128, 128)
    store.allocate_page(16, SINK, resident=True, pinned=True)
    store.allocate_page(16, WINDOW, resident=True, pinned=True)
    store.allocate_page(16, WINDOW, resident=True, pinned=True)
    tree = dci_indexing([(t, wl.keys[t, layer, h]) for t in idx], meta["r"], seed=tuple(meta["seed"]),
                        values=[wl.values[t, layer, h] for t in idx], store=store, page_size=meta["page_size"])
    return z, meta, wl, tree, store


def _check_struct(z, pre, tree, store):
    nodes = tree.nodes
    assert sorted(nodes) == list(range(len(z[f"{pre}node_level"])))
    assert [nodes[i].level for i in sorted(nodes)] == z[f"{pre}node_level"].tolist()
    assert [-1 if nodes[i].parent_id is None else nodes[i].parent_id for i in sorted(nodes)] == \
        z[f"{pre}node_parent"].tolist()
    assert [nodes[i].owner_id for i in sorted(nodes)] == z[f"{pre}node_owner"].tolist()
    assert [len(nodes[i].member_ids) for i in sorted(nodes)] == z[f"{pre}node_msize"].tolist()
    assert np.array_equal(np.concatenate([np.asarray(nodes[i].member_ids, np.int32) for i in sorted(nodes)]),
                          z[f"{pre}node_members"])
    pl = tree.point_level
    assert np.array_equal(np.array([[p, pl[p]] for p in sorted(pl)], np.int32), z[f"{pre}point_level"])
    pids = sorted(store.pages)
    assert pids == z[f"{pre}page_id"].tolist()
    assert [store.pages[p].fill for p in pids] == z[f"{pre}page_fill"].tolist()
    assert np.array_equal(np.concatenate([np.asarray(store.pages[p].token_ids, np.int32) for p in pids]),
                          z[f"{pre}page_tok"])


@pytest.mark.parametrize("name", ["tree_c2_32k", "tree_c3_128k"])
def test_tree_build_queries_inserts_vs_reference(cuda_ok, name):
    from paper_2604_10539_b200 import SENTINEL_LEVEL, SearchBudget, transform_query
    z, meta, wl, tree, store = _tree_case(name)
    layer, h = meta["layer"], meta["h"]
    assert tree.scale.c == meta["scale"] and tree.levels == meta["levels"]
    _check_struct(z, "b_", tree, store)
    c = tree.scale.c
    lifted = lift64(wl.keys[:, layer, h], c)
    budget = SearchBudget.for_k(meta["k"])
    flips = 0
    for i, (tk, qh) in enumerate(zip(meta["query_tokens"], meta["query_heads"])):
        q = wl.queries[tk, layer, qh]
        ql = transform_query(q)
        e0 = tree.distance_evals
        got = tree.query(ql, SENTINEL_LEVEL, meta["k"], budget)
        want = [int(x) for x in z["topk"][i]]
        d2 = lambda p: float(((lifted[p] - ql) ** 2).sum())   # noqa: E731
        assert ranked_ok(got, want, d2), (i, [(a, b) for a, b in zip(got, want) if a != b][:4])
        flips += got != want
        if set(got) == set(want):
            assert tree.distance_evals - e0 == meta["evals"][i], i
    levels = [tree.insert(t, wl.keys[t, layer, h], wl.values[t, layer, h]) for t in meta["insert_tokens"]]
    assert levels == meta["insert_levels"]
    tree.check_invariants()
    _check_struct(z, "a_", tree, store)
    for i, (tk, qh) in enumerate(zip(meta["query_tokens"][:16], meta["query_heads"][:16])):
        ql = transform_query(wl.queries[tk, layer, qh])
        got = tree.query(ql, SENTINEL_LEVEL, meta["k"], budget)
        d2 = lambda p: float(((lift64(wl.keys[p, layer, h], c) - ql) ** 2).sum())   # noqa: E731
        assert ranked_ok(got, [int(x) for x in z["topk_after"][i]], d2), i
    print(f"{name}: {flips} near-tie order flips in {len(meta['query_tokens'])} queries")


def test_tree_32k_bit_exact_vs_oracle(cuda_ok):
    """Device vs the fp32 restatement: every ranked list and eval count equal."""
    from oracle import numerics as nm
    from oracle.dci import SENTINEL, build
    from paper_2604_10539_b200 import SENTINEL_LEVEL, SearchBudget, transform_query
    z, meta, wl, tree, store = _tree_case("tree_c2_32k")
    layer, h = meta["layer"], meta["h"]
    idx = list(range(meta["sink_end"], meta["win_start"]))
    ot = build([(t, wl.keys[t, layer, h]) for t in idx], meta["r"], seed=tuple(meta["seed"]))
    assert ot.c == tree.scale.c
    for tk, qh in zip(meta["query_tokens"], meta["query_heads"]):
        q = wl.queries[tk, layer, qh]
        e0, o0 = tree.distance_evals, ot.distance_evals
        got = tree.query(transform_query(q), SENTINEL_LEVEL, 256, SearchBudget.for_k(256))
        want = ot.query(nm.lift_query32(q), SENTINEL, 256, 512, 1024)
        assert got == want
        assert tree.distance_evals - e0 == ot.distance_evals - o0


# ----------------------------------------------------------------------------- engines
def _engine_run(name, *, check_outputs):
    from paper_2604_10539_b200 import Engine, EngineConfig
    z, meta = load_golden(f"{name}.npz")
    sk, ck = meta["spec"], meta["cfg"]
    wl = workload(sk)
    n0, steps = meta["n_prefill"], meta["steps"]
    cfg = EngineConfig(layers=sk["layers"], kv_heads=sk["kv_heads"], query_heads_per_group=sk["query_heads_per_group"],
                       d=sk["d"], d_prime=sk["d_prime"], seed=sk["seed"], kv_dtype="fp32",
                       max_tokens=n0 + steps + 1, **ck)
    eng = Engine(cfg).prefill(wl, n0)
    H, G, s0 = cfg.kv_heads, cfg.query_heads_per_group, cfg.skip_layers
    calls = meta["calls"]
    full_at = {t: i for i, t in enumerate(meta["full_steps"])}
    lifted = {}
    flips = exempt = 0
    for t in range(steps):
        tok = n0 + t
        out, m = eng.decode_step(tok, wl.queries[tok], wl.keys[tok], wl.values[tok])
        ids, counts, _, _ = eng.selected()
        differs = False
        for i, (layer, h) in enumerate(calls):
            g = i % G
            tr = (layer - s0) * H + h
            got = [int(x) for x in ids[tr, g, :counts[tr, g]]]
            if digest(got) == int(z["digests"][t, i]) and t not in full_at:
                continue
            if tr not in lifted or t in full_at or digest(got) != int(z["digests"][t, i]):
                lifted[tr] = lift64(wl.keys[: tok + 1, layer, h], eng.forest.scale(tr))
            qh = h * G + g
            from paper_2604_10539_b200 import transform_query
            ql = transform_query(wl.queries[tok, layer, qh])
            d2 = lambda p: float(((lifted[tr][p] - ql) ** 2).sum())   # noqa: E731
            if t in full_at:
                want = [int(x) for x in z["tokens"][full_at[t], i] if x >= 0]
                assert ranked_ok(got, want, d2), (t, layer, h, g)
                flips += got != want
                differs |= set(got) != set(want)
            else:
                # only the set digest is recorded: the set must be the reference's
                # up to a near-tie at the k-th boundary, which we cannot name here
                # without the list; require the k-th distance to sit within NEAR of
                # the (k+1)-th candidate's
                kth = max(d2(p) for p in got)
                others = [d2(p) for p in range(tok + 1) if p not in set(got) and p in eng_indexed(eng, tr)]
                assert others and min(others) - kth <= NEAR, (t, layer, h, g)
                differs = True
        row = [getattr(m, k) for k in ROW_FIELDS]
        if differs:
            exempt += 1
        else:
            assert row == z["rows"][t].tolist(), (t, row, z["rows"][t].tolist())
        if check_outputs:
            ref = z["outputs"][t].astype(np.float64)
            o = out.cpu().numpy()
            err = np.linalg.norm(o - ref, axis=-1) / np.linalg.norm(ref, axis=-1)
            assert err.max() < (1e-3 if not differs else 5e-2), (t, err.max())
    print(f"{name}: {flips} near-tie order flips, {exempt} steps with near-tie set differences")
    assert exempt <= max(1, steps // 50)
    return eng


_INDEXED = {}


def eng_indexed(eng, tr):
    key = (id(eng), tr, eng.steps_done)
    if key not in _INDEXED:
        _INDEXED.clear()
        _INDEXED[key] = set(eng.forest.export(tr)["point_level"])
    return _INDEXED[key]


@pytest.mark.parametrize("seed", range(5))
def test_engine_c2_shape_vs_reference(cuda_ok, seed):
    _engine_run(f"engine_c2_s{seed}", check_outputs=(seed == 0))


def test_engine_c5_long_generation_vs_reference(cuda_ok):
    eng = _engine_run("engine_c5", check_outputs=False)
    from paper_2604_10539_b200.dci import DciTree
    f = eng.forest
    f.check()
    for tr in range(eng.T):
        # 8,144 prefill points + 129 rotations x 16 inserts
        assert f.info(tr)["n_points"] == len(eng.indexed_tokens) == 8144 + 129 * 16
        DciTree.bound(f, tr, f.scale(tr), 0.1, 16, f.caps.tok_cap).check_invariants()
