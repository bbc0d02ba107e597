"""The reference's DCI-tree tests (tests/test_dci.py) re-run against the
device-backed drop-in API (paper_2604_10539_b200.dci), plus structure parity
of dci_indexing / insert against the oracle."""

import numpy as np
import pytest

from oracle.dci import build as obuild

pytestmark = pytest.mark.gpu


def _api():
    from paper_2604_10539_b200 import dci
    return dci


def _pairs(keys):
    return [(i, k) for i, k in enumerate(keys)]


def _clustered(seed, n, d, clusters, spread=0.1):
    rng = np.random.default_rng(seed)
    centers = rng.normal(size=(clusters, d))
    centers /= np.linalg.norm(centers, axis=1, keepdims=True)
    labels = rng.integers(0, clusters, size=n)
    keys = centers[labels] + rng.normal(size=(n, d)) * spread / np.sqrt(d)
    return keys, labels, centers


def _exact_topk(q, keys, k):
    s = keys @ q
    return list(np.lexsort((np.arange(len(s)), -s))[:k])


def test_single_key_builds_degenerate_tree(cuda_ok):
    D = _api()
    tree = D.dci_indexing([(7, np.ones(4))], 0.3, seed=0, values=[np.ones(4)])
    assert tree.levels == 1 and len(tree.nodes) == 1
    top = tree.nodes[tree.top_node_id]
    assert top.owner_id == D.ROOT_OWNER and top.member_ids == [7]
    assert len(top.page_ids) == 1 and tree.page_fill(top.page_ids[0]) == 1
    tree.check_invariants()


def test_duplicate_point_ids_rejected(cuda_ok):
    D = _api()
    from paper_2604_10539_b200.errors import InputError
    with pytest.raises(InputError):
        D.dci_indexing([(1, np.ones(3)), (1, np.zeros(3))], 0.1)


def test_self_retrieval_of_indexed_keys(cuda_ok):
    D = _api()
    rng = np.random.default_rng(4)
    keys = rng.normal(size=(2000, 16))
    keys /= np.linalg.norm(keys, axis=1, keepdims=True)
    tree = D.dci_indexing(_pairs(keys), 0.1, seed=4)
    budget = D.SearchBudget(1, beam=32, visit_cap=128)
    sample = rng.choice(2000, size=200, replace=False)
    hits = sum(tree.query(D.transform_query(keys[p]), D.SENTINEL_LEVEL, 1, budget)[0] == p for p in sample)
    assert hits / len(sample) >= 0.99


def test_tree_structure_matches_oracle_and_invariants(cuda_ok):
    D = _api()
    keys, _, _ = _clustered(5, 1500, 12, 8)
    tree = D.dci_indexing(_pairs(keys), 0.2, seed=5, page_size=8)
    tree.check_invariants()
    ot = obuild(_pairs(keys), 0.2, seed=5, page_size=8)
    assert tree.point_level == ot.point_level
    got = sorted((n.node_id, n.level, n.owner_id, tuple(n.member_ids)) for n in tree.nodes.values())
    want = sorted((i, lv, own, tuple(mem)) for i, lv, _, own, mem, _ in ot.export()["nodes"])
    assert got == want


def test_query_with_everything_unbounded_returns_all_ids(cuda_ok):
    D = _api()
    rng = np.random.default_rng(10)
    keys = rng.normal(size=(300, 8))
    tree = D.dci_indexing(_pairs(keys), 0.2, seed=10)
    got = tree.query(D.transform_query(rng.normal(size=8)), D.SENTINEL_LEVEL, 300, D.SearchBudget.exhaustive(300))
    assert sorted(got) == list(range(300))


def test_exhaustive_budget_query_equals_exact_topk(cuda_ok):
    D = _api()
    rng = np.random.default_rng(11)
    for trial in range(12):
        n = int(rng.integers(50, 400))
        keys = rng.normal(size=(n, 12))
        tree = D.dci_indexing(_pairs(keys), 0.15, seed=trial)
        q = rng.normal(size=12)
        got = D.query_raw(tree, q, D.SENTINEL_LEVEL, 16, D.SearchBudget.exhaustive(16))
        assert set(got) == set(_exact_topk(q, keys, 16))


def test_query_clamps_target_level_above_top(cuda_ok):
    D = _api()
    keys = np.eye(5)
    tree = D.dci_indexing(_pairs(keys), 0.2, seed=12)
    got = tree.query(D.transform_query(keys[0]), tree.levels + 5, 2, D.SearchBudget.exhaustive(2))
    assert len(got) == min(2, len(tree.nodes[tree.top_node_id].member_ids))


def test_query_counters_and_empty_tree_error(cuda_ok):
    D = _api()
    from paper_2604_10539_b200.errors import InputError
    keys = np.eye(4)
    tree = D.dci_indexing(_pairs(keys), 0.2, seed=17)
    before = tree.query_count
    tree.query(D.transform_query(keys[0]), D.SENTINEL_LEVEL, 2)
    assert tree.query_count == before + 1
    empty = D.DciTree(4, D.KeyScale(1.0), 0.2, seed=0)
    with pytest.raises(InputError):
        empty.query(D.transform_query(keys[0]), D.SENTINEL_LEVEL, 1)


def test_insert_into_empty_tree(cuda_ok):
    D = _api()
    tree = D.DciTree(3, D.KeyScale(2.0), 0.2, seed=18, page_size=4)
    tree.insert(0, np.ones(3), np.ones(3), level=1)
    assert tree.levels == 1 and len(tree.nodes) == 1
    leaf = tree.nodes[tree.top_node_id]
    assert leaf.page_ids and tree.page_fill(leaf.page_ids[0]) == 1
    tree.check_invariants()


def test_insert_overflow_opens_second_page(cuda_ok):
    D = _api()
    s = 8
    tree = D.DciTree(2, D.KeyScale(5.0), 0.2, seed=19, page_size=s)
    rng = np.random.default_rng(19)
    for i in range(s + 1):
        tree.insert(i, np.array([1.0, 0.0]) + rng.normal(size=2) * 1e-3, np.zeros(2), level=1)
    leaf = next(n for n in tree.nodes.values() if 0 in n.member_ids and n.level == 1)
    assert [tree.page_fill(p) for p in leaf.page_ids] == [s, 1]
    tree.check_invariants()


def test_insert_duplicate_id_rejected(cuda_ok):
    D = _api()
    from paper_2604_10539_b200.errors import InputError
    tree = D.DciTree(2, D.KeyScale(5.0), 0.2, seed=20)
    tree.insert(1, np.ones(2))
    with pytest.raises(InputError):
        tree.insert(1, np.zeros(2))


def test_insert_above_top_grows_tree(cuda_ok):
    D = _api()
    rng = np.random.default_rng(21)
    keys = rng.normal(size=(50, 6))
    tree = D.dci_indexing(_pairs(keys), 0.1, seed=21, capacity=256)
    old = tree.levels
    tree.insert(100, rng.normal(size=6), level=old + 2)
    assert tree.levels == old + 2
    tree.check_invariants()
    got = tree.query(D.transform_query(keys[0]), D.SENTINEL_LEVEL, 51, D.SearchBudget.exhaustive(51))
    assert sorted(got) == sorted(tree.point_level)


def test_insert_clamps_out_of_envelope_keys(cuda_ok):
    D = _api()
    tree = D.DciTree(2, D.KeyScale(1.0), 0.2, seed=22)
    tree.insert(0, np.array([5.0, 0.0]))
    assert tree.scale_clamps == 1
    assert abs(np.linalg.norm(tree.lifted(0)) - 1.0) < 1e-6


def test_incremental_inserts_match_oracle(cuda_ok):
    """DciTree grown by inserts only: same structure as the oracle's inserts."""
    D = _api()
    from oracle.dci import OracleTree
    keys, _, _ = _clustered(23, 400, 16, 8)
    sc = D.KeyScale.from_keys(keys)
    tree = D.DciTree(16, sc, 0.1, seed=23, capacity=512)
    for i, k in enumerate(keys):
        tree.insert(i, k)
    tree.check_invariants()
    ot = OracleTree(16, sc.c, 0.1, 23)
    for i, k in enumerate(keys):
        ot.insert(i, k)
    assert tree.point_level == ot.point_level
    got = sorted((n.node_id, n.level, n.owner_id, tuple(n.member_ids)) for n in tree.nodes.values())
    want = sorted((i, lv, own, tuple(mem)) for i, lv, _, own, mem, _ in ot.export()["nodes"])
    assert got == want


def test_identical_seeds_build_identical_trees(cuda_ok):
    D = _api()
    keys, _, _ = _clustered(25, 800, 16, 8)
    a = D.dci_indexing(_pairs(keys), 0.15, seed=99)
    b = D.dci_indexing(_pairs(keys), 0.15, seed=99)
    assert a.point_level == b.point_level
    assert {(n.node_id, n.level, n.owner_id, tuple(n.member_ids)) for n in a.nodes.values()} == \
        {(n.node_id, n.level, n.owner_id, tuple(n.member_ids)) for n in b.nodes.values()}


def test_pdci_query_single_member_node(cuda_ok):
    D = _api()
    tree = D.dci_indexing([(3, np.array([1.0, 2.0]))], 0.5, seed=6)
    top = tree.nodes[tree.top_node_id]
    assert tree.pdci_query(np.array([0.0, 0.0, 1.0]), top, 5) == [3]


def test_pdci_query_exhaustive_cap_matches_brute_force(cuda_ok):
    D = _api()
    rng = np.random.default_rng(7)
    keys = rng.normal(size=(256, 10))
    tree = D.dci_indexing(_pairs(keys), 1e-9, seed=7)   # one flat node
    top = tree.nodes[tree.top_node_id]
    assert len(top.member_ids) == 256
    lifted = np.stack([tree.lifted(p) for p in range(256)])
    for _ in range(10):
        tq = D.transform_query(rng.normal(size=10))
        got = tree.pdci_query(tq, top, 8, D.SearchBudget(8, 16, 256))
        d2 = ((lifted - tq) ** 2).sum(axis=1)
        want = [int(i) for i in np.lexsort((np.arange(256), d2))[:8]]
        assert got == want


def test_pdci_query_full_k_returns_all_ranked(cuda_ok):
    D = _api()
    rng = np.random.default_rng(8)
    keys = rng.normal(size=(40, 6))
    tree = D.dci_indexing(_pairs(keys), 1e-9, seed=8)
    top = tree.nodes[tree.top_node_id]
    q = D.transform_query(rng.normal(size=6))
    got = tree.pdci_query(q, top, 40)
    assert sorted(got) == list(range(40))
    d2 = [float(((tree.lifted(p) - q) ** 2).sum()) for p in got]
    assert d2 == sorted(d2)


def test_pdci_projection_path_matches_oracle_and_cap(cuda_ok):
    """P-DCI visit order (visit_cap < size): same visited set / ranking as the
    oracle's heap merge, exactly visit_cap evaluations (reference test
    test_pdci_projection_path_respects_visit_cap)."""
    D = _api()
    from oracle import numerics as nm
    rng = np.random.default_rng(9)
    keys = rng.normal(size=(500, 8))
    tree = D.dci_indexing(_pairs(keys), 1e-9, seed=9)
    top = tree.nodes[tree.top_node_id]
    assert len(top.member_ids) > D.EXHAUSTIVE_NODE_LIMIT
    ot = obuild(_pairs(keys), 1e-9, seed=9)
    q = D.transform_query(rng.normal(size=8))
    before = tree.distance_evals
    got = tree.pdci_query(q, top, 4, D.SearchBudget(4, 8, 100))
    assert tree.distance_evals - before == 100
    q32 = np.zeros(nm.DPAD, np.float32)
    q32[:8] = q[:8].astype(np.float32)    # the lifted query as the device holds it (tail 0)
    q64 = np.concatenate([q32[:8].astype(np.float64), [0.0]])
    ids, d2 = ot._candidates(ot.nodes[ot.top], q32, np.float32(0.0), q64, 100)
    want = [int(ids[i]) for i in np.lexsort((ids, d2))[:4]]
    assert got == want
