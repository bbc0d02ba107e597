"""GPU parity of the DCI forest (build / query / insert / attention) against
the CPU oracle, which is itself pinned to the reference's golden vectors.
Bit-exact for structure, ids, pages and ranked top-k; attention within the
north-star tolerance (1e-3 relative fp32, 1e-2 bf16)."""

import numpy as np
import pytest
import torch

from conftest import load_golden
from oracle import numerics as nm
from oracle.dci import SENTINEL, build as obuild
from oracle.engine import full_attention
from oracle.store import OStore

pytestmark = pytest.mark.gpu

TREES = ["clu_d16", "clu_d128", "flat_d8", "clu_d64_r3"]


def _forest(meta, extra=0, kv="fp32", n_trees=1):
    from paper_2604_10539_b200 import DeviceForest
    n = meta["n"] + extra
    return DeviceForest(n_trees, meta["d"], 4, tok_cap=n + 16, promotion_ratio=meta["r"],
                        page_size=meta["page_size"], kv_dtype=kv)


def _seed(meta):
    return meta["seed"] if isinstance(meta["seed"], int) else tuple(meta["seed"])


def _oracle(z, meta):
    n = meta["n"]
    keys = z["keys"].astype(np.float64)
    vals = z["values"].astype(np.float64)
    store = OStore(meta["d"], 4)
    tree = obuild([(i, keys[i]) for i in range(n)], meta["r"], seed=_seed(meta),
                  values=[vals[i] for i in range(n)], store=store, page_size=meta["page_size"])
    return tree, store


def _device_build(z, meta, extra):
    f = _forest(meta, extra=extra)
    n = meta["n"]
    f.seed([0], [_seed(meta)])
    f.build([0], np.arange(n)[None, :], z["keys"][:n][None], z["values"][:n][None])
    f.check()
    return f


def _compare_structure(f, otree, ostore):
    ex = f.export(0)
    oexp = otree.export()
    assert ex["info"]["levels"] == oexp["levels"]
    assert ex["info"]["top_node"] == oexp["top"]
    assert ex["point_level"] == oexp["point_level"]
    dev_nodes = [(i, lv, par, own, mem) for i, lv, par, own, mem in ex["nodes"]]
    ora_nodes = [(i, lv, par, own, mem) for i, lv, par, own, mem, _ in oexp["nodes"]]
    assert dev_nodes == ora_nodes
    assert {p: toks for p, (role, toks) in ex["pages"].items() if role == 3} == \
        {p: pg.tokens for p, pg in ostore.pages.items()}
    for i, lv, _, _, _, pages in oexp["nodes"]:
        if lv == 1:
            assert ex["leaf_pages"][i] == sorted(pages)


@pytest.mark.parametrize("name", TREES)
def test_build_matches_oracle(cuda_ok, name):
    z, meta = load_golden(f"tree_{name}.npz")
    otree, ostore = _oracle(z, meta)
    f = _device_build(z, meta, 0)
    assert f.scale(0) == otree.c
    _compare_structure(f, otree, ostore)
    ex = f.export(0, with_rows=True)
    n = meta["n"]
    rows32, tail32, _ = nm.lift_keys32(z["keys"][:n].astype(np.float64), otree.c)
    assert np.array_equal(ex["lift"][:n], rows32)
    assert np.array_equal(ex["tail"][:n], tail32)


def _filter_case(kind, n, d, rng):
    if kind == "duplicates":      # exact ties everywhere: windows overflow, first-index tie break
        base = rng.standard_normal((24, d))
        return base[rng.integers(0, 24, n)]
    if kind == "near_ties":       # every candidate inside the f16 error window
        return rng.standard_normal(d)[None, :] + 1e-5 * rng.standard_normal((n, d))
    if kind == "tiny_norms":      # coordinates in f16's subnormal range
        return rng.standard_normal((n, d)) * 10.0 ** rng.uniform(-6, 0, (n, 1))
    if kind == "spiky":           # one dominant coordinate: coarse int8 digits for all the others
        x = 1e-3 * rng.standard_normal((n, d))
        x[np.arange(n), rng.integers(0, d, n)] += rng.choice([-1.0, 1.0], n) * rng.uniform(0.5, 1.0, n)
        return x
    if kind == "near_ties_spiky":  # near-ties whose rows also quantise coarsely
        base = np.zeros(d)
        base[3] = 1.0
        return base[None, :] + 1e-4 * rng.standard_normal((n, d))
    return rng.standard_normal((n, d)) + 3.0 * rng.standard_normal((8, d))[rng.integers(0, 8, n)]


@pytest.mark.parametrize("kind,r", [("duplicates", 0.1), ("near_ties", 0.1), ("tiny_norms", 0.1),
                                    ("clustered", 0.3), ("spiky", 0.1), ("near_ties_spiky", 0.1)])
def test_build_parent_filter_edge_cases(cuda_ok, kind, r):
    """The tensor-core parent filter (nn_tc.cuh nn_tc_filter_kernel) must pick
    the exact fp64 1-NN parent, first index on ties, on inputs built to defeat
    it (exact ties, near-ties, tiny and spiky coordinates)."""
    n, d = 3000, 128
    rng = np.random.default_rng(hash(kind) % 2**32)
    keys = _filter_case(kind, n, d, rng).astype(np.float32)
    vals = rng.standard_normal((n, 4)).astype(np.float32)
    meta = {"n": n, "d": d, "r": r, "seed": 7, "page_size": 16}
    otree, ostore = _oracle({"keys": keys, "values": vals}, meta)
    f = _device_build({"keys": keys, "values": vals}, meta, 0)
    _compare_structure(f, otree, ostore)


@pytest.mark.parametrize("name", TREES)
def test_query_matches_oracle(cuda_ok, name):
    z, meta = load_golden(f"tree_{name}.npz")
    otree, _ = _oracle(z, meta)
    f = _device_build(z, meta, 0)
    k = meta["k"]
    qs = z["queries"].astype(np.float32)
    nq = len(qs)
    # all queries as G heads of one tree call (G <= 8 per call)
    for s in range(0, nq, 8):
        chunk = qs[s:s + 8]
        before = f.info(0)["distance_evals"]
        ids, counts, pages, npages = f.query([0], chunk[None], k, 2 * k, 4 * k)
        f.check()
        ids, counts = ids.cpu().numpy()[0], counts.cpu().numpy()[0]
        evals = 0
        want_pages = set()
        for g, q in enumerate(chunk):
            e0 = otree.distance_evals
            want = otree.query(nm.lift_query32(q.astype(np.float64)), SENTINEL, k, 2 * k, 4 * k)
            evals += otree.distance_evals - e0
            assert list(ids[g, :counts[g]]) == want
            want_pages |= {otree.store.token_to_page[t] for t in want}
        assert f.info(0)["distance_evals"] - before == evals
        assert list(pages.cpu().numpy()[0, :int(npages[0])]) == sorted(want_pages)
    # exhaustive budget: equals the oracle's exact ranking
    ids, counts, _, _ = f.query([0], qs[:4][None], k, 2**62, 2**62)
    for g in range(4):
        want = otree.query(nm.lift_query32(qs[g].astype(np.float64)), SENTINEL, k, 2**62, 2**62)
        assert list(ids[0, g, :counts[0, g]].cpu().numpy()) == want


@pytest.mark.parametrize("name", TREES)
def test_inserts_match_oracle(cuda_ok, name):
    z, meta = load_golden(f"tree_{name}.npz")
    otree, ostore = _oracle(z, meta)
    nins = len(meta["insert_levels"])
    f = _device_build(z, meta, nins)
    n = meta["n"]
    keys, vals = z["keys"].astype(np.float64), z["values"].astype(np.float64)
    want_levels = [otree.insert(i, keys[i], vals[i]) for i in range(n, n + nins)]
    assert want_levels == meta["insert_levels"]
    got = []
    for i in range(n, n + nins):   # one insert per call: exercises the call boundary too
        lv = f.insert([0], np.array([[i]]), z["keys"][i][None, None], z["values"][i][None, None])
        got.append(int(lv.cpu()[0, 0]))
    f.check()
    assert got == want_levels
    _compare_structure(f, otree, ostore)
    info = f.info(0)
    assert info["query_count"] == otree.query_count
    assert info["distance_evals"] == otree.distance_evals
    # batched: all inserts in one call give the same tree
    f2 = _device_build(z, meta, nins)
    f2.insert([0], np.arange(n, n + nins)[None], z["keys"][n:n + nins][None], z["values"][n:n + nins][None])
    f2.check()
    assert f2.export(0)["nodes"] == f.export(0)["nodes"]


@pytest.mark.parametrize("kv,tol", [("fp32", 1e-3), ("bf16", 1e-2)])
def test_sparse_attention_matches_fp64(cuda_ok, kv, tol):
    from paper_2604_10539_b200 import DeviceForest
    rng = np.random.default_rng(0)
    T, G, d, dv, n = 3, 4, 128, 128, 900
    keys = (rng.normal(size=(T, n, d)) / np.sqrt(d)).astype(np.float32)
    vals = (rng.normal(size=(T, n, dv)) / np.sqrt(dv)).astype(np.float32)
    f = DeviceForest(T, d, dv, tok_cap=n + 64, promotion_ratio=0.1, kv_dtype=kv)
    f.seed(range(T), [(1, t) for t in range(T)])
    # sink 16 tokens, window 24 tokens (2 pages), indexed rest
    f.alloc_resident(range(T), 1, 1, np.tile(np.arange(16), (T, 1)), keys[:, :16], vals[:, :16])
    f.alloc_resident(range(T), 2, 2, np.tile(np.arange(n - 24, n), (T, 1)), keys[:, n - 24:], vals[:, n - 24:])
    mid = np.arange(16, n - 24)
    f.build(range(T), np.tile(mid, (T, 1)), keys[:, 16:n - 24], vals[:, 16:n - 24])
    f.check()
    q = (rng.normal(size=(T, G, d))).astype(np.float32)
    ids, counts, pages, npages = f.query(range(T), q, 64, 128, 256)
    stats = torch.zeros((T, 5), dtype=torch.int64, device="cuda")
    out = f.attention(range(T), q, pages, npages, stats=stats).cpu().numpy()
    f.check()
    for t in range(T):
        ex = f.export(t)
        sel = list(pages[t, :int(npages[t])].cpu().numpy())
        toks = []
        for p in ex["sink"] + ex["win"] + sel:
            toks += ex["pages"][p][1]
        for g in range(G):
            _, ref = full_attention(q[t, g].astype(np.float64), keys[t, toks].astype(np.float64),
                                    vals[t, toks].astype(np.float64))
            err = np.linalg.norm(out[t, g] - ref) / np.linalg.norm(ref)
            assert err < tol, (t, g, err)
        st = stats[t].cpu().numpy()
        assert st[0] == len(sel) and st[2] == len(sel)   # first step: everything loads
        assert st[1] == sum(len(ex["pages"][p][1]) for p in sel)
    # identical queries reload nothing (pagestore residency)
    stats.zero_()
    f.attention(range(T), q, pages, npages, stats=stats)
    assert stats[:, 2].sum().item() == 0 and stats[:, 4].sum().item() == 0


@pytest.mark.parametrize("kv,tol", [("fp32", 1e-3), ("bf16", 1e-2)])
def test_dense_attention(cuda_ok, kv, tol):
    from paper_2604_10539_b200 import dense_attention
    rng = np.random.default_rng(1)
    n, G, T, d = 4, 4, 5000, 128
    k = torch.tensor(rng.normal(size=(n, T, d)) / np.sqrt(d), dtype=torch.float32, device="cuda")
    v = torch.tensor(rng.normal(size=(n, T, d)) / np.sqrt(d), dtype=torch.float32, device="cuda")
    q = torch.tensor(rng.normal(size=(n, G, d)), dtype=torch.float32, device="cuda")
    kk, vv = (k.bfloat16(), v.bfloat16()) if kv == "bf16" else (k, v)
    out = dense_attention(q, kk, vv, 4321).cpu().numpy()
    for b in range(n):
        for g in range(G):
            _, ref = full_attention(q[b, g].cpu().double().numpy(), k[b, :4321].cpu().double().numpy(),
                                    v[b, :4321].cpu().double().numpy())
            assert np.linalg.norm(out[b, g] - ref) / np.linalg.norm(ref) < tol


@pytest.mark.parametrize("G,ntok", [(4, 1), (4, 63), (4, 64), (4, 33000), (1, 777), (3, 5000), (8, 4097)])
def test_dense_flash_attention(cuda_ok, G, ntok):
    """The TMA + tensor-core dense kernel (bf16, d = d' = 128; csrc/dense.cu)
    against fp64 over the bf16-stored K/V, and the device-position variant."""
    import torch
    from paper_2604_10539_b200 import dense_attention
    rng = np.random.default_rng(ntok + G)
    n, T, d = 3, 33024, 128
    k = torch.tensor(rng.normal(size=(n, T, d)) / np.sqrt(d), dtype=torch.float32, device="cuda").bfloat16()
    v = torch.tensor(rng.normal(size=(n, T, d)) / np.sqrt(d), dtype=torch.float32, device="cuda").bfloat16()
    q = torch.tensor(rng.normal(size=(n, G, d)) * np.sqrt(d) * 0.3, dtype=torch.float32, device="cuda")
    out = dense_attention(q, k, v, ntok).cpu().numpy()
    pos = torch.tensor([ntok - 1], dtype=torch.int32, device="cuda")
    out_dev = dense_attention(q, k, v, pos).cpu().numpy()
    kd, vd = k.double().cpu().numpy(), v.double().cpu().numpy()
    for b in range(n):
        for g in range(G):
            _, ref = full_attention(q[b, g].cpu().double().numpy(), kd[b, :ntok], vd[b, :ntok])
            err = np.linalg.norm(out[b, g] - ref) / np.linalg.norm(ref)
            assert err < 2e-3, (b, g, err)
            assert np.linalg.norm(out_dev[b, g] - ref) / np.linalg.norm(ref) < 2e-3
