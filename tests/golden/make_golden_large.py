"""Golden vectors at the sizes the bench reports, made by running the
UNMODIFIED reference package (read-only import of /root/reference/pkg/src).

Runs only in the build container; the .npz fixtures are committed and travel
to the GPU box.  Inputs are NOT stored: every case records its
WorkloadSpec (or its clustered() seed) and the tests regenerate the same
bits with a NumPy restatement of the reference generator
(paper_2604_10539_b200.workload.generate_workload, oracle.workload.generate).

  python tests/golden/make_golden_large.py [tree32k tree128k c2 c5]

Cases
  tree_c2_32k   one C2 tree (n_idx = 32,720, d = 128, r = 0.1, seed (0, 2, 0)):
                structure, 64 ranked top-256 queries (+ distance evals),
                16 inserts, structure after, 16 queries after
  tree_c3_128k  one C3 tree (n_idx = 131,024; > 98,304 points: the device's
                exact-parent build path), structure, 32 queries, 16 inserts
  engine_c2_s{0..4}  C2-shaped engine (3 layers: 2 dense skip + 1 indexed,
                8 kv heads, G = 4, d = 128, 32k prefill), 16 decode steps
                (two rotations): metric rows, every ranked token list,
                outputs (seed 0)
  engine_c5     C5-shaped long generation (8k prompt, 2 kv heads, G = 4,
                d = 128), 2,048 decode steps = 128 rotations x 16 inserts per
                tree: metric rows every step, a digest of every head's token
                set every step, full ranked lists every 16th step
"""

from __future__ import annotations

import json
import os
import sys
import time
import zlib

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
import icecache as ic  # noqa: E402
from icecache.dci import SENTINEL_LEVEL  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def f32(x):
    return np.asarray(x, dtype=np.float64).astype(np.float32).astype(np.float64)


def set_digest(tokens) -> int:
    """crc32 of the sorted token set as little-endian int32 (order-free)."""
    return zlib.crc32(np.asarray(sorted(int(t) for t in tokens), dtype="<i4").tobytes())


def workload(spec_kw):
    wl = ic.generate_workload(ic.WorkloadSpec(kind="clustered", **spec_kw))
    wl.keys[:] = f32(wl.keys)
    wl.values[:] = f32(wl.values)
    wl.queries[:] = f32(wl.queries)
    return wl


def tree_struct(tree, store):
    """Flat structure arrays: nodes (id order) with level / parent / owner,
    concatenated members, per-point levels, pages with their token lists."""
    nodes = sorted(tree.nodes.values(), key=lambda x: x.node_id)
    assert [n.node_id for n in nodes] == list(range(len(nodes)))
    lvl = np.array([n.level for n in nodes], np.int32)
    par = np.array([-1 if n.parent_id is None else n.parent_id for n in nodes], np.int32)
    own = np.array([n.owner_id for n in nodes], np.int32)
    msz = np.array([len(n.member_ids) for n in nodes], np.int32)
    mem = np.concatenate([np.asarray(n.member_ids, np.int32) for n in nodes])
    pids = sorted(store.pages)
    pg_id = np.array(pids, np.int32)
    pg_fill = np.array([store.pages[p].fill for p in pids], np.int32)
    pg_tok = np.concatenate([np.asarray(store.pages[p].token_ids, np.int32) for p in pids])
    pts = sorted(tree.point_level)
    pl = np.array([[p, tree.point_level[p]] for p in pts], np.int32)
    return dict(node_level=lvl, node_parent=par, node_owner=own, node_msize=msz, node_members=mem,
                page_id=pg_id, page_fill=pg_fill, page_tok=pg_tok, point_level=pl)


def tree_case(name, n_tokens, seed, n_queries, n_inserts, layer=2, h=0):
    """One (layer, kv head) tree of the engine's layout: sink = 1 page,
    window = 2 pages, the middle indexed (engine.py:254-281)."""
    t0 = time.time()
    spec = dict(n_tokens=n_tokens + 64, d=128, d_prime=128, clusters=32, layers=layer + 1, kv_heads=h + 1,
                query_heads_per_group=4, seed=seed)
    wl = workload(spec)
    s = 16
    sink_end, win_start = s, n_tokens - 2 * s
    idx = list(range(sink_end, win_start))
    store = ic.TierStore(128, 128)
    store.allocate_page(s, ic.pagestore.SINK, resident=True, pinned=True)
    store.allocate_page(s, ic.pagestore.WINDOW, resident=True, pinned=True)
    store.allocate_page(s, ic.pagestore.WINDOW, resident=True, pinned=True)
    table = ic.PageTable()
    tree = ic.dci_indexing([(t, wl.keys[t, layer, h]) for t in idx], 0.1, seed=(seed, layer, h),
                           values=[wl.values[t, layer, h] for t in idx], store=store, table=table, page_size=s)
    build_s = time.time() - t0
    before = tree_struct(tree, store)
    budget = ic.SearchBudget.for_k(256)
    qtok = [n_tokens + i // 4 for i in range(n_queries)]
    qhead = [h * 4 + i % 4 for i in range(n_queries)]
    topk, evals = [], []
    for tk, qh in zip(qtok, qhead):
        e0 = tree.distance_evals
        topk.append(tree.query(ic.transform_query(wl.queries[tk, layer, qh]), SENTINEL_LEVEL, 256, budget))
        evals.append(tree.distance_evals - e0)
    ins = list(range(win_start, win_start + n_inserts))
    levels = [tree.insert(t, wl.keys[t, layer, h], wl.values[t, layer, h]) for t in ins]
    tree.check_invariants()
    after = tree_struct(tree, store)
    topk_after = [tree.query(ic.transform_query(wl.queries[tk, layer, qh]), SENTINEL_LEVEL, 256, budget)
                  for tk, qh in zip(qtok[:16], qhead[:16])]
    meta = dict(name=name, spec=spec, layer=layer, h=h, n_tokens=n_tokens, sink_end=sink_end,
                win_start=win_start, r=0.1, seed=[seed, layer, h], page_size=s, k=256, scale=tree.scale.c,
                levels=tree.levels, query_tokens=qtok, query_heads=qhead, evals=evals, insert_tokens=ins,
                insert_levels=levels, build_s=build_s)
    arrs = {f"b_{k}": v for k, v in before.items()}
    arrs.update({f"a_{k}": v for k, v in after.items()})
    np.savez_compressed(os.path.join(OUT, f"{name}.npz"), topk=np.array(topk, np.int32),
                        topk_after=np.array(topk_after, np.int32), meta=json.dumps(meta), **arrs)
    print(name, "levels", tree.levels, "nodes", len(tree.nodes), f"{time.time() - t0:.1f}s", flush=True)


def engine_case(name, spec_kw, cfg_kw, n_prefill, steps, *, outputs, full_every=1):
    t0 = time.time()
    wl = workload(spec_kw)
    cfg = ic.EngineConfig(layers=spec_kw["layers"], kv_heads=spec_kw["kv_heads"],
                          query_heads_per_group=spec_kw["query_heads_per_group"], d=spec_kw["d"],
                          d_prime=spec_kw["d_prime"], seed=spec_kw["seed"], **cfg_kw)
    eng = ic.Engine(cfg).prefill(wl, n_prefill)
    log = []
    orig = eng._select_tokens

    def spy(q, layer, kv_head, budget=None):
        res = orig(q, layer, kv_head, budget)
        log[-1].append((layer, kv_head, list(map(int, res))))
        return res
    eng._select_tokens = spy
    rows, outs, digests, full, full_steps = [], [], [], [], []
    for t in range(steps):
        log.append([])
        o, m = eng.decode_step(wl.decode_step(n_prefill, t))
        rows.append([m.pages_selected, m.pages_loaded, m.tokens_loaded, m.bytes_moved, m.transactions,
                     m.dci_queries])
        digests.append([set_digest(tok) for _, _, tok in log[-1]])
        if t % full_every == 0:
            full_steps.append(t)
            full.append([tok + [-1] * (256 - len(tok)) for _, _, tok in log[-1]])
        if outputs:
            outs.append(np.stack([[o[l][qh].value_out for qh in range(cfg.n_query_heads)]
                                  for l in range(cfg.layers)]).astype(np.float32))
        log[-1] = [(a, b, None) for a, b, _ in log[-1]]
    calls = [(a, b) for a, b, _ in log[0]]
    meta = dict(name=name, spec=spec_kw, cfg=cfg_kw, n_prefill=n_prefill, steps=steps, calls=calls,
                row_fields=["pages_selected", "pages_loaded", "tokens_loaded", "bytes_moved", "transactions",
                            "dci_queries"], full_steps=full_steps)
    extra = {"outputs": np.stack(outs)} if outputs else {}
    np.savez_compressed(os.path.join(OUT, f"{name}.npz"), rows=np.array(rows, np.int64),
                        digests=np.array(digests, np.uint32), tokens=np.array(full, np.int32),
                        meta=json.dumps(meta), **extra)
    print(name, rows[0], rows[-1], f"{time.time() - t0:.1f}s", flush=True)


C2_SPEC = dict(d=128, d_prime=128, clusters=32, layers=3, kv_heads=8, query_heads_per_group=4)
C2_CFG = dict(token_budget=256, skip_layers=2)


if __name__ == "__main__":
    which = sys.argv[1:] or ["tree32k", "tree128k", "c2", "c5"]
    if "tree32k" in which:
        tree_case("tree_c2_32k", 32768, 0, 64, 16)
    if "tree128k" in which:
        tree_case("tree_c3_128k", 131072, 0, 32, 16)
    if "c2" in which:
        for s in range(5):
            engine_case(f"engine_c2_s{s}", dict(C2_SPEC, n_tokens=32768 + 16, seed=s), C2_CFG, 32768, 16,
                        outputs=(s == 0))
    if "c5" in which:
        engine_case("engine_c5", dict(d=128, d_prime=128, clusters=32, layers=3, kv_heads=2,
                                      query_heads_per_group=4, n_tokens=8192 + 2048, seed=0),
                    C2_CFG, 8192, 2048, outputs=False, full_every=16)
