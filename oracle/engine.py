"""Oracle engine: restates engine.py (prefill :226-301, decode_step :383-514,
_rotate_layer :516-534) and attention.py (:55-103) over the oracle tree.
TEST INFRASTRUCTURE ONLY."""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import numerics as nm
from .dci import SENTINEL, build
from .store import SINK, WINDOW, OStore, find_page_index


def full_attention(q, keys, values):
    """attention.py:55-74 in fp64: softmax(K q / sqrt(d)) V."""
    q = np.asarray(q, dtype=np.float64)
    k = np.asarray(keys, dtype=np.float64)
    v = np.asarray(values, dtype=np.float64)
    logits = (k @ q) / np.sqrt(q.size)
    logits -= logits.max()
    w = np.exp(logits)
    w /= w.sum()
    return w, w @ v


@dataclass
class OConfig:
    layers: int = 4
    kv_heads: int = 2
    query_heads_per_group: int = 1
    d: int = 64
    d_prime: int = 64
    page_size: int = 16
    token_budget: int = 64
    promotion_ratio: float = 0.1
    sink_pages: int = 1
    window_pages: int = 2
    skip_layers: int = 2
    beam: int | None = None
    visit_cap: int | None = None
    seed: int = 0
    scalar_bytes: int = 4
    reuse_stride: int = 0

    def budget(self):
        k = self.token_budget
        return (k, self.beam if self.beam is not None else 2 * k,
                self.visit_cap if self.visit_cap is not None else 4 * k)


class _Head:
    def __init__(self, tree, store, sink, window):
        self.tree, self.store, self.sink, self.window = tree, store, sink, window


class OracleEngine:
    def __init__(self, cfg: OConfig):
        self.cfg = cfg
        self.heads: dict[tuple[int, int], _Head] = {}
        self.fallback = False
        self.n_prefill = 0
        self.steps = 0
        self.mk: dict[tuple[int, int], list] = {}
        self.mv: dict[tuple[int, int], list] = {}
        self.sink_tokens: list[int] = []
        self.indexed_tokens: list[int] = []
        self.selection_queries = 0
        self.trace: list[dict] = []   # per step: selected tokens / pages
        self._anchor_tokens: dict[int, set] = {}

    def prefill(self, keys, values, n_prefill):
        """keys [n,L,H,d], values [n,L,H,d'] fp64 (fp32-representable)."""
        cfg = self.cfg
        self.n_prefill = n_prefill
        for layer in range(cfg.layers):
            for h in range(cfg.kv_heads):
                self.mk[(layer, h)] = [keys[:n_prefill, layer, h]]
                self.mv[(layer, h)] = [values[:n_prefill, layer, h]]
        s = cfg.page_size
        pages = math.ceil(n_prefill / s)
        if pages < cfg.sink_pages + cfg.window_pages + 1 or cfg.skip_layers >= cfg.layers:
            self.fallback = True
            return self
        sink_end = cfg.sink_pages * s
        win_start = (pages - cfg.window_pages) * s
        self.sink_tokens = list(range(sink_end))
        self.indexed_tokens = list(range(sink_end, win_start))
        for layer in range(cfg.skip_layers, cfg.layers):
            for h in range(cfg.kv_heads):
                store = OStore(cfg.d, cfg.d_prime, cfg.scalar_bytes)
                sink, window = [], []
                for start in range(0, sink_end, s):
                    p = store.allocate(s, SINK, resident=True, pinned=True)
                    for t in range(start, min(start + s, n_prefill)):
                        p.tokens.append(t)
                        p.keys.append(keys[t, layer, h])
                        p.values.append(values[t, layer, h])
                    sink.append(p)
                for start in range(win_start, n_prefill, s):
                    p = store.allocate(s, WINDOW, resident=True, pinned=True)
                    for t in range(start, min(start + s, n_prefill)):
                        p.tokens.append(t)
                        p.keys.append(keys[t, layer, h])
                        p.values.append(values[t, layer, h])
                    window.append(p)
                mid = self.indexed_tokens
                tree = build([(t, keys[t, layer, h]) for t in mid], cfg.promotion_ratio,
                             seed=(cfg.seed, layer, h), values=[values[t, layer, h] for t in mid],
                             store=store, page_size=s)
                self.heads[(layer, h)] = _Head(tree, store, sink, window)
        return self

    def select_tokens(self, q, layer, h):
        k, beam, cap = self.cfg.budget()
        self.selection_queries += 1
        return self.heads[(layer, h)].tree.query(nm.lift_query32(q), SENTINEL, k, beam, cap)

    def page_select(self, q, layer, h):
        toks = self.select_tokens(q, layer, h)
        return find_page_index(toks, self.heads[(layer, h)].store.token_to_page)

    def _rotate(self, layer):
        cfg = self.cfg
        rotated = None
        for h in range(cfg.kv_heads):
            st = self.heads[(layer, h)]
            old = st.window.pop(0)
            st.store.offload(old.page_id)
            for t, k, v in zip(old.tokens, old.keys, old.values):
                st.tree.insert(t, k, v)
            st.store.release(old.page_id)
            st.window.append(st.store.allocate(cfg.page_size, WINDOW, resident=True, pinned=True))
            rotated = list(old.tokens)
        if layer == cfg.skip_layers and rotated:
            self.indexed_tokens.extend(rotated)

    def decode_step(self, token, queries, keys, values):
        """One decode token (engine.py:383-514).  queries [L,H*G,d], keys
        [L,H,d], values [L,H,d'].  Returns (outputs [L,H*G,d'], metrics, trace)."""
        cfg = self.cfg
        G = cfg.query_heads_per_group
        out = np.zeros((cfg.layers, cfg.kv_heads * G, cfg.d_prime))
        m = dict(pages_selected=0, pages_loaded=0, tokens_loaded=0, bytes_moved=0,
                 transactions=0)
        q0 = self.selection_queries
        trace = dict(tokens={}, pages={})
        rotate = False
        if not self.fallback:
            rotate = self.heads[(cfg.skip_layers, 0)].window[-1].fill >= cfg.page_size - 1
        for layer in range(cfg.layers):
            for h in range(cfg.kv_heads):
                self.mk[(layer, h)].append(keys[layer, h][None, :])
                self.mv[(layer, h)].append(values[layer, h][None, :])
            if self.fallback or layer < cfg.skip_layers:
                for qh in range(cfg.kv_heads * G):
                    h = qh // G
                    _, out[layer, qh] = full_attention(queries[layer, qh],
                                                       np.concatenate(self.mk[(layer, h)]),
                                                       np.concatenate(self.mv[(layer, h)]))
                continue
            if rotate:
                self._rotate(layer)
            for h in range(cfg.kv_heads):
                st = self.heads[(layer, h)]
                tgt = next(p for p in st.window if not p.full)
                tgt.tokens.append(token)
                tgt.keys.append(keys[layer, h])
                tgt.values.append(values[layer, h])
            for h in range(cfg.kv_heads):
                st = self.heads[(layer, h)]
                if cfg.reuse_stride >= 2 and (layer - cfg.skip_layers) % cfg.reuse_stride != 0:
                    # select_with_reuse (engine.py:331-363): the latest anchor's
                    # token union, mapped through this layer's page table
                    toks = self._anchor_tokens[h]
                    for g in range(G):
                        trace["tokens"][(layer, h * G + g)] = sorted(toks)
                    sel = find_page_index(sorted(toks), st.store.token_to_page)
                else:
                    per = []
                    union = set()
                    for g in range(G):
                        qh = h * G + g
                        toks = self.select_tokens(queries[layer, qh], layer, h)
                        trace["tokens"][(layer, qh)] = toks
                        union.update(toks)
                        per.append(find_page_index(toks, st.store.token_to_page))
                    if cfg.reuse_stride >= 2:
                        self._anchor_tokens[h] = union
                    sel = sorted(set().union(*per))
                trace["pages"][(layer, h)] = sel
                delta = st.store.backload(sel)
                ents_k, ents_v = [], []
                for p in st.sink + st.window:
                    ents_k += p.keys
                    ents_v += p.values
                for pid in sel:
                    ents_k += st.store.pages[pid].keys
                    ents_v += st.store.pages[pid].values
                for g in range(G):
                    qh = h * G + g
                    _, out[layer, qh] = full_attention(queries[layer, qh], ents_k, ents_v)
                st.store.evict_unselected(sel)
                m["pages_selected"] += len(sel)
                m["tokens_loaded"] += sum(st.store.pages[p].fill for p in sel)
                m["pages_loaded"] += delta["pages_backloaded"]
                m["bytes_moved"] += delta["bytes_moved"]
                m["transactions"] += delta["transactions"]
        self.steps += 1
        m["dci_queries"] = self.selection_queries - q0
        self.trace.append(trace)
        return out, m, trace
