"""DeviceForest: T DCI trees resident in HBM, driven through the C ABI.

Host code here only moves pointers, sizes and streams; every operation of
the hot path (lifting, level draws, 1-NN, node/page construction, search,
page union, insert, attention) runs in the sm_100a kernels of
libicecache_b200.so.  Reference interfaces replaced are listed in
include/icecache_b200.h.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N
from .errors import ConfigError, InputError

DPAD = 128
ROWF = 128   # device row stride in floats (512 B); the lifted tail lives in its own array


def entropy_words(seed) -> list[int]:
    """NumPy SeedSequence entropy coercion (bit_generator.pyx
    _coerce_to_uint32_array): each int -> little-endian uint32 words."""
    items = [seed] if isinstance(seed, (int, np.integer)) else list(seed)
    out: list[int] = []
    for x in items:
        x = int(x)
        if x < 0:
            raise InputError("seed entropy must be non-negative")
        if x == 0:
            out.append(0)
        while x > 0:
            out.append(x & 0xFFFFFFFF)
            x >>= 32
    return out


def _ptr(t):
    return ctypes.c_void_p(0 if t is None else t.data_ptr())


def _stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


@dataclass
class ForestCaps:
    tok_cap: int
    node_cap: int
    page_cap: int
    member_cap: int
    own_cap: int
    dirs_cap: int = 64

    @staticmethod
    def for_stream(n_build: int, n_decode: int, r: float, page_size: int, resident_pages: int,
                   tight: bool = True) -> "ForestCaps":
        """Capacities for trees built over n_build points and then decoded for
        n_decode tokens.  Page K/V dominate HBM (8 KB per page at d = 128,
        bf16), so the page capacity is sized close to use:
        - build: every leaf is owned by a point of level >= 2 (Binomial(n, r):
          bounded at 8 standard deviations), and a leaf of m members takes
          ceil(m / s) pages; `tight` budgets half a page of fill slack per s
          points (C2: 4.2k pages used of a 4.8k estimate), the fallback
          (tight=False) the worst case of for_tokens.  A build that outgrows the
          tight estimate raises ConfigError and the Engine rebuilds with the
          worst case.
        - decode: each rotation inserts s points (at most one new page each)
          and opens one window page: at most s + 1 pages per s - 1 tokens."""
        tok_cap = n_build + n_decode
        base = ForestCaps.for_tokens(tok_cap, r, page_size, extra_pages=resident_pages + n_decode // page_size)
        if not tight:
            return base
        leaves = r * n_build + 8.0 * (n_build * r * (1.0 - r)) ** 0.5 + 16
        build_pages = int(leaves + n_build / (2.0 * page_size)) + 1
        decode_pages = (page_size + 1) * (n_decode // max(1, page_size - 1) + 2)
        base.page_cap = min(base.page_cap, resident_pages + build_pages + decode_pages + 8)
        return base

    @staticmethod
    def for_tokens(tok_cap: int, r: float, page_size: int, extra_pages: int = 64) -> "ForestCaps":
        frac = r / (1.0 - r)
        node_cap = int(tok_cap * frac * 1.6) + 256
        own_cap = int(tok_cap * frac * 1.6) + 256
        page_cap = int(tok_cap * (frac * 1.6 + 1.0 / page_size)) + extra_pages + 64
        member_cap = int(tok_cap / (1.0 - r) * 3) + 4096
        return ForestCaps(tok_cap, node_cap, page_cap, member_cap, own_cap)


class DeviceForest:
    """T independent DCI trees plus their page stores, resident on one GPU."""

    def __init__(self, n_trees: int, dim: int, dim_v: int, *, tok_cap: int, promotion_ratio: float = 0.1,
                 page_size: int = 16, kv_dtype: str = "fp32", caps: ForestCaps | None = None,
                 device=None, kv_host: bool = False, pool_pages: int = 0):
        """kv_host: page K/V live in pinned, device-mapped host memory; each fused
        decode step gathers the pages it attends into a per-tree HBM pool of
        `pool_pages` slots (TierStore backload / evict, pagestore.py:117-215)."""
        if not torch.cuda.is_available():
            raise RuntimeError("DeviceForest needs a CUDA device (B200); there is no CPU path")
        if dim > DPAD or dim_v > DPAD:
            raise ConfigError("the device path supports d, d' <= 128")
        self.device = torch.device(device or "cuda")
        self.n_trees, self.dim, self.dim_v, self.page_size = n_trees, dim, dim_v, page_size
        self.r = promotion_ratio
        self.kv_dtype = kv_dtype
        self.caps = caps or ForestCaps.for_tokens(tok_cap, promotion_ratio, page_size)
        c = N.icb_forest_config(n_trees, dim, dim_v, page_size,
                                N.KV_BF16 if kv_dtype == "bf16" else N.KV_F32,
                                self.caps.tok_cap, self.caps.node_cap, self.caps.page_cap,
                                self.caps.member_cap, self.caps.own_cap, self.caps.dirs_cap,
                                promotion_ratio, int(bool(kv_host)), int(pool_pages))
        self.kv_host = bool(kv_host)
        h = ctypes.c_void_p()
        with torch.cuda.device(self.device):
            N.check(N.lib().icb_forest_create(ctypes.byref(c), ctypes.byref(h)))
        self.h = h

    def pool_stats(self) -> np.ndarray:
        """KV offload: [n_trees, 2] = bytes gathered host -> HBM pool so far, pages
        resident in the pool now."""
        out = np.zeros((self.n_trees, 2), dtype=np.int64)
        N.check(N.lib().icb_pool_stats(self.h, out.ctypes.data_as(ctypes.c_void_p)))
        return out

    def close(self):
        if getattr(self, "h", None):
            N.lib().icb_forest_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- helpers ------------------------------------------------------------
    def _trees(self, trees):
        if isinstance(trees, torch.Tensor):
            return trees.to(device=self.device, dtype=torch.int32).contiguous()
        return torch.as_tensor(np.asarray(trees, dtype=np.int32), device=self.device)

    def _f32(self, x, shape=None):
        t = torch.as_tensor(x, dtype=torch.float32, device=self.device).contiguous()
        return t if shape is None else t.reshape(shape)

    def check(self, clear: bool = True):
        """Raise the reference exception for any sticky device error bits."""
        errs = np.zeros(self.n_trees, dtype=np.int32)
        N.check(N.lib().icb_errors(self.h, errs.ctypes.data_as(ctypes.c_void_p), int(clear)))
        bad = np.flatnonzero(errs)
        if bad.size:
            N.raise_device_error(int(errs[bad[0]]))

    # -- operations ---------------------------------------------------------------
    def seed(self, trees, seeds):
        trees = np.asarray(trees, dtype=np.int32)
        words = [entropy_words(s) for s in seeds]
        stride = max(len(w) for w in words)
        arr = np.zeros((len(words), stride), dtype=np.uint32)
        nw = np.zeros(len(words), dtype=np.int32)
        for i, w in enumerate(words):
            arr[i, : len(w)] = w
            nw[i] = len(w)
        N.check(N.lib().icb_seed_trees(self.h, trees.ctypes.data_as(ctypes.c_void_p), len(trees),
                                       arr.ctypes.data_as(ctypes.c_void_p), stride,
                                       nw.ctypes.data_as(ctypes.c_void_p)))

    def alloc_resident(self, trees, role: int, count: int, tokens, keys, values):
        tr = self._trees(trees)
        n = tr.numel()
        tok = torch.as_tensor(tokens, dtype=torch.int32, device=self.device).reshape(n, -1).contiguous()
        k = self._f32(keys, (n, tok.shape[1], self.dim))
        v = self._f32(values, (n, tok.shape[1], self.dim_v))
        N.check(N.lib().icb_alloc_resident_pages(self.h, _ptr(tr), n, role, count, tok.shape[1], _ptr(tok),
                                                 _ptr(k), _ptr(v), _stream()))

    def build(self, trees, tokens, keys, values=None, scales=None):
        """dci_indexing for every listed tree (dci.py:479-568)."""
        tr = self._trees(trees)
        n = tr.numel()
        tok = torch.as_tensor(tokens, dtype=torch.int32, device=self.device).reshape(n, -1).contiguous()
        P = tok.shape[1]
        k = self._f32(keys, (n, P, self.dim))
        v = None if values is None else self._f32(values, (n, P, self.dim_v))
        sc = None if scales is None else torch.as_tensor(scales, dtype=torch.float64,
                                                         device=self.device).reshape(n).contiguous()
        N.check(N.lib().icb_build(self.h, _ptr(tr), n, P, _ptr(tok), _ptr(k), _ptr(v), _ptr(sc), _stream()))

    def query(self, trees, queries, k, beam, visit_cap, target_level=N.SENTINEL_LEVEL, *, lifted=False,
              k_out=None, pages_cap=None, want_pages=True, out=None):
        """Search G query heads per tree; returns (ids [n,G,k_out], counts [n,G],
        pages [n,pages_cap], npages [n]) as device tensors."""
        tr = self._trees(trees)
        n = tr.numel()
        q = torch.as_tensor(queries, dtype=torch.float32, device=self.device)
        width = self.dim + (1 if lifted else 0)
        q = q.reshape(n, -1, width).contiguous()
        G = q.shape[1]
        beam = int(min(beam, 2**62))
        visit_cap = int(min(visit_cap, 2**62))
        k = int(min(k, 2**30))
        if k_out is None:
            k_out = min(k, self.caps.tok_cap)
        if pages_cap is None:
            pages_cap = min(self.caps.page_cap, G * k_out)
        if out is None:
            ids = torch.empty((n, G, k_out), dtype=torch.int32, device=self.device)
            counts = torch.empty((n, G), dtype=torch.int32, device=self.device)
            pages = torch.empty((n, max(1, pages_cap)), dtype=torch.int32, device=self.device) if want_pages else None
            npages = torch.empty((n,), dtype=torch.int32, device=self.device) if want_pages else None
        else:
            ids, counts, pages, npages = out
        N.check(N.lib().icb_query(self.h, _ptr(tr), n, G, _ptr(q), int(lifted), k, beam, visit_cap,
                                  int(target_level), _ptr(ids), k_out, _ptr(counts), _ptr(pages),
                                  pages_cap if want_pages else 0, _ptr(npages), _stream()))
        return ids, counts, pages, npages

    def query_attend(self, trees, queries, k, beam, visit_cap, *, out, attn_out, stats=None, scalar_bytes=4):
        """The decode step's selection + sparse attention in one launch
        (icb_query_attend): out = (ids, counts, pages, npages) buffers as for
        query(); attn_out [n,G,dim_v] fp32; stats [n,5] residency counters."""
        tr = self._trees(trees)
        n = tr.numel()
        q = self._f32(queries).reshape(n, -1, self.dim).contiguous()
        G = q.shape[1]
        ids, counts, pages, npages = out
        N.check(N.lib().icb_query_attend(self.h, _ptr(tr), n, G, _ptr(q), int(min(k, 2**30)), int(min(beam, 2**62)),
                                         int(min(visit_cap, 2**62)), _ptr(ids), ids.shape[2], _ptr(counts),
                                         _ptr(pages), pages.shape[1], _ptr(npages), _ptr(attn_out), _ptr(stats),
                                         scalar_bytes, _stream()))
        return attn_out

    def step_attend(self, trees, queries, k, beam, visit_cap, *, out, attn_out, token_dev, keys, values,
                    rotate=False, rot_stats=None, stats=None, scalar_bytes=4):
        """A whole decode step of these trees in one launch (icb_step_attend):
        per tree, rotate_window (if `rotate`), append_window(token_dev, keys,
        values), then query_attend.  Same results as those calls in sequence."""
        tr = self._trees(trees)
        n = tr.numel()
        q = self._f32(queries).reshape(n, -1, self.dim).contiguous()
        G = q.shape[1]
        ids, counts, pages, npages = out
        kk, vv = self._f32(keys, (n, self.dim)), self._f32(values, (n, self.dim_v))
        N.check(N.lib().icb_step_attend(self.h, _ptr(tr), n, G, _ptr(q), int(min(k, 2**30)), int(min(beam, 2**62)),
                                        int(min(visit_cap, 2**62)), _ptr(ids), ids.shape[2], _ptr(counts),
                                        _ptr(pages), pages.shape[1], _ptr(npages), _ptr(attn_out), _ptr(stats),
                                        scalar_bytes, int(bool(rotate)), _ptr(rot_stats), _ptr(token_dev),
                                        _ptr(kk), _ptr(vv), _stream()))
        return attn_out

    def insert(self, trees, tokens, keys, values=None, levels=None):
        tr = self._trees(trees)
        n = tr.numel()
        tok = torch.as_tensor(tokens, dtype=torch.int32, device=self.device).reshape(n, -1).contiguous()
        m = tok.shape[1]
        k = self._f32(keys, (n, m, self.dim))
        v = None if values is None else self._f32(values, (n, m, self.dim_v))
        lv = None if levels is None else torch.as_tensor(levels, dtype=torch.int32,
                                                         device=self.device).reshape(n, m).contiguous()
        out = torch.empty((n, m), dtype=torch.int32, device=self.device)
        N.check(N.lib().icb_insert(self.h, _ptr(tr), n, m, _ptr(tok), _ptr(k), _ptr(v), _ptr(lv), _ptr(out),
                                   _stream()))
        return out

    def pages_from_tokens(self, trees, src_rows, ids, counts, out_pages, out_npages):
        """select_with_reuse's page lists (engine.py:331-363): tree trees[b]'s
        sorted unique pages of the token lists in query-output row src_rows[b]
        (ids [rows][G][k], counts [rows][G] as written by query())."""
        tr = self._trees(trees)
        n = tr.numel()
        G, ks = ids.shape[1], ids.shape[2]
        N.check(N.lib().icb_pages_from_tokens(self.h, _ptr(tr), n, _ptr(src_rows), _ptr(ids), _ptr(counts), G, ks,
                                              _ptr(out_pages), out_pages.shape[1], _ptr(out_npages), _stream()))

    def attended_mask(self, trees, pages, npages, out):
        """out uint8 [n, tok_cap]: 1 for tokens of the sink, window and
        selected pages of each tree (the attended set)."""
        tr = self._trees(trees)
        N.check(N.lib().icb_attended_mask(self.h, _ptr(tr), tr.numel(), _ptr(pages), pages.shape[1], _ptr(npages),
                                          _ptr(out), _stream()))
        return out

    def rotate_window(self, trees, scalar_bytes=4, stats=None):
        tr = self._trees(trees)
        N.check(N.lib().icb_rotate_window(self.h, _ptr(tr), tr.numel(), scalar_bytes, _ptr(stats), _stream()))

    def append_window(self, trees, token, keys, values):
        """`token`: an int, or an int32 device tensor holding it (CUDA-graph replays)."""
        tr = self._trees(trees)
        n = tr.numel()
        k, v = _ptr(self._f32(keys, (n, self.dim))), _ptr(self._f32(values, (n, self.dim_v)))
        if isinstance(token, torch.Tensor):
            N.check(N.lib().icb_append_window_dev(self.h, _ptr(tr), n, _ptr(token), k, v, _stream()))
        else:
            N.check(N.lib().icb_append_window(self.h, _ptr(tr), n, int(token), k, v, _stream()))

    def attention(self, trees, queries, pages, npages, *, out=None, stats=None, scalar_bytes=4, splits=0):
        tr = self._trees(trees)
        n = tr.numel()
        q = self._f32(queries).reshape(n, -1, self.dim).contiguous()
        G = q.shape[1]
        if out is None:
            out = torch.empty((n, G, self.dim_v), dtype=torch.float32, device=self.device)
        N.check(N.lib().icb_sparse_attention(self.h, _ptr(tr), n, G, _ptr(q), _ptr(pages), pages.shape[1],
                                             _ptr(npages), _ptr(out), _ptr(stats), scalar_bytes, splits,
                                             _stream()))
        return out

    # -- host mirror ------------------------------------------------------------------
    def info(self, tree: int) -> dict:
        out = np.zeros(16, dtype=np.int64)
        N.check(N.lib().icb_tree_info(self.h, int(tree), out.ctypes.data_as(ctypes.c_void_p)))
        keys = ["levels", "top_node", "n_nodes", "next_page", "n_points", "err", "n_window", "n_sink",
                "query_count", "distance_evals", "scale_clamps", "member_top", "own_top", "n_dirs",
                "rows_read", "owner_rereads"]
        return {k: int(v) for k, v in zip(keys, out)}

    def scale(self, tree: int) -> float:
        c = np.zeros(1, dtype=np.float64)
        N.check(N.lib().icb_read_meta_c(self.h, int(tree), c.ctypes.data_as(ctypes.c_void_p)))
        return float(c[0])

    def export(self, tree: int, with_rows: bool = False) -> dict:
        """Canonical host mirror of one tree (nodes, pages, token map)."""
        cp = self.caps
        s = self.page_size
        arrs = dict(
            node_level=np.zeros(cp.node_cap, np.int32), node_parent=np.zeros(cp.node_cap, np.int32),
            node_owner=np.zeros(cp.node_cap, np.int32), node_off=np.zeros(cp.node_cap, np.int32),
            node_size=np.zeros(cp.node_cap, np.int32), node_lastpage=np.zeros(cp.node_cap, np.int32),
            members=np.zeros(cp.member_cap, np.int32), page_fill=np.zeros(cp.page_cap, np.int32),
            page_role=np.zeros(cp.page_cap, np.int8), page_tok=np.zeros(cp.page_cap * s, np.int32),
            tok2page=np.zeros(cp.tok_cap, np.int32), level=np.zeros(cp.tok_cap, np.int8),
            own_base=np.zeros(cp.tok_cap, np.int32), own_list=np.zeros(cp.own_cap, np.int32))
        lift = np.zeros(cp.tok_cap * ROWF, np.float32) if with_rows else None
        tail = np.zeros(cp.tok_cap, np.float32) if with_rows else None
        win = np.zeros(8, np.int32)
        sink = np.zeros(8, np.int32)
        order = ["node_level", "node_parent", "node_owner", "node_off", "node_size", "node_lastpage", "members",
                 "page_fill", "page_role", "page_tok", "tok2page", "level", "own_base", "own_list"]
        ptrs = [arrs[k].ctypes.data_as(ctypes.c_void_p) for k in order]
        ptrs += [None if lift is None else lift.ctypes.data_as(ctypes.c_void_p),
                 None if tail is None else tail.ctypes.data_as(ctypes.c_void_p),
                 win.ctypes.data_as(ctypes.c_void_p), sink.ctypes.data_as(ctypes.c_void_p)]
        N.check(N.lib().icb_export_tree(self.h, int(tree), *ptrs))
        info = self.info(tree)
        nn = info["n_nodes"]
        nodes = []
        for i in range(nn):
            lv = int(arrs["node_level"][i])
            off, sz = int(arrs["node_off"][i]), int(arrs["node_size"][i])
            members = tuple(int(x) for x in arrs["members"][off:off + sz])
            nodes.append([i, lv, int(arrs["node_parent"][i]), int(arrs["node_owner"][i]), members])
        pages = {}
        for p in range(info["next_page"]):
            role = int(arrs["page_role"][p])
            if role == 0:
                continue
            fill = int(arrs["page_fill"][p])
            pages[p] = (role, [int(x) for x in arrs["page_tok"][p * s:p * s + fill]])
        # leaf page lists: pages whose tokens belong to the leaf, in id order
        leaf_pages: dict[int, list[int]] = {}
        t2p = arrs["tok2page"]
        for i, lv, _, _, members in nodes:
            if lv == 1:
                leaf_pages[i] = sorted({int(t2p[m]) for m in members})
        point_level = {int(t): int(l) for t, l in enumerate(arrs["level"]) if l > 0}
        out = dict(info=info, nodes=nodes, pages=pages, leaf_pages=leaf_pages, point_level=point_level,
                   tok2page=t2p, win=[int(x) for x in win if x >= 0], sink=[int(x) for x in sink if x >= 0],
                   own_base=arrs["own_base"], own_list=arrs["own_list"])
        if with_rows:
            rows = lift.reshape(cp.tok_cap, ROWF)
            out["lift"] = rows[:, :DPAD]
            out["tail"] = tail
        return out

    def read_pages(self, tree: int, pages):
        pages = np.asarray(pages, dtype=np.int32)
        k = np.zeros((len(pages), self.page_size, self.dim), np.float32)
        v = np.zeros((len(pages), self.page_size, self.dim_v), np.float32)
        N.check(N.lib().icb_read_pages(self.h, int(tree), pages.ctypes.data_as(ctypes.c_void_p), len(pages),
                                       k.ctypes.data_as(ctypes.c_void_p), v.ctypes.data_as(ctypes.c_void_p)))
        return k, v


def dense_attention(q, k, v, n_tokens=None, *, splits=0, out=None, dim_v=None):
    """full_attention (attention.py:55-74) over the first n_tokens rows of
    contiguous K/V on the device.  q [n,G,d] fp32; k [n,T,ceil4(d)],
    v [n,T,ceil4(d')] fp32 or bf16 (same dtype, contiguous; rows padded to 4
    elements as dense_append writes them); d' = dim_v (default v's width).
    Logits are scaled by 1/sqrt(d), d = q.shape[-1].  `n_tokens` may be an
    int32 device tensor holding the decode position p (rows [0, p + 1) are
    attended)."""
    n, G, d = q.shape
    dv = int(dim_v) if dim_v is not None else v.shape[-1]
    if k.shape[-1] != (d + 3) // 4 * 4 or v.shape[-1] != (dv + 3) // 4 * 4:
        raise ConfigError("dense K/V rows must be padded to ceil4(d) / ceil4(d')")
    if n_tokens is None:
        n_tokens = k.shape[1]
    if out is None:
        out = torch.empty((n, G, dv), dtype=torch.float32, device=q.device)
    kvd = N.KV_BF16 if k.dtype == torch.bfloat16 else N.KV_F32
    q = q.contiguous()
    if isinstance(n_tokens, torch.Tensor):
        N.check(N.lib().icb_dense_attention_dev(n, G, d, dv, kvd, _ptr(q), _ptr(k), _ptr(v), k.shape[1],
                                                _ptr(n_tokens), _ptr(out), splits, _stream()))
    else:
        N.check(N.lib().icb_dense_attention(n, G, d, dv, kvd, _ptr(q), _ptr(k), _ptr(v), k.shape[1],
                                            int(n_tokens), _ptr(out), splits, _stream()))
    return out


def dense_append(k, v, dense_k, dense_v, token_dev):
    """Write row token_dev[0] of each dense K/V plane: k [n,d], v [n,d'] fp32
    into dense_k [n,T,ceil4(d)], dense_v [n,T,ceil4(d')] (fp32 or bf16)."""
    n, d = k.shape
    dv = v.shape[-1]
    kvd = N.KV_BF16 if dense_k.dtype == torch.bfloat16 else N.KV_F32
    N.check(N.lib().icb_dense_append(n, d, dv, kvd, _ptr(k.contiguous()), _ptr(v.contiguous()), _ptr(dense_k),
                                     _ptr(dense_v), dense_k.shape[1], _ptr(token_dev), _stream()))
