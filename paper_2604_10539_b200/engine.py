"""Decode engine on the device: the drop-in for Engine.prefill / page_select /
decode_step (/root/reference/pkg/src/icecache/engine.py:226-514).

Layout: indexed layers (layer >= skip_layers) x kv heads form one forest of
T = (L - skip) * H trees, tree t = (layer - skip) * H + h.  Skip layers keep
their full K/V token-major in HBM and attend densely.  All per-step work of
every indexed tree runs in a handful of batched kernel launches (rotation,
window append, search + page union, paged attention), which the reference's
semantics allow: its layers are independent within a step (the engine is
not a transformer; every layer's q/k/v come from the workload stream).
`layer_serial=True` processes one layer at a time instead (the latency a
real model would see, reported separately).
"""

from __future__ import annotations

import math
from dataclasses import asdict, dataclass

import numpy as np
import torch

from . import _native as N
from .errors import ConfigError, InputError
from .forest import DeviceForest, ForestCaps, _ptr, _stream, dense_append, dense_attention


@dataclass
class EngineConfig:
    """Field names and validation follow engine.py:37-92 verbatim; the last
    five fields are device options."""

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
    reuse_stride: int = 0
    beam: int | None = None
    visit_cap: int | None = None
    seed: int = 0
    scalar_bytes: int = 4
    evaluate: bool = False
    compare_baseline: bool = False
    workers: int = 1
    kv_dtype: str = "fp32"        # page K/V storage: "fp32" | "bf16"
    max_tokens: int | None = None  # token capacity (prefill + decode); default prefill + 1024
    layer_serial: bool = False
    overlap_dense: bool = True     # skip layers' dense attention on a side stream, concurrent with the search
    cuda_graph: bool = False       # replay captured decode steps (metrics=False steps)
    # rotation steps as one launch (icb_step_attend: rotate + append + search +
    # attend per tree).  Off: measured slower at C2 (1.38 vs 1.15 ms per
    # rotation step), the inserts lose issue slots to co-resident
    # search CTAs
    fuse_rotation: bool = False
    # BASELINE config 3: indexed layers' page K/V in pinned host memory, each
    # step's pages gathered into a per-tree HBM pool (TierStore,
    # pagestore.py:117-215); sink / window / skip layers stay resident
    kv_offload: bool = False

    def __post_init__(self) -> None:
        if min(self.layers, self.kv_heads, self.query_heads_per_group, self.d, self.d_prime) < 1:
            raise ConfigError("layers, head counts and dims must be >= 1")
        if self.page_size < 2:
            raise ConfigError("page_size must be >= 2")
        if self.token_budget < 1:
            raise ConfigError("token_budget must be >= 1")
        if not 0.0 < self.promotion_ratio < 1.0:
            raise ConfigError("promotion_ratio must lie in (0, 1)")
        if self.sink_pages < 1 or self.window_pages < 1:
            raise ConfigError("sink_pages and window_pages must be >= 1")
        if self.skip_layers < 0:
            raise ConfigError("skip_layers must be >= 0")
        if self.reuse_stride == 1 or self.reuse_stride < 0:
            raise ConfigError("reuse_stride must be 0 (off) or >= 2")
        if self.workers < 1:
            raise ConfigError("workers must be >= 1")
        if self.scalar_bytes < 1:
            raise ConfigError("scalar_bytes must be >= 1")
        if self.kv_dtype not in ("fp32", "bf16"):
            raise ConfigError("kv_dtype must be fp32 or bf16")
        if self.kv_offload and self.fuse_rotation:
            raise ConfigError("kv_offload does not combine with fuse_rotation (the fused step would read host "
                              "rows it wrote in the same launch)")

    @property
    def n_query_heads(self) -> int:
        return self.kv_heads * self.query_heads_per_group

    def budget(self):
        """engine.py:97-98: the decode SearchBudget."""
        from .dci import SearchBudget
        return SearchBudget.for_k(self.token_budget, self.beam, self.visit_cap)

    def head_groups(self):
        """engine.py:100-103."""
        from .attention import HeadGroup
        g = self.query_heads_per_group
        return [HeadGroup(h, tuple(range(h * g, (h + 1) * g))) for h in range(self.kv_heads)]


@dataclass
class StepMetrics:
    """engine.py:95-111 (oracle-only fields keep their defaults unless evaluate)."""

    step: int
    token_id: int
    recall_at_k: float
    page_hit_rate: float
    covered_attention_mass: float
    approx_rel_error: float
    pages_selected: int
    pages_loaded: int
    tokens_loaded: int
    bytes_moved: int
    transactions: int
    dci_queries: int
    baseline_hit_rate: float | None = None


def _dev(x, device, dtype=torch.float32):
    return torch.as_tensor(x, dtype=dtype, device=device)


def _on_device(x, device):
    dev = torch.device(device)
    if isinstance(x, torch.Tensor) and x.is_floating_point() and x.device.type == dev.type and \
            (dev.index is None or x.device.index == dev.index):
        return x
    return torch.as_tensor(x, dtype=torch.float32, device=device)


def _budget_tuple(b):
    """A SearchBudget (dci.py:50-74) or a (k, beam, visit_cap) tuple."""
    if hasattr(b, "visit_cap"):
        return int(b.k), int(b.beam), int(b.visit_cap)
    return tuple(int(x) for x in b)


class Engine:
    def __init__(self, cfg: EngineConfig, device=None):
        self.cfg = cfg
        self.device = torch.device(device or "cuda")
        self.prefilled = False
        self.fallback = False
        self.n_prefill = 0
        self.steps_done = 0
        self.sink_tokens: list[int] = []
        self.indexed_tokens: list[int] = []
        self.selection_queries = 0
        self.forest: DeviceForest | None = None
        self._win_fills: list[int] = []
        self.last_pages = None
        self.last_npages = None
        self._side = None
        self._graphs = {}
        self._warmed = set()
        self._gbuf = None
        self._io = None
        self._cum_stats = None     # [T, 5] host: residency counters summed over metric steps
        self._baseline_hit = None  # TokenOrderBaseline hit rate of the last evaluated step
        self._anchor_tokens: dict[int, list[int]] = {}

    # -- prefill ---------------------------------------------------------------
    def prefill(self, workload, n_prefill, *more) -> "Engine":
        """engine.py:226-301.  Reference form: prefill(workload, n_prefill) with
        a Workload (this package's or the reference's: anything with `spec`
        and `prefill_view`).  Array form: prefill(keys [n, L, H, d],
        values [n, L, H, d'], n_prefill) (numpy or tensors; only the first
        n_prefill tokens are read)."""
        if self.prefilled:
            raise ConfigError("engine already prefilled")
        if hasattr(workload, "prefill_view"):
            if more:
                raise InputError("prefill(workload, n_prefill) takes no further arguments")
            self._check_workload(workload)
            if n_prefill < 1:
                raise ConfigError("prefill needs at least one token")
            keys, values = workload.prefill_view(n_prefill)
        else:
            if len(more) != 1:
                raise InputError("prefill(keys, values, n_prefill) or prefill(workload, n_prefill)")
            keys, values, n_prefill = workload, n_prefill, more[0]
        if n_prefill < 1:
            raise ConfigError("prefill needs at least one token")
        cfg = self.cfg
        # device tensors keep their dtype (an fp32 / bf16 stream is converted per
        # chunk of layers, never materialised whole in fp32); numpy / host -> fp32
        keys = _on_device(keys[:n_prefill], self.device)
        values = _on_device(values[:n_prefill], self.device)
        if tuple(keys.shape[1:]) != (cfg.layers, cfg.kv_heads, cfg.d) or \
                tuple(values.shape[1:]) != (cfg.layers, cfg.kv_heads, cfg.d_prime):
            raise ConfigError("workload dims do not match the engine config")
        geo = self._prefill_begin(n_prefill)
        for layer in range(cfg.layers):
            self._store_layer(layer, keys[:, layer], values[:, layer])
        if not self.fallback:
            try:
                self._new_forest(geo, tight=True)
                self._build_layers(geo, cfg.skip_layers, cfg.layers, keys[:, cfg.skip_layers:],
                                   values[:, cfg.skip_layers:])
                self.forest.check()
            except ConfigError as e:
                if "page capacity" not in str(e):
                    raise
                # the trees outgrew the tight page estimate: rebuild at the worst case
                self.forest.close()
                self._new_forest(geo, tight=False)
                self._build_layers(geo, cfg.skip_layers, cfg.layers, keys[:, cfg.skip_layers:],
                                   values[:, cfg.skip_layers:])
                self.forest.check()
        return self._prefill_end()

    def prefill_layers(self, n_prefill: int, group: int = 4) -> "LayerPrefill":
        """Layer-streaming prefill: hand each layer's prompt K/V to the engine
        as the model produces it; that layer's trees build on the engine's own
        CUDA stream while the caller computes the next layer (the pipelined
        prefill of PAPER.md:245-249 / engine.py:587-604, here real overlap on
        the device).  Same trees as prefill(keys, values, n).

            with torch.no_grad():
                pf = eng.prefill_layers(n)
                for layer in range(L):
                    k, v = ...            # [n, kv_heads, d] / [n, kv_heads, d'] on the device
                    pf.layer(layer, k, v)
                pf.finish()
        """
        if self.prefilled:
            raise ConfigError("engine already prefilled")
        if n_prefill < 1:
            raise ConfigError("prefill needs at least one token")
        return LayerPrefill(self, n_prefill, group)

    def _prefill_begin(self, n_prefill):
        """Shapes, dense / evaluation mirrors and the page layout of a prefill
        of n_prefill tokens (engine.py:240-276); returns the sink / window
        geometry."""
        cfg, dev = self.cfg, self.device
        self.n_prefill = n_prefill
        self.max_tokens = cfg.max_tokens or (n_prefill + 1024)
        s = cfg.page_size
        pages = math.ceil(n_prefill / s)
        self.fallback = pages < cfg.sink_pages + cfg.window_pages + 1 or cfg.skip_layers >= cfg.layers
        self.n_dense = cfg.layers if self.fallback else cfg.skip_layers
        kvt = torch.bfloat16 if cfg.kv_dtype == "bf16" else torch.float32
        # dense mirror of skip layers (or every layer in fallback): [L_dense*H, max_tokens, d]
        dpad = (cfg.d + 3) // 4 * 4
        dvpad = (cfg.d_prime + 3) // 4 * 4
        nd = self.n_dense * cfg.kv_heads
        self._tok_dev = torch.zeros(1, dtype=torch.int32, device=dev)   # decode position on the device
        if cfg.evaluate:
            # exact-reference mirrors of every layer (engine.py:536-566, _full_reference)
            self._mk = torch.zeros((cfg.layers, cfg.kv_heads, self.max_tokens, cfg.d), dtype=torch.float32, device=dev)
            self._mv = torch.zeros((cfg.layers, cfg.kv_heads, self.max_tokens, cfg.d_prime), dtype=torch.float32,
                                   device=dev)
            self._indexed_mask = torch.zeros(self.max_tokens, dtype=torch.bool, device=dev)
        self._dense_res = torch.empty((max(nd, 1), cfg.query_heads_per_group, cfg.d_prime), dtype=torch.float32,
                                      device=dev)   # dense attention output (nd planes)
        self.dense_k = torch.zeros((max(nd, 1), self.max_tokens, dpad), dtype=kvt, device=dev)
        self.dense_v = torch.zeros((max(nd, 1), self.max_tokens, dvpad), dtype=kvt, device=dev)
        if self.fallback:
            return None
        sink_end = cfg.sink_pages * s
        win_start = (pages - cfg.window_pages) * s
        self.sink_tokens = list(range(sink_end))
        self.indexed_tokens = list(range(sink_end, win_start))
        if cfg.evaluate:
            self._indexed_mask[sink_end:win_start] = True
        self.T = (cfg.layers - cfg.skip_layers) * cfg.kv_heads
        # KV offload: the pool holds a step's sink, window and largest selection
        pool = (cfg.query_heads_per_group * min(cfg.token_budget, self.max_tokens) + cfg.sink_pages
                + cfg.window_pages + 2)
        self.trees_dev = torch.arange(self.T, dtype=torch.int32, device=dev)
        self._win_fills = [min(s, max(0, (n_prefill - win_start) - i * s)) for i in range(cfg.window_pages)]
        self._win_start = [win_start + i * s for i in range(cfg.window_pages)]
        return dict(n=n_prefill, sink_end=sink_end, win_start=win_start, pool=pool)

    def _store_layer(self, layer, k, v):
        """One layer's prompt K/V [n, H, d] into the dense mirror (dense
        layers) and the evaluation mirrors."""
        cfg = self.cfg
        n = self.n_prefill
        if cfg.evaluate:
            self._mk[layer, :, :n] = k.permute(1, 0, 2).float()
            self._mv[layer, :, :n] = v.permute(1, 0, 2).float()
        if layer < self.n_dense:
            H = cfg.kv_heads
            self.dense_k[layer * H:(layer + 1) * H, :n, : cfg.d] = k.permute(1, 0, 2).to(self.dense_k.dtype)
            self.dense_v[layer * H:(layer + 1) * H, :n, : cfg.d_prime] = v.permute(1, 0, 2).to(self.dense_v.dtype)

    def _new_forest(self, geo, tight):
        cfg, dev, T, H, s = self.cfg, self.device, self.T, self.cfg.kv_heads, self.cfg.page_size
        caps = ForestCaps.for_stream(geo["win_start"] - geo["sink_end"], self.max_tokens - geo["n"],
                                     cfg.promotion_ratio, s, cfg.sink_pages + cfg.window_pages, tight=tight)
        caps.tok_cap = self.max_tokens
        self.forest = f = DeviceForest(T, cfg.d, cfg.d_prime, tok_cap=self.max_tokens,
                                       promotion_ratio=cfg.promotion_ratio, page_size=s, kv_dtype=cfg.kv_dtype,
                                       device=dev, kv_host=cfg.kv_offload,
                                       pool_pages=geo["pool"] if cfg.kv_offload else 0, caps=caps)
        trees = list(range(T))
        f.seed(trees, [(cfg.seed, cfg.skip_layers + t // H, t % H) for t in trees])
        self._tok_ar = torch.arange(geo["n"], dtype=torch.int32, device=dev)

    def _build_layers(self, geo, la, lb, keys, values):
        """Trees of indexed layers [la, lb) from their prompt K/V ([n, lb - la,
        H, d]): sink and window pages, then dci_indexing (engine.py:254-281), in
        chunks of whole layers (~2 GB of fp32 keys + values at a time)."""
        cfg, H, f = self.cfg, self.cfg.kv_heads, self.forest
        n, sink_end, win_start = geo["n"], geo["sink_end"], geo["win_start"]
        tok = self._tok_ar
        per_layer = H * n * (cfg.d + cfg.d_prime) * 4
        lchunk = max(1, min(lb - la, (2 << 30) // max(1, per_layer)))
        for l0 in range(la, lb, lchunk):
            l1 = min(lb, l0 + lchunk)
            c0, c1 = (l0 - cfg.skip_layers) * H, (l1 - cfg.skip_layers) * H
            trs = self.trees_dev[c0:c1]
            ki = keys[:, l0 - la:l1 - la].permute(1, 2, 0, 3).reshape(c1 - c0, n, cfg.d)
            vi = values[:, l0 - la:l1 - la].permute(1, 2, 0, 3).reshape(c1 - c0, n, cfg.d_prime)
            # pages: sink ids 0.., window next, then indexed (engine.py:263-281)
            f.alloc_resident(trs, N.ROLE_SINK, cfg.sink_pages, tok[:sink_end].expand(c1 - c0, -1),
                             ki[:, :sink_end], vi[:, :sink_end])
            f.alloc_resident(trs, N.ROLE_WINDOW, cfg.window_pages, tok[win_start:].expand(c1 - c0, -1),
                             ki[:, win_start:], vi[:, win_start:])
            f.build(trs, tok[sink_end:win_start].expand(c1 - c0, -1), ki[:, sink_end:win_start],
                    vi[:, sink_end:win_start])
            del ki, vi

    def _prefill_end(self):
        cfg = self.cfg
        if not self.fallback:
            f = self.forest
            k, beam, cap = _budget_tuple(cfg.budget())
            self.k_eff = int(min(k, self.max_tokens))
            self.beam, self.visit_cap = int(min(beam, 2**62)), int(min(cap, 2**62))
            G = cfg.query_heads_per_group
            self.pages_cap = int(min(f.caps.page_cap, G * self.k_eff))
            if cfg.reuse_stride >= 2 and cfg.layer_serial:
                raise ConfigError("reuse_stride is supported with layers batched per step (layer_serial=False)")
            self._alloc_step_buffers()
        self.prefilled = True
        return self

    def _check_workload(self, workload) -> None:
        """engine.py:216-224."""
        spec, cfg = workload.spec, self.cfg
        if (spec.layers, spec.kv_heads, spec.query_heads_per_group) != \
                (cfg.layers, cfg.kv_heads, cfg.query_heads_per_group):
            raise ConfigError("workload head/layer shape does not match the engine config")
        if (spec.d, spec.d_prime) != (cfg.d, cfg.d_prime):
            raise ConfigError("workload dims do not match the engine config")

    def _alloc_step_buffers(self):
        cfg, dev, T = self.cfg, self.device, self.T
        G = cfg.query_heads_per_group
        self.ids = torch.empty((T, G, self.k_eff), dtype=torch.int32, device=dev)
        self.counts = torch.empty((T, G), dtype=torch.int32, device=dev)
        self.pages = torch.empty((T, max(1, self.pages_cap)), dtype=torch.int32, device=dev)
        self.npages = torch.empty((T,), dtype=torch.int32, device=dev)
        self.stats = torch.zeros((T, 5), dtype=torch.int64, device=dev)
        self.rot_stats = torch.zeros((T, 2), dtype=torch.int64, device=dev)
        # per-step outputs live in fixed buffers (no allocation on the step path)
        self._attn_out = torch.empty((T, G, cfg.d_prime), dtype=torch.float32, device=dev)
        if cfg.reuse_stride >= 2:
            # selection reuse (engine.py:321-363): anchor trees are searched,
            # the others map their anchor's tokens through their own pages
            H = cfg.kv_heads
            anchors = [t for t in range(T) if self.is_anchor_layer(cfg.skip_layers + t // H)]
            reuse = [t for t in range(T) if t not in set(anchors)]
            src = [((t // H) // cfg.reuse_stride * cfg.reuse_stride) * H + t % H for t in reuse]
            ix = lambda v: torch.tensor(v, dtype=torch.int64, device=dev)   # noqa: E731
            self._anchor_rows, self._reuse_rows = ix(anchors), ix(reuse)
            self._anchor_trees = self.trees_dev[self._anchor_rows].contiguous()
            self._reuse_trees = self.trees_dev[self._reuse_rows].contiguous()
            self._reuse_src = torch.tensor(src, dtype=torch.int32, device=dev)
            nA, nR = len(anchors), len(reuse)
            self._ids_a = torch.empty((nA, G, self.k_eff), dtype=torch.int32, device=dev)
            self._counts_a = torch.empty((nA, G), dtype=torch.int32, device=dev)
            self._pages_a = torch.empty((nA, max(1, self.pages_cap)), dtype=torch.int32, device=dev)
            self._npages_a = torch.empty((nA,), dtype=torch.int32, device=dev)
            self._pages_r = torch.empty((max(1, nR), max(1, self.pages_cap)), dtype=torch.int32, device=dev)
            self._npages_r = torch.empty((max(1, nR),), dtype=torch.int32, device=dev)

    # -- selection -------------------------------------------------------------
    def is_anchor_layer(self, layer: int) -> bool:
        """engine.py:321-325."""
        if self.cfg.reuse_stride < 2:
            raise ConfigError("selection reuse is disabled")
        return layer >= self.cfg.skip_layers and (layer - self.cfg.skip_layers) % self.cfg.reuse_stride == 0

    def anchor_layers(self) -> list[int]:
        """engine.py:327-329."""
        return [l for l in range(self.cfg.skip_layers, self.cfg.layers) if self.is_anchor_layer(l)]

    def _queries_per_step(self) -> int:
        G = self.cfg.query_heads_per_group
        if self.cfg.reuse_stride >= 2:
            return len(self.anchor_layers()) * self.cfg.kv_heads * G
        return self.T * G

    def page_select(self, q, layer: int, kv_head: int, budget=None) -> list[int]:
        """Pages holding the tree's top-budget tokens for one query
        (engine.py:305-310): the search kernel's page epilogue
        (find_page_index on the device)."""
        return self._select(q, layer, kv_head, budget)[1]

    def select_tokens(self, q, layer: int, kv_head: int, budget=None) -> list[int]:
        """engine.py:312-319 (_select_tokens): the ranked top-k token ids."""
        return self._select(q, layer, kv_head, budget)[0]

    _select_tokens = select_tokens

    def _select(self, q, layer, kv_head, budget):
        t = self._tree(layer, kv_head)
        k, beam, cap = _budget_tuple(budget if budget is not None else self.cfg.budget())
        self.selection_queries += 1
        q = _dev(q, self.device).reshape(1, 1, self.cfg.d)
        k_out = int(min(k, self.forest.caps.tok_cap))
        ids, counts, pages, npages = self.forest.query([t], q, k, beam, cap, k_out=k_out, pages_cap=k_out)
        self.forest.check()
        return ([int(x) for x in ids[0, 0, : int(counts[0, 0])].cpu().tolist()],
                [int(x) for x in pages[0, : int(npages[0])].cpu().tolist()])

    def token_census(self, layer: int, kv_head: int) -> int:
        """engine.py:568-575: tokens across the tree's sink, window and indexed pages."""
        ex = self.forest.export(self._tree(layer, kv_head))
        return sum(len(toks) for _, toks in ex["pages"].values())

    def _tree(self, layer, kv_head):
        if self.fallback or layer < self.cfg.skip_layers or layer >= self.cfg.layers:
            raise ConfigError(f"no tree for layer {layer}, head {kv_head}")
        return (layer - self.cfg.skip_layers) * self.cfg.kv_heads + kv_head

    # -- decode ------------------------------------------------------------------
    def rotation_due(self) -> bool:
        """engine.py:408-411: newest window page at fill >= s - 1."""
        return (not self.fallback) and self._win_fills[-1] >= self.cfg.page_size - 1

    def decode_step(self, token_id, queries=None, keys=None, values=None, *, metrics: bool = True, out=None):
        """One decode token through every layer (engine.py:383-514).

        Reference form: decode_step(step) with a DecodeStep (anything with
        token_id / queries / keys / values) returns (outputs, StepMetrics)
        with outputs[layer][query head] an AttentionOutput (weights over the
        attended tokens in entry order, value_out) as the reference does.

        Array form: decode_step(token_id, queries, keys, values).
        queries [L, Hq, d], keys [L, H, d], values [L, H, d'] (device tensors,
        or host tensors: staged through a copy stream, overlapping the previous
        step's compute).  Returns (outputs [L, Hq, d'] fp32, StepMetrics |
        None).  With EngineConfig.cuda_graph and metrics=False the step is a
        replay of a captured graph and the returned device tensor is the
        engine's static output buffer (valid until the next step).  `out`: a
        device tensor receives a copy; a host (pinned) tensor is filled
        asynchronously on the copy stream (synchronize before reading it) and
        is returned."""
        if queries is None and hasattr(token_id, "token_id"):
            return self._decode_reference(token_id)
        if not self.prefilled:
            raise ConfigError("decode_step before prefill")
        cfg = self.cfg
        token = self.n_prefill + self.steps_done
        if token_id != token:
            raise InputError(f"stream misaligned: expected token {token}, got {token_id}")
        if token >= self.max_tokens:
            raise ConfigError("token capacity exhausted (raise EngineConfig.max_tokens)")
        dev = self.device
        rotate = self.rotation_due()
        L, H, G = cfg.layers, cfg.kv_heads, cfg.query_heads_per_group
        self._tok_dev.fill_(token)
        graph = cfg.cuda_graph and not metrics and dev.type == "cuda"
        host_in = dev.type == "cuda" and any(isinstance(x, torch.Tensor) and x.device.type == "cpu"
                                             for x in (queries, keys, values))
        host_out = out is not None and out.device.type == "cpu"
        if host_in:
            queries, keys, values, slot = self._stage_in(queries, keys, values)
        if graph:
            res = self._graph_step(rotate, queries, keys, values)
            if cfg.evaluate:
                self._mk[:, :, token] = self._gbuf["k"]
                self._mv[:, :, token] = self._gbuf["v"]
        else:
            q = _dev(queries, dev)
            kk = _dev(keys, dev)
            vv = _dev(values, dev)
            res = out if (out is not None and not host_out) else \
                torch.empty((L, H * G, cfg.d_prime), dtype=torch.float32, device=dev)
            if metrics and not self.fallback:
                self.stats.zero_()
            if cfg.evaluate:
                self._mk[:, :, token] = kk
                self._mv[:, :, token] = vv
            self._device_step(q, kk, vv, rotate, res)
            if not self.fallback:
                self._warmed.add(bool(rotate))
        if host_in:
            self._io["in_free"][slot].record(torch.cuda.current_stream(dev))
        if host_out:
            res = self._stage_out(res, out)
        elif graph and out is not None:
            out.copy_(res)
            res = out
        if not self.fallback:
            self.selection_queries += self._queries_per_step()
            if rotate:
                start, fill = self._win_start[0], self._win_fills[0]
                self.indexed_tokens.extend(range(start, start + fill))
                if cfg.evaluate:
                    self._indexed_mask[start:start + fill] = True
                self._win_fills = self._win_fills[1:] + [0]
                self._win_start = self._win_start[1:] + [token]
            i = next(j for j, fl in enumerate(self._win_fills) if fl < cfg.page_size)
            if self._win_fills[i] == 0:
                self._win_start[i] = token
            self._win_fills[i] += 1
        self.steps_done += 1
        m = None
        if metrics:
            m = self._metrics(token)
            if cfg.evaluate and not self.fallback and not graph:
                rec, hit, mass, rel = self._evaluate(token, q, res)
                m.recall_at_k, m.page_hit_rate, m.covered_attention_mass, m.approx_rel_error = rec, hit, mass, rel
                m.baseline_hit_rate = self._baseline_hit
        return res, m

    def _decode_reference(self, step):
        """decode_step(DecodeStep) -> (list[list[AttentionOutput]], StepMetrics):
        the device step, then every query head's output with its weights
        (icb_attention_weights over the attended set in entry order;
        icb_dense_weights over all tokens for dense layers)."""
        from .attention import AttentionOutput
        if not self.prefilled:
            raise ConfigError("decode_step before prefill")
        cfg, dev = self.cfg, self.device
        L, H, G = cfg.layers, cfg.kv_heads, cfg.query_heads_per_group
        q = _dev(np.asarray(step.queries, dtype=np.float64), dev).reshape(L, H * G, cfg.d)
        res, m = self.decode_step(int(step.token_id), q, np.asarray(step.keys, dtype=np.float64),
                                  np.asarray(step.values, dtype=np.float64))
        token = int(step.token_id)
        vals = res.double().cpu().numpy()
        outs: list[list] = [[None] * (H * G) for _ in range(L)]
        nd = self.n_dense
        if nd:
            ntok = token + 1
            w = torch.empty((nd * H, G, ntok), dtype=torch.float64, device=dev)
            qd = q[:nd].reshape(nd * H, G, cfg.d).contiguous()
            kvd = N.KV_BF16 if self.dense_k.dtype == torch.bfloat16 else N.KV_F32
            N.check(N.lib().icb_dense_weights(nd * H, G, cfg.d, kvd, _ptr(qd), _ptr(self.dense_k),
                                              self.dense_k.shape[1], ntok, _ptr(w), _stream()))
            wn = w.cpu().numpy()
            for layer in range(nd):
                for qh in range(H * G):
                    row = wn[layer * H + qh // G, qh % G]
                    outs[layer][qh] = AttentionOutput(dict(enumerate(row.tolist())), vals[layer, qh])
        if not self.fallback:
            s0, T = cfg.skip_layers, self.T
            f = self.forest
            cap = (cfg.sink_pages + cfg.window_pages + self.pages.shape[1]) * cfg.page_size
            toks = torch.empty((T, cap), dtype=torch.int32, device=dev)
            w = torch.empty((T, G, cap), dtype=torch.float64, device=dev)
            cnt = torch.empty((T,), dtype=torch.int32, device=dev)
            qi = q[s0:].reshape(T, G, cfg.d).contiguous()
            N.check(N.lib().icb_attention_weights(f.h, _ptr(self.trees_dev), T, G, _ptr(qi), _ptr(self.pages),
                                                  self.pages.shape[1], _ptr(self.npages), _ptr(toks), _ptr(w), cap,
                                                  _ptr(cnt), _stream()))
            toks, w, cnt = toks.cpu().numpy(), w.cpu().numpy(), cnt.cpu().numpy()
            for t in range(T):
                layer, h = s0 + t // H, t % H
                n = min(int(cnt[t]), cap)
                ids = toks[t, :n].tolist()
                for g in range(G):
                    outs[layer][h * G + g] = AttentionOutput(dict(zip(ids, w[t, g, :n].tolist())),
                                                             vals[layer, h * G + g])
        return outs, m

    def _device_step(self, q, kk, vv, rotate, out):
        """All device work of one step (capturable: the position comes from
        self._tok_dev, every buffer is static)."""
        cfg, dev = self.cfg, self.device
        overlap = cfg.overlap_dense and not self.fallback and self.n_dense > 0 and dev.type == "cuda"
        if not overlap:
            self._dense_part(q, kk, vv, out)
            dense_hook = None
        else:
            # The skip layers' dense attention depends only on this step's
            # inputs: it runs on a side stream, issued right after the search
            # kernel so its CTAs fill the SMs the search leaves idle (the
            # search runs one CTA per tree, two per SM at most).
            # The side stream forks after the window append, the search kernel's
            # own predecessor, and its work is issued after the search launch:
            # in eager order and in a captured graph alike the search's CTAs
            # are dispatched first and the dense CTAs fill what is left.
            main = torch.cuda.current_stream(dev)
            if self._side is None:
                self._side = torch.cuda.Stream(device=dev)
            ready, done = torch.cuda.Event(), torch.cuda.Event()

            def fork():
                ready.record(main)

            def dense_hook():
                self._side.wait_event(ready)
                with torch.cuda.stream(self._side):
                    self._dense_part(q, kk, vv, out)
                done.record(self._side)
        if not self.fallback:
            self._indexed_part(q, kk, vv, rotate, out, dense_hook, fork if overlap else None)
            if overlap:
                main.wait_event(done)

    def _io_init(self):
        cfg, dev = self.cfg, self.device
        L, H, G = cfg.layers, cfg.kv_heads, cfg.query_heads_per_group
        shapes = dict(q=(L, H * G, cfg.d), k=(L, H, cfg.d), v=(L, H, cfg.d_prime))
        self._io = dict(
            h2d=torch.cuda.Stream(device=dev), d2h=torch.cuda.Stream(device=dev),
            stage=[{n: torch.empty(sh, dtype=torch.float32, device=dev) for n, sh in shapes.items()}
                   for _ in range(2)],
            outbuf=[torch.empty((L, H * G, cfg.d_prime), dtype=torch.float32, device=dev) for _ in range(2)],
            in_ready=[torch.cuda.Event() for _ in range(2)], in_free=[torch.cuda.Event() for _ in range(2)],
            out_ready=[torch.cuda.Event() for _ in range(2)], out_done=[torch.cuda.Event() for _ in range(2)],
            n_in=0, n_out=0)

    def _stage_in(self, queries, keys, values):
        """H2D of host inputs on the input copy stream into one of two device slots
        (the slot's previous step must have consumed it)."""
        if self._io is None:
            self._io_init()
        io = self._io
        slot = io["n_in"] % 2
        io["n_in"] += 1
        cs, main = io["h2d"], torch.cuda.current_stream(self.device)
        st = io["stage"][slot]
        cs.wait_event(io["in_free"][slot])
        with torch.cuda.stream(cs):
            st["q"].copy_(torch.as_tensor(queries).reshape(st["q"].shape), non_blocking=True)
            st["k"].copy_(torch.as_tensor(keys).reshape(st["k"].shape), non_blocking=True)
            st["v"].copy_(torch.as_tensor(values).reshape(st["v"].shape), non_blocking=True)
        io["in_ready"][slot].record(cs)
        main.wait_event(io["in_ready"][slot])
        return st["q"], st["k"], st["v"], slot

    def _stage_out(self, res, out_host):
        """D2H of the step's output on the output copy stream from a rotating device
        buffer, so the copy never blocks the next step's compute."""
        if self._io is None:
            self._io_init()
        io = self._io
        slot = io["n_out"] % 2
        io["n_out"] += 1
        cs, main = io["d2h"], torch.cuda.current_stream(self.device)
        buf = io["outbuf"][slot]
        main.wait_event(io["out_done"][slot])
        buf.copy_(res)
        io["out_ready"][slot].record(main)
        cs.wait_event(io["out_ready"][slot])
        with torch.cuda.stream(cs):
            out_host.copy_(buf, non_blocking=True)
        io["out_done"][slot].record(cs)
        return out_host

    def _graph_buffers(self):
        cfg, dev = self.cfg, self.device
        L, H, G = cfg.layers, cfg.kv_heads, cfg.query_heads_per_group
        if self._gbuf is None:
            self._gbuf = dict(q=torch.empty((L, H * G, cfg.d), dtype=torch.float32, device=dev),
                              k=torch.empty((L, H, cfg.d), dtype=torch.float32, device=dev),
                              v=torch.empty((L, H, cfg.d_prime), dtype=torch.float32, device=dev),
                              out=torch.empty((L, H * G, cfg.d_prime), dtype=torch.float32, device=dev))
        return self._gbuf

    def _capture(self, key):
        b = self._graph_buffers()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            self._device_step(b["q"], b["k"], b["v"], key, b["out"])
        self._graphs[key] = g

    def capture_graphs(self) -> None:
        """Capture both decode-step variants (plain, rotating) as CUDA graphs
        without running them, so no later step pays a capture.  Each variant
        must have run once (eagerly or replayed) so every lazily allocated
        scratch exists."""
        if not self.cfg.cuda_graph:
            raise ConfigError("capture_graphs needs EngineConfig.cuda_graph")
        if self.fallback:
            raise ConfigError("fallback engines run no graph-captured step")
        if {False, True} - self._warmed:
            raise ConfigError("run a plain and a rotating step before capture_graphs()")
        for key in (False, True):
            if key not in self._graphs:
                self._capture(key)

    def _graph_step(self, rotate, queries, keys, values):
        b = self._graph_buffers()
        b["q"].copy_(torch.as_tensor(queries), non_blocking=True)
        b["k"].copy_(torch.as_tensor(keys), non_blocking=True)
        b["v"].copy_(torch.as_tensor(values), non_blocking=True)
        key = bool(rotate)
        g = self._graphs.get(key)
        if g is None and key in self._warmed:
            # second occurrence of this step variant: every lazily allocated
            # scratch exists (first occurrence ran eagerly) -> capture
            self._capture(key)
            g = self._graphs[key]
        if g is None:
            self._warmed.add(key)
            self._device_step(b["q"], b["k"], b["v"], rotate, b["out"])
        else:
            g.replay()
        return b["out"]

    def _dense_part(self, q, kk, vv, out, splits=0):
        cfg = self.cfg
        nd = self.n_dense
        if nd == 0:
            return
        H, G = cfg.kv_heads, cfg.query_heads_per_group
        dense_append(kk[:nd].reshape(nd * H, cfg.d), vv[:nd].reshape(nd * H, cfg.d_prime), self.dense_k,
                     self.dense_v, self._tok_dev)
        qd = q[:nd].reshape(nd * H, G, cfg.d)
        # logits scaled by 1/sqrt(d) with the unpadded d (attention.py:70)
        res = dense_attention(qd.contiguous(), self.dense_k, self.dense_v, self._tok_dev, splits=splits,
                              out=self._dense_res[: nd * H], dim_v=cfg.d_prime)
        out[:nd] = res.reshape(nd, H * G, cfg.d_prime)

    def _indexed_part(self, q, kk, vv, rotate, out, after_query=None, before_query=None):
        cfg, f = self.cfg, self.forest
        s0, H, G = cfg.skip_layers, cfg.kv_heads, cfg.query_heads_per_group
        T = self.T
        qi = q[s0:].reshape(T, G, cfg.d)
        ki = kk[s0:].reshape(T, cfg.d)
        vi = vv[s0:].reshape(T, cfg.d_prime)
        k = self.k_eff
        groups = [(0, T)] if not cfg.layer_serial else [(l * H, (l + 1) * H) for l in range(T // H)]
        for a, b in groups:
            trees = self.trees_dev[a:b]
            fused_step = rotate and cfg.fuse_rotation and cfg.reuse_stride < 2
            if fused_step:
                # rotation, window append, search and attention of each tree in
                # one CTA (icb_step_attend): the slowest tree's rotation no
                # longer holds back every other tree's search
                if before_query is not None:
                    before_query()
                    before_query = None
                o = f.step_attend(trees, qi[a:b], k, self.beam, self.visit_cap,
                                  out=(self.ids[a:b], self.counts[a:b], self.pages[a:b], self.npages[a:b]),
                                  attn_out=self._attn_out[a:b], token_dev=self._tok_dev, keys=ki[a:b],
                                  values=vi[a:b], rotate=True, rot_stats=self.rot_stats[a:b],
                                  stats=self.stats[a:b], scalar_bytes=cfg.scalar_bytes)
                if after_query is not None:
                    after_query()
                    after_query = None
                out[s0 + a // H: s0 + b // H] = o.reshape((b - a) // H, H * G, cfg.d_prime)
                continue
            if rotate:
                f.rotate_window(trees, cfg.scalar_bytes, self.rot_stats[a:b])
            f.append_window(trees, self._tok_dev, ki[a:b], vi[a:b])
            if before_query is not None:
                before_query()
                before_query = None
            if cfg.reuse_stride >= 2:
                self._select_with_reuse(qi)
                if after_query is not None:
                    after_query()
                    after_query = None
                o = f.attention(trees, qi[a:b], self.pages[a:b], self.npages[a:b], stats=self.stats[a:b],
                                scalar_bytes=cfg.scalar_bytes, out=self._attn_out[a:b])
            else:
                # selection + sparse attention fused: each tree's CTA attends its
                # pages right after its search (icb_query_attend)
                o = f.query_attend(trees, qi[a:b], k, self.beam, self.visit_cap,
                                   out=(self.ids[a:b], self.counts[a:b], self.pages[a:b], self.npages[a:b]),
                                   attn_out=self._attn_out[a:b], stats=self.stats[a:b],
                                   scalar_bytes=cfg.scalar_bytes)
                if after_query is not None:
                    after_query()
                    after_query = None
            out[s0 + a // H: s0 + b // H] = o.reshape((b - a) // H, H * G, cfg.d_prime)

    def _select_with_reuse(self, qi):
        """engine.py:331-363, all layers of the step at once: anchors' searches,
        then every other layer's pages from its anchor's token lists."""
        f, k = self.forest, self.k_eff
        f.query(self._anchor_trees, qi.index_select(0, self._anchor_rows), k, self.beam, self.visit_cap, k_out=k,
                pages_cap=self.pages_cap, out=(self._ids_a, self._counts_a, self._pages_a, self._npages_a))
        self.ids.index_copy_(0, self._anchor_rows, self._ids_a)
        self.counts.index_copy_(0, self._anchor_rows, self._counts_a)
        self.pages.index_copy_(0, self._anchor_rows, self._pages_a)
        self.npages.index_copy_(0, self._anchor_rows, self._npages_a)
        nR = self._reuse_rows.numel()
        if nR:
            f.pages_from_tokens(self._reuse_trees, self._reuse_src, self.ids, self.counts, self._pages_r[:nR],
                                self._npages_r[:nR])
            self.pages.index_copy_(0, self._reuse_rows, self._pages_r[:nR])
            self.npages.index_copy_(0, self._reuse_rows, self._npages_r[:nR])

    def _evaluate(self, token, q, out):
        """_evaluate_head (engine.py:536-566) for every indexed layer and query
        head, on the device in fp64: recall of the exact top-k over indexed
        tokens (exact_topk, geometry.py:107-126: descending score, ties to the
        smaller token), hit rate of the exact top-k over all tokens in the
        attended set, covered attention mass, relative output error; averaged
        over heads."""
        cfg, dev = self.cfg, self.device
        H, G, d = cfg.kv_heads, cfg.query_heads_per_group, cfg.d
        n = token + 1
        att = self.forest.attended_mask(self.trees_dev, self.pages, self.npages,
                                        torch.empty((self.T, self.forest.caps.tok_cap), dtype=torch.uint8,
                                                    device=dev))[:, :n].bool()
        idx_mask = self._indexed_mask[:n]
        k_eff = min(cfg.token_budget, len(self.indexed_tokens))
        k_all = min(cfg.token_budget, n)
        rec, hit, mass, rel, base = [], [], [], [], []
        for layer in range(cfg.skip_layers, cfg.layers):
            li = layer - cfg.skip_layers
            K = self._mk[layer, :, :n].double()
            V = self._mv[layer, :, :n].double()
            ql = q[layer].double().reshape(H, G, d)
            scores = torch.einsum("hnd,hgd->hgn", K, ql)
            w = torch.softmax(scores / (d ** 0.5), dim=-1)
            ref = torch.einsum("hgn,hnv->hgv", w, V)
            order_idx = torch.sort(-scores.masked_fill(~idx_mask, float("-inf")), dim=-1, stable=True).indices
            order_all = torch.sort(-scores, dim=-1, stable=True).indices[..., :k_all]
            # each head's selected tokens (reuse mode: the anchor's group union, engine.py:358-361)
            src = li if cfg.reuse_stride < 2 else (li // cfg.reuse_stride) * cfg.reuse_stride
            sel = torch.zeros((H, G, n + 1), dtype=torch.bool, device=dev)   # column n: padding slots
            ids = self.ids[src * H:(src + 1) * H].long()
            cnt = self.counts[src * H:(src + 1) * H]
            valid = torch.arange(ids.shape[-1], device=dev)[None, None, :] < cnt[..., None]
            if cfg.reuse_stride >= 2:
                # under reuse every layer, anchors included, scores the group's
                # token union (engine.py:346-352, 431-433)
                ids = ids.reshape(H, 1, -1).expand(H, G, -1)
                valid = valid.reshape(H, 1, -1).expand(H, G, -1)
            ok = valid & (ids >= 0) & (ids < n)
            sel.scatter_(-1, torch.where(ok, ids, torch.full_like(ids, n)), ok)
            sel = sel[..., :n]
            a = att[li * H:(li + 1) * H][:, None, :].expand(H, G, n)
            rec.append(sel.gather(-1, order_idx[..., :k_eff]).sum(-1).double() / max(k_eff, 1))
            hit.append(a.gather(-1, order_all).sum(-1).double() / k_all)
            mass.append((w * a).sum(-1))
            o = out[layer].double().reshape(H, G, -1)
            rel.append(torch.linalg.norm(o - ref, dim=-1) / torch.linalg.norm(ref, dim=-1).clamp_min(1e-300))
            if cfg.compare_baseline:
                base.append(self._token_order_hits(layer, li, ql, order_all, k_all, n))
        f = lambda xs: float(torch.cat([x.reshape(-1) for x in xs]).mean())   # noqa: E731
        self._baseline_hit = f(base) if base else None
        return f(rec), f(hit), f(mass), f(rel)

    def _token_order_hits(self, layer, li, ql, order_all, k_all, n):
        """TokenOrderBaseline (engine.py:148-182) for one layer's heads, on the
        device in fp64: indexed tokens in arrival order (prefill middle, then
        each rotated window page) fill pages of s; a page's score for q is
        sum_i max(q_i lo_i, q_i hi_i) over its coordinate envelope; the
        top-n pages (n = the group's selected page count; ties to the older
        page) plus sink and window tokens form the baseline's attended set;
        returns the exact top-k's hit rate in it per head."""
        cfg, dev = self.cfg, self.device
        H, G, s = cfg.kv_heads, cfg.query_heads_per_group, cfg.page_size
        order = torch.as_tensor(self.indexed_tokens, dtype=torch.long, device=dev)
        P = (order.numel() + s - 1) // s
        K = self._mk[layer][:, order].double()                                    # [H, m, d]
        pad = P * s - order.numel()
        lo = torch.cat([K, K[:, -1:].expand(H, pad, -1)], 1).reshape(H, P, s, -1).amin(2)
        hi = torch.cat([K, K[:, -1:].expand(H, pad, -1)], 1).reshape(H, P, s, -1).amax(2)
        sc = torch.maximum(lo[:, None] * ql[:, :, None], hi[:, None] * ql[:, :, None]).sum(-1)   # [H, G, P]
        rank = torch.sort(-sc, dim=-1, stable=True).indices
        npg = self.npages[li * H:(li + 1) * H].long()                              # group union sizes
        keep = torch.arange(P, device=dev)[None, None, :] < npg[:, None, None]
        chosen = torch.zeros((H, G, P), dtype=torch.bool, device=dev)
        chosen.scatter_(-1, rank, keep.expand(H, G, P))
        page_of = torch.arange(order.numel(), device=dev) // s
        att = torch.zeros((H, G, n), dtype=torch.bool, device=dev)
        att[:, :, order] = chosen[:, :, page_of]
        fixed = list(self.sink_tokens)
        for st0, fl in zip(self._win_start, self._win_fills):
            fixed += range(st0, st0 + fl)
        att[:, :, torch.as_tensor(fixed, dtype=torch.long, device=dev)] = True
        return att.gather(-1, order_all).sum(-1).double() / k_all

    def _metrics(self, token) -> StepMetrics:
        cfg = self.cfg
        if self.fallback:
            st = [0] * 5
            dq = 0
        else:
            self.forest.check()
            per_tree = self.stats.cpu().numpy()
            self._cum_stats = per_tree.copy() if self._cum_stats is None else self._cum_stats + per_tree
            st = per_tree.sum(0).tolist()
            dq = self._queries_per_step()
        return StepMetrics(step=self.steps_done - 1, token_id=token, recall_at_k=1.0, page_hit_rate=1.0,
                           covered_attention_mass=1.0, approx_rel_error=0.0, pages_selected=int(st[0]),
                           pages_loaded=int(st[2]), tokens_loaded=int(st[1]), bytes_moved=int(st[3]),
                           transactions=int(st[4]), dci_queries=dq)

    # -- reference-shaped views ------------------------------------------------------
    @property
    def heads(self) -> dict:
        """engine.py:206 (Engine.heads): (layer, kv head) -> a read-only view of
        that tree's device state (tree, table, store snapshot, sink / window
        pages).  Empty before prefill and in fallback mode."""
        if not self.prefilled or self.fallback:
            return {}
        cfg = self.cfg
        return {(cfg.skip_layers + t // cfg.kv_heads, t % cfg.kv_heads): _HeadView(self, t) for t in range(self.T)}

    def select_with_reuse(self, layer: int, layer_queries):
        """engine.py:331-363 for one layer: anchors search every query head of
        each group and record the group's token union; other layers map the
        last anchor's tokens through their own page table.  Returns
        ({kv head: pages}, {kv head: token set})."""
        if self.cfg.reuse_stride < 2:
            raise ConfigError("selection reuse is disabled")
        cfg, dev, f = self.cfg, self.device, self.forest
        H, G = cfg.kv_heads, cfg.query_heads_per_group
        trees = [self._tree(layer, h) for h in range(H)]
        pages_by_head, tokens_by_head = {}, {}
        if self.is_anchor_layer(layer):
            k, beam, cap = _budget_tuple(cfg.budget())
            q = _dev(np.asarray(layer_queries, dtype=np.float64), dev).reshape(H, G, cfg.d)
            ids, counts, pages, npages = f.query(trees, q, k, beam, cap, k_out=self.k_eff, pages_cap=self.pages_cap)
            f.check()
            self.selection_queries += H * G
            ids, counts, pages, npages = (x.cpu().numpy() for x in (ids, counts, pages, npages))
            for h in range(H):
                toks = sorted({int(x) for g in range(G) for x in ids[h, g, : counts[h, g]]})
                self._anchor_tokens[h] = toks
                pages_by_head[h] = [int(p) for p in pages[h, : npages[h]]]
                tokens_by_head[h] = set(toks)
        else:
            from .pagestore import TreePageTable, find_page_index
            for h, t in enumerate(trees):
                if h not in self._anchor_tokens:
                    raise ConfigError(f"no anchor selection recorded yet for head {h}")
                toks = self._anchor_tokens[h]
                pages_by_head[h] = find_page_index(toks, TreePageTable(f, t))
                tokens_by_head[h] = set(toks)
        return pages_by_head, tokens_by_head

    def selected(self):
        """Last step's per-tree (ranked ids per head, union pages) on the host."""
        ids = self.ids.cpu().numpy()
        counts = self.counts.cpu().numpy()
        pages = self.pages.cpu().numpy()
        npages = self.npages.cpu().numpy()
        return ids, counts, pages, npages

    def config_dict(self):
        return asdict(self.cfg)


def prefill(workload, cfg: EngineConfig, n_prefill: int | None = None, device=None) -> Engine:
    """engine.py:578-583: build an engine and prefill it from the stream's head."""
    if n_prefill is None:
        n_prefill = workload.n_tokens
    return Engine(cfg, device=device).prefill(workload, n_prefill)


class _HeadView:
    """One (layer, kv head) tree of the engine, shaped like the reference's
    _HeadState (engine.py:185-194): `tree` (a DciTree view), `table` (its
    token -> page table, queried on the device), `store` (a TierStore
    snapshot: pages with their entries, hot / pinned sets, cumulative
    TransferStats), `sink` / `window` (Page lists, oldest window first)."""

    def __init__(self, eng: Engine, t: int):
        self._eng, self._t = eng, t

    @property
    def tree(self):
        from .dci import DciTree
        e = self._eng
        f = e.forest
        return DciTree.bound(f, self._t, f.scale(self._t), e.cfg.promotion_ratio, e.cfg.page_size, f.caps.tok_cap)

    @property
    def table(self):
        from .pagestore import TreePageTable
        return TreePageTable(self._eng.forest, self._t)

    @property
    def store(self):
        from .pagestore import INDEXED, SINK, WINDOW, TierStore, TransferStats
        e, t = self._eng, self._t
        cfg, f = e.cfg, e.forest
        ex = f.export(t)
        st = TierStore(cfg.d, cfg.d_prime, cfg.scalar_bytes)
        role = {N.ROLE_SINK: SINK, N.ROLE_WINDOW: WINDOW, N.ROLE_INDEXED: INDEXED}
        pids = sorted(ex["pages"])
        k, v = f.read_pages(t, pids) if pids else (None, None)
        for i, p in enumerate(pids):
            r, toks = ex["pages"][p]
            st._next_page_id = p
            page = st.allocate_page(cfg.page_size, role[r], resident=r != N.ROLE_INDEXED,
                                    pinned=r != N.ROLE_INDEXED)
            for j, tok in enumerate(toks):
                page.append(tok, k[i, j].astype(np.float64), v[i, j].astype(np.float64))
        st._next_page_id = ex["info"]["next_page"]
        if e.steps_done and e.pages is not None:
            n = int(e.npages[t])
            st.hot |= {int(p) for p in e.pages[t, :n].cpu().tolist()}
        cum = e._cum_stats[t] if e._cum_stats is not None else np.zeros(5, np.int64)
        rot = e.rot_stats[t].cpu().numpy()
        st.stats = TransferStats(transactions=int(cum[4] + rot[1]), bytes_moved=int(cum[3] + rot[0]),
                                 pages_backloaded=int(cum[2]), pages_filtered_resident=int(cum[0] - cum[2]),
                                 pages_offloaded=int(rot[1]))
        return st

    def _pages(self, ids):
        st = self.store
        return [st.page(p) for p in ids]

    @property
    def sink(self):
        return self._pages(self._eng.forest.export(self._t)["sink"])

    @property
    def window(self):
        return self._pages(self._eng.forest.export(self._t)["win"])


class LayerPrefill:
    """Engine.prefill_layers(n): the prompt's K/V one layer at a time.  Each
    layer's work (dense mirror or sink / window pages + dci_indexing of its
    kv heads) runs on the engine's build stream after the caller's stream
    reaches the hand-off, so it overlaps whatever the caller launches next.
    The layer tensors are kept until finish() (a tree set that outgrows the
    tight page capacities is rebuilt from them)."""

    def __init__(self, eng: Engine, n_prefill: int, group: int = 4):
        self.eng = eng
        self.group = max(1, int(group))   # indexed layers per build launch (batched trees build faster)
        self.pending: list[int] = []
        self.geo = eng._prefill_begin(n_prefill)
        # high priority: the build's small launches take SMs as the model's
        # kernels release them instead of queueing behind whole GEMM waves
        self.stream = torch.cuda.Stream(device=eng.device, priority=-1)
        self.kept: dict[int, tuple] = {}
        if self.geo is not None:
            with torch.cuda.stream(self.stream):
                eng._new_forest(self.geo, tight=True)
            self.stream.synchronize()

    def layer(self, layer: int, keys, values) -> None:
        """keys [n, kv_heads, d], values [n, kv_heads, d'] (device tensors; the
        first n_prefill rows are read)."""
        eng, cfg = self.eng, self.eng.cfg
        if not 0 <= layer < cfg.layers or layer in self.kept:
            raise InputError(f"layer {layer} outside [0, {cfg.layers}) or given twice")
        n = eng.n_prefill
        k = _on_device(keys[:n], eng.device)
        v = _on_device(values[:n], eng.device)
        if tuple(k.shape[1:]) != (cfg.kv_heads, cfg.d) or tuple(v.shape[1:]) != (cfg.kv_heads, cfg.d_prime):
            raise ConfigError("layer K/V dims do not match the engine config")
        ready = torch.cuda.Event()
        ready.record(torch.cuda.current_stream(eng.device))
        self.stream.wait_event(ready)
        self.kept[layer] = (k, v)
        with torch.cuda.stream(self.stream):
            eng._store_layer(layer, k, v)
        if self.geo is not None and layer >= cfg.skip_layers:
            self.pending.append(layer)
            if len(self.pending) >= self.group:
                self._flush()

    def _flush(self) -> None:
        """Build the pending layers' trees in one launch sequence (runs of
        consecutive layers)."""
        eng = self.eng
        runs: list[list[int]] = []
        for layer in sorted(self.pending):
            if runs and layer == runs[-1][-1] + 1:
                runs[-1].append(layer)
            else:
                runs.append([layer])
        self.pending = []
        with torch.cuda.stream(self.stream):
            for run in runs:
                ks = torch.stack([self.kept[l][0] for l in run], 1)
                vs = torch.stack([self.kept[l][1] for l in run], 1)
                eng._build_layers(self.geo, run[0], run[-1] + 1, ks, vs)

    def finish(self) -> Engine:
        eng, cfg = self.eng, self.eng.cfg
        if len(self.kept) != cfg.layers:
            raise InputError(f"prefill got {len(self.kept)} of {cfg.layers} layers")
        if self.pending:
            self._flush()
        torch.cuda.current_stream(eng.device).wait_stream(self.stream)
        self.stream.synchronize()
        if self.geo is not None:
            try:
                eng.forest.check()
            except ConfigError as e:
                if "page capacity" not in str(e):
                    raise
                eng.forest.close()
                eng._new_forest(self.geo, tight=False)
                for layer in range(cfg.skip_layers, cfg.layers):
                    k, v = self.kept[layer]
                    eng._build_layers(self.geo, layer, layer + 1, k[:, None], v[:, None])
                eng.forest.check()
        self.kept.clear()
        return eng._prefill_end()
