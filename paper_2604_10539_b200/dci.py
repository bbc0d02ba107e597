"""The reference's DCI-tree API (icecache/dci.py) on the device.

Drop-in names and semantics for one tree: `dci_indexing` (dci.py:479-568),
`DciTree` with `query` (:318-364), `insert` (:385-431), `check_invariants`
(:453-476), `levels`, `point_level` and the `query_count` /
`distance_evals` / `scale_clamps` counters; `query_raw` (:571-574);
`SearchBudget` / `PARENT_BUDGET` (:50-78); `assign_level` (:81-88);
`KeyScale` (geometry.py:37-56).  Each tree is a one-tree DeviceForest: build,
search and insert run in the library's kernels (the same ones the Engine
batches over a forest).  Point ids index device rows, so they must lie in
[0, capacity).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N
from .attention import gqa_union  # noqa: F401  (re-exported: attention.py:96-103)
from .errors import ConfigError, InputError
from .forest import DeviceForest, ForestCaps
from .pagestore import INDEXED, PageTable

SENTINEL_LEVEL = -1            # dci.py:35
ROOT_OWNER = -1                # dci.py:38
EXHAUSTIVE_NODE_LIMIT = 64     # dci.py:41
NUM_PROJECTIONS = 8            # dci.py:44
UNBOUNDED = 2**62              # dci.py:47
DEFAULT_PAGE_SIZE = 16


@dataclass(frozen=True)
class SearchBudget:
    """dci.py:50-74: result count, per-level survivors, evaluations per node."""

    k: int
    beam: int
    visit_cap: int

    def __post_init__(self) -> None:
        if self.k < 1:
            raise ConfigError(f"k must be >= 1, got {self.k}")
        if self.beam < self.k:
            raise ConfigError(f"beam ({self.beam}) must be >= k ({self.k})")
        if self.visit_cap < self.k:
            raise ConfigError(f"visit_cap ({self.visit_cap}) must be >= k ({self.k})")

    @classmethod
    def for_k(cls, k: int, beam: int | None = None, visit_cap: int | None = None) -> "SearchBudget":
        return cls(k, beam if beam is not None else 2 * k, visit_cap if visit_cap is not None else 4 * k)

    @classmethod
    def exhaustive(cls, k: int) -> "SearchBudget":
        return cls(k, UNBOUNDED, UNBOUNDED)


PARENT_BUDGET = SearchBudget(k=1, beam=8, visit_cap=64)   # dci.py:78


def assign_level(r: float, rng: np.random.Generator) -> int:
    """dci.py:81-88: 1 + the number of consecutive uniforms below r."""
    if not 0.0 < r < 1.0:
        raise ConfigError(f"promotion ratio must lie in (0, 1), got {r}")
    level = 1
    while rng.random() < r:
        level += 1
    return level


def transform_query(q) -> np.ndarray:
    """geometry.py:89-98: [q / ||q||, 0]; a zero query is degenerate."""
    from .errors import DegenerateQueryError
    q = np.asarray(q, dtype=np.float64).reshape(-1)
    n = float(np.sqrt((q * q).sum()))
    if n == 0.0:
        raise DegenerateQueryError("zero query vector")
    return np.concatenate([q / n, [0.0]])


@dataclass(frozen=True)
class DciNode:
    """Read-only view of a device node (dci.py:139-153)."""

    node_id: int
    level: int
    parent_id: int | None
    owner_id: int
    member_ids: list
    page_ids: list

    @property
    def is_leaf(self) -> bool:
        return self.level == 1


@dataclass(frozen=True)
class KeyScale:
    """geometry.py:37-56: c = 1.05 * max ||k|| over the build keys (1.05 for
    all-zero keys); fixed for the tree's lifetime."""

    c: float

    @classmethod
    def from_keys(cls, keys, headroom: float = 1.05) -> "KeyScale":
        k = np.asarray(keys, dtype=np.float64)
        if k.size == 0:
            raise InputError("cannot derive a scale from an empty key set")
        m = float(np.sqrt((k * k).sum(axis=-1).max()))
        return cls(headroom * (m if m > 0.0 else 1.0))


class DciTree:
    """One device-resident DCI tree (dci.py:156-476).  Construct empty with a
    KeyScale and grow it by inserts, or batch-build with dci_indexing."""

    def __init__(self, dim: int, scale: KeyScale | None, promotion_ratio: float, seed: int | tuple = 0, *,
                 store=None, table=None, page_size: int = DEFAULT_PAGE_SIZE,
                 parent_budget: SearchBudget = PARENT_BUDGET, capacity: int = 4096, dim_v: int | None = None,
                 device=None):
        if not 0.0 < promotion_ratio < 1.0:
            raise ConfigError(f"promotion ratio must lie in (0, 1), got {promotion_ratio}")
        if dim < 1:
            raise ConfigError(f"dim must be >= 1, got {dim}")
        if parent_budget != PARENT_BUDGET:
            raise ConfigError("the device insert path implements PARENT_BUDGET (k=1, beam=8, visit_cap=64)")
        self.dim = dim
        self.dim_v = dim_v or dim
        self.scale = scale
        self.promotion_ratio = promotion_ratio
        self.page_size = page_size
        # store / table (dci.py:176-177): the device tree's pages are mirrored
        # into them as the reference's _place_entry writes them (dci.py:368-381)
        self.store = store
        self.table = table if table is not None else (PageTable() if store is not None else None)
        self._dev2store: dict[int, int] = {}
        self.parent_budget = parent_budget
        self.capacity = int(capacity)
        self.forest = DeviceForest(1, dim, self.dim_v, tok_cap=self.capacity, promotion_ratio=promotion_ratio,
                                   page_size=page_size, kv_dtype="fp32", device=device,
                                   caps=ForestCaps.for_tokens(self.capacity, promotion_ratio, page_size))
        self._t = 0
        self.forest.seed([0], [seed])
        if scale is not None:
            N.check(N.lib().icb_set_scale(self.forest.h, 0, float(scale.c)))
        self._export = None

    @classmethod
    def bound(cls, forest: DeviceForest, tree: int, scale: float, promotion_ratio: float, page_size: int,
              capacity: int) -> "DciTree":
        """A view of tree `tree` of an existing forest (the Engine's trees):
        the same read / query / insert API, no store mirror."""
        self = cls.__new__(cls)
        self.dim, self.dim_v = forest.dim, forest.dim_v
        self.scale = KeyScale(float(scale))
        self.promotion_ratio, self.page_size = promotion_ratio, page_size
        self.store, self.table = None, None
        self._dev2store = {}
        self.parent_budget = PARENT_BUDGET
        self.capacity = int(capacity)
        self.forest = forest
        self._t = int(tree)
        self._export = None
        self._live = True    # the engine mutates the tree between calls: never cache its export
        return self

    # -- counters / structure (host mirror) ------------------------------------------
    def _info(self):
        return self.forest.info(self._t)

    def __len__(self) -> int:
        return self._info()["n_points"]

    @property
    def levels(self) -> int:
        return self._info()["levels"]

    @property
    def query_count(self) -> int:
        return self._info()["query_count"]

    @property
    def distance_evals(self) -> int:
        return self._info()["distance_evals"]

    @property
    def scale_clamps(self) -> int:
        return self._info()["scale_clamps"]

    def export(self) -> dict:
        if self._export is None or getattr(self, "_live", False):
            self._export = self.forest.export(self._t)
        return self._export

    @property
    def point_level(self) -> dict[int, int]:
        return dict(self.export()["point_level"])

    def point_ids(self) -> list[int]:
        return sorted(self.point_level)

    @property
    def top_node_id(self) -> int | None:
        top = self._info()["top_node"]
        return top if self.levels > 0 else None

    @property
    def nodes(self) -> dict[int, DciNode]:
        ex = self.export()
        top = ex["info"]["top_node"]
        pid = (lambda p: self._dev2store[p]) if self.store is not None else (lambda p: p)   # noqa: E731
        return {i: DciNode(i, lv, None if i == top else par, own, list(mem),
                           [pid(p) for p in ex["leaf_pages"].get(i, [])])
                for i, lv, par, own, mem in ex["nodes"]}

    def lifted(self, point_id: int) -> np.ndarray:
        """The stored lifted key [dim + 1] (fp32 rows, returned as fp64)."""
        ex = self.forest.export(self._t, with_rows=True)
        return np.concatenate([ex["lift"][point_id, : self.dim].astype(np.float64),
                               [float(ex["tail"][point_id])]])

    def page_fill(self, page_id: int) -> int:
        return len(self.export()["pages"][int(page_id)][1])

    # -- store / table mirror (dci.py:368-381) -----------------------------------------
    def _mirror_page(self, dev_page: int, leaf: int):
        sp = self._dev2store.get(dev_page)
        if sp is None:
            page = self.store.allocate_page(self.page_size, INDEXED, resident=False)
            sp = self._dev2store[dev_page] = page.page_id
            self.table.assign_page(leaf, sp)
        return self.store.page(sp)

    def _mirror_build(self, ids, keys, values):
        """Write the built tree's pages into the store in device page order
        (leaves in node-id order, members in order: the reference's order)."""
        ex = self.export()
        row = {int(p): i for i, p in enumerate(ids)}
        leaf_of = {p: leaf for leaf, pages in ex["leaf_pages"].items() for p in pages}
        for dp in sorted(p for p, (role, _) in ex["pages"].items() if role == N.ROLE_INDEXED):
            page = self._mirror_page(dp, leaf_of[dp])
            for tok in ex["pages"][dp][1]:
                r = row[tok]
                page.append(tok, keys[r], values[r] if values is not None else np.zeros(self.store.d_prime))
                self.table.map_token(tok, page.page_id)

    def _mirror_insert(self, point_id: int, key, value):
        ex = self.export()
        dp = int(ex["tok2page"][point_id])
        leaf = next(i for i, lv, _, _, mem in ex["nodes"] if lv == 1 and point_id in mem)
        page = self._mirror_page(dp, leaf)
        page.append(point_id, key, value if value is not None else np.zeros(self.store.d_prime))
        self.table.map_token(point_id, page.page_id)

    # -- search --------------------------------------------------------------------
    def query(self, q_vec, target_level: int, k: int, budget: SearchBudget | None = None) -> list[int]:
        """dci.py:318-364: q_vec is the lifted query [dim + 1]; ids ranked by
        (d2, id); target_level SENTINEL_LEVEL collects every level."""
        if budget is None:
            budget = SearchBudget.for_k(k)
        q = np.asarray(q_vec, dtype=np.float64).reshape(-1)
        if q.shape != (self.dim + 1,):
            raise InputError(f"lifted query must have shape ({self.dim + 1},), got {q.shape}")
        return self._query(torch.as_tensor(q.astype(np.float32)), target_level, k, budget, lifted=True)

    def _query(self, q, target_level, k, budget, lifted):
        ids, counts, _, _ = self.forest.query([self._t], q.reshape(1, 1, -1), k, budget.beam, budget.visit_cap,
                                              target_level, lifted=lifted, want_pages=False)
        self.forest.check()
        return [int(x) for x in ids[0, 0, : int(counts[0, 0])].cpu().tolist()]

    def pdci_query(self, q_vec, node, k: int, budget: SearchBudget | None = None) -> list[int]:
        """dci.py:282-298: the node's k nearest members to a lifted query
        (exact up to EXHAUSTIVE_NODE_LIMIT members or when the visit cap covers
        the node; else the P-DCI order truncated at visit_cap evaluations)."""
        from .forest import _ptr, _stream
        node_id = node.node_id if isinstance(node, DciNode) else int(node)
        if budget is None:
            budget = SearchBudget.for_k(k)
        q = np.asarray(q_vec, dtype=np.float64).reshape(-1)
        if q.shape != (self.dim + 1,):
            raise InputError(f"lifted query must have shape ({self.dim + 1},), got {q.shape}")
        dev = self.forest.device
        qd = torch.as_tensor(q.astype(np.float32), device=dev)
        ids = torch.empty(max(1, min(int(k), self.capacity)), dtype=torch.int32, device=dev)
        cnt = torch.zeros(1, dtype=torch.int32, device=dev)
        N.check(N.lib().icb_node_query(self.forest.h, self._t, node_id, _ptr(qd), int(min(k, ids.numel())),
                                       int(min(budget.visit_cap, 2**62)), _ptr(ids), _ptr(cnt), _stream()))
        self.forest.check()
        return [int(x) for x in ids[: int(cnt.item())].cpu().tolist()]

    # -- insert --------------------------------------------------------------------
    def insert(self, point_id: int, key, value=None, *, rng: np.random.Generator | None = None,
               level: int | None = None) -> int:
        """dci.py:385-431; returns the assigned level.  The level is drawn from
        the tree's own stream on the device unless `rng` or `level` is given."""
        point_id = int(point_id)
        key = np.asarray(key, dtype=float)
        if key.shape != (self.dim,):
            raise InputError(f"key must have shape ({self.dim},), got {key.shape}")
        if not 0 <= point_id < self.capacity:
            raise ConfigError(f"point id {point_id} outside the tree's capacity {self.capacity}")
        if level is None and rng is not None:
            level = assign_level(self.promotion_ratio, rng)
        if self.levels == 0 and self.scale is None:
            raise ConfigError("an empty tree needs a KeyScale before its first insert")
        val = np.zeros(self.dim_v) if value is None else np.asarray(value, dtype=float).reshape(self.dim_v)
        lv = None if level is None else np.array([[int(level)]], dtype=np.int32)
        out = self.forest.insert([self._t], np.array([[point_id]], dtype=np.int32), key.reshape(1, 1, -1),
                                 val.reshape(1, 1, -1), levels=lv)
        self._export = None
        self.forest.check()
        if self.store is not None:
            self._mirror_insert(point_id, key, None if value is None else np.asarray(value, dtype=float))
        return int(out[0, 0])

    # -- integrity -----------------------------------------------------------------
    def check_invariants(self) -> None:
        """dci.py:453-476 on the exported device structure (AssertionError on
        violation)."""
        ex = self.forest.export(self._t)
        levels, top = ex["info"]["levels"], ex["info"]["top_node"]
        nodes = {n[0]: n for n in ex["nodes"]}
        assert levels >= 1 and top >= 0
        assert {n[1] for n in nodes.values()} == set(range(1, levels + 1)), "empty level present"
        leaf_members: list[int] = []
        for i, lv, par, own, mem in nodes.values():
            assert mem, f"empty node {i}"
            if i == top:
                assert par == -1 and own == ROOT_OWNER
            else:
                assert nodes[par][1] == lv + 1, "parent not one level up"
                assert own in nodes[par][4], "owner missing from parent"
            if lv == 1:
                leaf_members += list(mem)
                fills = sum(len(ex["pages"][p][1]) for p in ex["leaf_pages"][i])
                assert fills == len(mem), "page fill != leaf membership"
        assert sorted(leaf_members) == sorted(ex["point_level"]), "leaf coverage broken"
        assert len(set(leaf_members)) == len(leaf_members), "duplicate leaf membership"


def dci_indexing(keys, promotion_ratio: float, seed: int | tuple = 0, *, values=None, store=None, table=None,
                 page_size: int = DEFAULT_PAGE_SIZE, scale: KeyScale | None = None,
                 parent_budget: SearchBudget = PARENT_BUDGET, capacity: int | None = None,
                 device=None) -> DciTree:
    """dci.py:479-568: batch-build over (point id, key vector) pairs (levels,
    exact 1-NN parents, nodes, pages -- identical to the reference's)."""
    pairs = list(keys)
    if not pairs:
        raise InputError("cannot index an empty key set")
    ids = np.array([int(p) for p, _ in pairs], dtype=np.int64)
    if len(set(ids.tolist())) != len(ids):
        raise InputError("duplicate point ids")
    mat = np.stack([np.asarray(k, dtype=np.float64) for _, k in pairs])
    if ids.min() < 0:
        raise ConfigError("point ids must be non-negative")
    dim = mat.shape[1]
    vals = None if values is None else np.stack([np.asarray(v, dtype=np.float64) for v in values])
    cap = int(capacity) if capacity is not None else max(2 * (int(ids.max()) + 1), 64)
    tree = DciTree(dim, scale, promotion_ratio, seed, store=store, table=table, page_size=page_size,
                   parent_budget=parent_budget, capacity=cap, dim_v=None if vals is None else vals.shape[1],
                   device=device)
    sc = None if scale is None else np.array([scale.c])
    tree.forest.build([0], ids.astype(np.int32).reshape(1, -1), mat.reshape(1, len(ids), dim),
                      None if vals is None else vals.reshape(1, len(ids), -1), scales=sc)
    tree.forest.check()
    if tree.scale is None:
        tree.scale = KeyScale(tree.forest.scale(0))
    if store is not None:
        tree._mirror_build(ids, mat, vals)
    return tree


def query_raw(tree: DciTree, q, target_level: int, k: int, budget: SearchBudget | None = None) -> list[int]:
    """dci.py:571-574: lift the raw query (transform_query) and search."""
    if budget is None:
        budget = SearchBudget.for_k(k)
    q = np.asarray(q, dtype=np.float64).reshape(-1)
    if q.shape != (tree.dim,):
        raise InputError(f"query must have shape ({tree.dim},), got {q.shape}")
    return tree._query(torch.as_tensor(q.astype(np.float32)), target_level, k, budget, lifted=False)
