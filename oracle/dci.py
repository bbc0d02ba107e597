"""Oracle DCI tree: CPU restatement of /root/reference/pkg/src/icecache/dci.py
with the device precision contract (see oracle/__init__.py).

TEST INFRASTRUCTURE ONLY.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

from . import numerics as nm
from .store import INDEXED, OStore

SENTINEL = -1                 # dci.py:35
ROOT_OWNER = -1               # dci.py:38
EXHAUSTIVE_NODE_LIMIT = 64    # dci.py:41
NUM_PROJECTIONS = 8           # dci.py:44
PARENT_BUDGET = (1, 8, 64)    # dci.py:78  (k, beam, visit_cap)

from .clib import lib as _lib  # noqa: E402


def _dptr(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def nn_parents(pts64: np.ndarray, cands64: np.ndarray) -> np.ndarray:
    """Index into cands of each point's exact nearest lifted neighbour
    (dci.py:535-543, fp64, first index on ties)."""
    pts64 = np.ascontiguousarray(pts64, dtype=np.float64)
    cands64 = np.ascontiguousarray(cands64, dtype=np.float64)
    out = np.empty(pts64.shape[0], dtype=np.int32)
    _lib().oracle_nn_parents(_dptr(pts64), pts64.shape[0], _dptr(cands64), cands64.shape[0],
                             pts64.shape[1], out.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)))
    return out


def project(dirs: np.ndarray, vecs: np.ndarray) -> np.ndarray:
    dirs = np.ascontiguousarray(dirs, dtype=np.float64)
    vecs = np.ascontiguousarray(np.atleast_2d(vecs), dtype=np.float64)
    out = np.empty((vecs.shape[0], dirs.shape[0]), dtype=np.float64)
    _lib().oracle_project(_dptr(dirs), dirs.shape[0], _dptr(vecs), vecs.shape[0], dirs.shape[1],
                          _dptr(out))
    return out


def level_stream(entropy):
    """The tree's level stream (dci.py:180-183)."""
    base = np.random.SeedSequence(entropy)
    return base.entropy, np.random.default_rng(
        np.random.SeedSequence(entropy=base.entropy, spawn_key=(0,)))


def draw_level(r, rng) -> int:
    """assign_level (dci.py:81-88)."""
    level = 1
    while rng.random() < r:
        level += 1
    return level


def pdci_dirs(seed_entropy, node_id, dim1):
    """Per-node unit projection directions (dci.py:268-273)."""
    rng = np.random.default_rng(np.random.SeedSequence(entropy=seed_entropy,
                                                       spawn_key=(1, node_id)))
    dirs = rng.normal(size=(NUM_PROJECTIONS, dim1))
    norms = np.sqrt(nm.pairwise_sum(dirs * dirs))
    return dirs / norms[:, None]


def visit_order(dirs, member_ids, member_vecs64, q64, cap) -> list[int]:
    """Prioritized-projection visit order (dci.py:106-135) as an explicit
    merge of 2m monotone chains: each ladder j is the members sorted by
    (projection, id); its left chain walks down from the query's insertion
    point, its right chain walks up.  At every step the chain head with the
    smallest (gap, j, pos, step) is popped; a member is emitted once popped
    from all m ladders.  Identical pop sequence to the reference's heap.
    """
    m = dirs.shape[0]
    ids = np.asarray(member_ids, dtype=np.int64)
    proj = project(dirs, member_vecs64)            # [n, m]
    qp = project(dirs, q64[None, :])[0]             # [m]
    ladders = []
    for j in range(m):
        order = np.lexsort((ids, proj[:, j]))
        ladders.append((proj[order, j], ids[order]))
    heads = []  # (gap, j, pos, step)
    for j in range(m):
        vals, _ = ladders[j]
        start = int(np.searchsorted(vals, qp[j], side="left"))
        for pos, step in ((start - 1, -1), (start, 1)):
            if 0 <= pos < len(vals):
                heads.append((abs(vals[pos] - qp[j]), j, pos, step))
    seen: dict[int, int] = {}
    out: list[int] = []
    while heads and len(out) < cap:
        best = min(range(len(heads)), key=lambda i: heads[i])
        _, j, pos, step = heads[best]
        vals, lid = ladders[j]
        pid = int(lid[pos])
        cnt = seen.get(pid, 0) + 1
        seen[pid] = cnt
        if cnt == m:
            out.append(pid)
        nxt = pos + step
        if 0 <= nxt < len(vals):
            heads[best] = (abs(vals[nxt] - qp[j]), j, nxt, step)
        else:
            heads.pop(best)
    return out


class ONode:
    __slots__ = ("node_id", "level", "parent", "owner", "members", "pages")

    def __init__(self, node_id, level, parent, owner, members):
        self.node_id, self.level, self.parent, self.owner = node_id, level, parent, owner
        self.members = list(members)
        self.pages: list[int] = []


class OracleTree:
    """Restatement of DciTree (dci.py:156-476) over fp32 lifted rows."""

    def __init__(self, dim, c, r, seed=0, *, store: OStore | None = None, page_size=16,
                 parent_budget=PARENT_BUDGET):
        self.dim, self.c, self.r = dim, float(c), r
        entropy = seed if isinstance(seed, int) else list(seed)
        self.seed_entropy, self.rng = level_stream(entropy)
        self.store, self.page_size, self.parent_budget = store, page_size, parent_budget
        self.levels = 0
        self.nodes: dict[int, ONode] = {}
        self.top = None
        self.point_level: dict[int, int] = {}
        self.row: dict[int, np.ndarray] = {}     # fp32 [DPAD]
        self.tail: dict[int, np.float32] = {}
        self.own: dict[tuple[int, int], int] = {}         # (owner, level) -> node
        self.member_of: dict[tuple[int, int], int] = {}   # (point, level) -> node
        self.next_node = 0
        self.query_count = 0
        self.distance_evals = 0
        self.scale_clamps = 0
        self._dirs: dict[int, np.ndarray] = {}

    # -- helpers ----------------------------------------------------------
    def _new_node(self, level, parent, owner, members):
        node = ONode(self.next_node, level, parent, owner, members)
        self.next_node += 1
        self.nodes[node.node_id] = node
        self.own[(owner, level)] = node.node_id
        for p in node.members:
            self.member_of[(p, level)] = node.node_id
        return node

    def _add_member(self, node, pid):
        node.members.append(pid)
        self.member_of[(pid, node.level)] = node.node_id

    def vec64(self, pid):
        d = self.dim
        return np.concatenate([self.row[pid][:d].astype(np.float64), [np.float64(self.tail[pid])]])

    def _candidates(self, node, q32, qt, q64, visit_cap):
        members = node.members
        if len(members) <= EXHAUSTIVE_NODE_LIMIT or visit_cap >= len(members):
            ids = list(members)
        else:
            if node.node_id not in self._dirs:
                self._dirs[node.node_id] = pdci_dirs(self.seed_entropy, node.node_id, self.dim + 1)
            vecs = np.stack([self.vec64(p) for p in members])
            ids = visit_order(self._dirs[node.node_id], members, vecs, q64, visit_cap)
        rows = np.stack([self.row[p] for p in ids]) if ids else np.zeros((0, nm.DPAD), np.float32)
        tails = np.array([self.tail[p] for p in ids], dtype=np.float32)
        self.distance_evals += len(ids)
        return np.asarray(ids, dtype=np.int64), nm.d2_fp32(rows, tails, q32, qt)

    def query(self, q32, target_level, k, beam, visit_cap, q_tail=0.0) -> list[int]:
        """DciTree.query (dci.py:318-364) with fp32 keys.  `q32` is the lifted
        query (padded to DPAD) and `q_tail` its last lifted coordinate."""
        if self.levels == 0:
            raise ValueError("query on an empty tree")
        q32 = np.asarray(q32, dtype=np.float32)
        qt = np.float32(q_tail)
        q64 = np.concatenate([q32[: self.dim].astype(np.float64), [np.float64(qt)]])
        collect_all = target_level == SENTINEL
        floor = 1 if collect_all else min(target_level, self.levels)
        self.query_count += 1
        best: dict[int, np.uint64] = {}
        survivors: list[int] = []
        for level in range(self.levels, floor - 1, -1):
            if level == self.levels:
                nids = [self.top]
            else:
                nids = [self.own[(p, level)] for p in survivors]
            all_ids, all_d2 = [], []
            for nid in nids:
                ids, d2 = self._candidates(self.nodes[nid], q32, qt, q64, visit_cap)
                all_ids.append(ids)
                all_d2.append(d2)
            ids = np.concatenate(all_ids) if all_ids else np.zeros(0, np.int64)
            d2 = np.concatenate(all_d2) if all_d2 else np.zeros(0, np.float32)
            keys = nm.pack_keys(d2, ids)
            if collect_all or level == floor:
                for kk, pid in zip(keys.tolist(), ids.tolist()):
                    if pid not in best or kk < best[pid]:
                        best[pid] = kk
            if level > floor:
                order = np.argsort(keys, kind="stable")[:beam]
                survivors = [int(ids[i]) for i in order]
        ranked = sorted(best.items(), key=lambda kv: kv[1])
        return [pid for pid, _ in ranked[:k]]

    def query_keys(self, q32, k, beam, visit_cap):
        """SENTINEL query returning (ids, fp32 d2) in ranked order."""
        ids = self.query(q32, SENTINEL, k, beam, visit_cap)
        rows = np.stack([self.row[p] for p in ids])
        tails = np.array([self.tail[p] for p in ids], dtype=np.float32)
        return ids, nm.d2_fp32(rows, tails, q32)

    # -- pages -----------------------------------------------------------------
    def _place(self, leaf, pid, key, value):
        st = self.store
        if st is None:
            return
        if value is None:
            value = np.zeros(st.d_prime)
        if leaf.pages and not st.pages[leaf.pages[-1]].full:
            page = st.pages[leaf.pages[-1]]
        else:
            page = st.allocate(self.page_size, INDEXED)
            leaf.pages.append(page.page_id)
            st.node_to_pages.setdefault(leaf.node_id, []).append(page.page_id)
        page.tokens.append(int(pid))
        page.keys.append(np.asarray(key, dtype=np.float64))
        page.values.append(np.asarray(value, dtype=np.float64))
        st.token_to_page[int(pid)] = page.page_id

    # -- insertion ---------------------------------------------------------------
    def _lift_one(self, key):
        rows, tail, over = nm.lift_keys32(np.asarray(key, dtype=np.float64)[None, :], self.c)
        self.scale_clamps += int(over[0])
        return rows[0], tail[0]

    def insert(self, pid, key, value=None, *, level=None) -> int:
        """DciTree.insert (dci.py:385-431) and _grow_top (:433-449)."""
        pid = int(pid)
        if pid in self.point_level:
            raise ValueError(f"point id {pid} already indexed")
        if level is None:
            level = draw_level(self.r, self.rng)
        row, tail = self._lift_one(key)
        self.row[pid], self.tail[pid] = row, tail
        if self.levels == 0:
            self.levels = level
            top = self._new_node(level, None, ROOT_OWNER, [pid])
            self.top = top.node_id
            chain_from = level - 1
        elif level > self.levels:
            chain_from = self.levels - 1
            self._grow_top(pid, level)
        else:
            if level == self.levels:
                container = self.nodes[self.top]
            else:
                k, beam, cap = self.parent_budget
                parent = self.query(row, level + 1, k, beam, cap, q_tail=tail)[0]
                container = self.nodes[self.own[(parent, level)]]
            self._add_member(container, pid)
            chain_from = level - 1
        for lv in range(chain_from, 0, -1):
            self._new_node(lv, self.member_of[(pid, lv + 1)], pid, [pid])
        self.point_level[pid] = level
        self._place(self.nodes[self.member_of[(pid, 1)]], pid, key, value)
        return level

    def _grow_top(self, pid, new_level):
        old = self.nodes[self.top]
        old_level = self.levels
        top = self._new_node(new_level, None, ROOT_OWNER, [pid])
        del self.own[(ROOT_OWNER, old_level)]
        self.top = top.node_id
        prev = top
        for lv in range(new_level - 1, old_level, -1):
            prev = self._new_node(lv, prev.node_id, pid, [pid])
        old.owner = pid
        old.parent = prev.node_id
        self.own[(pid, old_level)] = old.node_id
        self._add_member(old, pid)
        self.levels = new_level

    # -- canonical export -----------------------------------------------------------
    def export(self):
        nodes = sorted((n.node_id, n.level, -1 if n.parent is None else n.parent, n.owner,
                        tuple(n.members), tuple(n.pages)) for n in self.nodes.values())
        return dict(levels=self.levels, top=self.top, point_level=dict(self.point_level),
                    nodes=nodes)

    def check_invariants(self):
        """dci.py:453-476."""
        assert self.levels >= 1 and self.top is not None
        assert {n.level for n in self.nodes.values()} == set(range(1, self.levels + 1))
        leaf = []
        for n in self.nodes.values():
            assert n.members
            if n.node_id == self.top:
                assert n.parent is None and n.owner == ROOT_OWNER
            else:
                par = self.nodes[n.parent]
                assert par.level == n.level + 1 and n.owner in par.members
            if n.level == 1:
                leaf.extend(n.members)
                if self.store is not None:
                    assert sum(self.store.pages[p].fill for p in n.pages) == len(n.members)
        assert sorted(leaf) == sorted(self.point_level)
        assert len(set(leaf)) == len(leaf)


def build(keys_by_id, r, seed=0, *, values=None, store=None, page_size=16, c=None,
          parent_budget=PARENT_BUDGET) -> OracleTree:
    """dci_indexing (dci.py:479-568) restated."""
    pairs = list(keys_by_id)
    ids = [int(p) for p, _ in pairs]
    mat = np.asarray([np.asarray(k, dtype=np.float64) for _, k in pairs])
    if c is None:
        c = nm.key_scale(mat)
    tree = OracleTree(mat.shape[1], c, r, seed, store=store, page_size=page_size,
                      parent_budget=parent_budget)
    drawn = [draw_level(r, tree.rng) for _ in ids]
    occupied = sorted(set(drawn))
    compact = {lv: i + 1 for i, lv in enumerate(occupied)}
    top = {pid: compact[lv] for pid, lv in zip(ids, drawn)}
    L = len(occupied)
    rows64, tail64, over = nm.lift_keys64(mat, c)
    tree.scale_clamps += int(over.sum())
    rows32 = np.zeros((len(ids), nm.DPAD), np.float32)
    rows32[:, : mat.shape[1]] = rows64.astype(np.float32)
    tail32 = tail64.astype(np.float32)
    full64 = np.concatenate([rows64, tail64[:, None]], axis=1)
    index = {pid: i for i, pid in enumerate(ids)}
    for pid, i in index.items():
        tree.row[pid], tree.tail[pid] = rows32[i], tail32[i]
    parent_of = {}
    for lv in range(L - 1, 0, -1):
        pts = [p for p in ids if top[p] == lv]
        cands = [p for p in ids if top[p] > lv]
        if not pts:
            continue
        nn = nn_parents(full64[[index[p] for p in pts]], full64[[index[p] for p in cands]])
        for p, ci in zip(pts, nn.tolist()):
            parent_of[p] = cands[ci]
    tree.levels = L
    tree.top = tree._new_node(L, None, ROOT_OWNER, [p for p in ids if top[p] == L]).node_id
    for lv in range(L - 1, 0, -1):
        groups: dict[int, list[int]] = {}
        for p in ids:
            if top[p] < lv:
                continue
            owner = parent_of[p] if top[p] == lv else p
            groups.setdefault(owner, []).append(p)
        for owner, members in groups.items():
            tree._new_node(lv, tree.member_of[(owner, lv + 1)], owner, members)
    tree.point_level = dict(top)
    if store is not None:
        for node in list(tree.nodes.values()):
            if node.level == 1:
                for p in node.members:
                    v = values[index[p]] if values is not None else None
                    tree._place(node, p, mat[index[p]], v)
    return tree
