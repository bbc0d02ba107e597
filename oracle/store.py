"""Oracle page store: restates pagestore.py (Page :50-88, PageTable :91-108,
find_page_index :111-113, TierStore :116-229) as plain dictionaries."""

from __future__ import annotations

import numpy as np

SINK, WINDOW, INDEXED = "sink", "window", "indexed"


class OPage:
    __slots__ = ("page_id", "capacity", "role", "tokens", "keys", "values")

    def __init__(self, page_id, capacity, role):
        self.page_id = page_id
        self.capacity = capacity
        self.role = role
        self.tokens: list[int] = []
        self.keys: list[np.ndarray] = []
        self.values: list[np.ndarray] = []

    @property
    def fill(self):
        return len(self.tokens)

    @property
    def full(self):
        return self.fill >= self.capacity


class OStore:
    """Hot/cold residency with transfer counters (pagestore.py:116-215)."""

    def __init__(self, d, d_prime, scalar_bytes=4):
        self.d, self.d_prime, self.scalar_bytes = d, d_prime, scalar_bytes
        self.pages: dict[int, OPage] = {}
        self.hot: set[int] = set()
        self.pinned: set[int] = set()
        self.next_id = 0
        self.node_to_pages: dict[int, list[int]] = {}
        self.token_to_page: dict[int, int] = {}
        self.stats = dict(transactions=0, bytes_moved=0, pages_backloaded=0,
                          pages_filtered_resident=0, pages_offloaded=0)

    def allocate(self, capacity, role, resident=False, pinned=False):
        page = OPage(self.next_id, capacity, role)
        self.next_id += 1
        self.pages[page.page_id] = page
        if resident:
            self.hot.add(page.page_id)
        if pinned:
            self.pinned.add(page.page_id)
        return page

    def release(self, pid):
        del self.pages[pid]
        self.hot.discard(pid)
        self.pinned.discard(pid)

    def page_bytes(self, pid):
        return self.pages[pid].fill * (self.d + self.d_prime) * self.scalar_bytes

    def backload(self, selected):
        selected = list(selected)
        move = [p for p in selected if p not in self.hot]
        delta = dict(transactions=1 if move else 0,
                     bytes_moved=sum(self.page_bytes(p) for p in move),
                     pages_backloaded=len(move),
                     pages_filtered_resident=len(selected) - len(move),
                     pages_offloaded=0)
        self.hot.update(move)
        for key, v in delta.items():
            self.stats[key] += v
        return delta

    def offload(self, pid):
        self.hot.discard(pid)
        self.pinned.discard(pid)
        self.stats["transactions"] += 1
        self.stats["bytes_moved"] += self.page_bytes(pid)
        self.stats["pages_offloaded"] += 1

    def evict_unselected(self, keep):
        self.hot = set(keep) | self.pinned

    def tokens_in(self, pids):
        out = []
        for p in pids:
            out.extend(self.pages[p].tokens)
        return out


def find_page_index(tokens, token_to_page) -> list[int]:
    """pagestore.py:111-113: sorted unique page ids of the tokens."""
    return sorted({token_to_page[int(t)] for t in tokens})
