"""Largest DCI nodes over every tree of a C2/C3-shaped forest (after prefill
and `steps` decode steps): the P-DCI cost drivers.
  python tools/node_sizes.py [ctx] [steps]"""
import ctypes
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2604_10539_b200 import _native as N  # noqa: E402
from paper_2604_10539_b200.engine import Engine, EngineConfig  # noqa: E402
from paper_2604_10539_b200.workload import clustered_stream  # noqa: E402

ctx = int(sys.argv[1]) if len(sys.argv) > 1 else 131072
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 0
C2 = dict(layers=32, kv_heads=8, query_heads_per_group=4, d=128, d_prime=128, page_size=16,
          token_budget=256, promotion_ratio=0.1, sink_pages=1, window_pages=2, skip_layers=2)
st = clustered_stream(ctx, max(steps, 1), 32, 8, 4, 128, 128, device="cuda")
eng = Engine(EngineConfig(**C2, kv_dtype="bf16", max_tokens=ctx + steps + 2)).prefill(st.keys, st.values, ctx)
for i in range(steps):
    eng.decode_step(ctx + i, st.queries[i], st.keys[ctx + i], st.values[ctx + i], metrics=False)
f = eng.forest
cp = f.caps
lv = np.zeros(cp.node_cap, np.int32)
sz = np.zeros(cp.node_cap, np.int32)
P = ctypes.c_void_p
big = []
for t in range(eng.T):
    N.check(N.lib().icb_export_tree(f.h, t, lv.ctypes.data_as(P), None, None, None, sz.ctypes.data_as(P),
                                    *([None] * 15)))
    nn = f.info(t)["n_nodes"]
    for lvl in range(1, int(lv[:nn].max()) + 1):
        s = sz[:nn][lv[:nn] == lvl]
        big.append((int(s.max()), t, lvl, int((s > 64).sum()), int((s > 1024).sum())))
big.sort(reverse=True)
print("largest nodes (size, tree, level, nodes>64 at that level, nodes>1024):", big[:12])
allsz = [b[0] for b in big if b[2] == 1]
print("leaf max size over trees: p50 %d p90 %d max %d" % (np.median(allsz), np.percentile(allsz, 90), max(allsz)))
print("trees with a node > 1024:", sorted({b[1] for b in big if b[0] > 1024}))
