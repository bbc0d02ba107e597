"""Time the window-rotation insert kernel (16 inserts per tree, every 16
decode steps) at C2 with CUDA events around Forest.rotate_window."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2604_10539_b200.engine import Engine, EngineConfig  # noqa: E402
from paper_2604_10539_b200.workload import clustered_stream  # noqa: E402

ctx = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
C2 = dict(layers=32, kv_heads=8, query_heads_per_group=4, d=128, d_prime=128, page_size=16,
          token_budget=256, promotion_ratio=0.1, sink_pages=1, window_pages=2, skip_layers=2)
steps = 96
st = clustered_stream(ctx, steps, 32, 8, 4, 128, 128, device="cuda")
eng = Engine(EngineConfig(**C2, kv_dtype="bf16", max_tokens=ctx + steps + 1)).prefill(st.keys, st.values, ctx)
f = eng.forest
orig = f.rotate_window
times = []


def timed(*a, **kw):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    r = orig(*a, **kw)
    e1.record()
    times.append((e0, e1))
    return r


f.rotate_window = timed
qtimes = []
orig_qa = f.query_attend


def timed_qa(*a, **kw):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    r = orig_qa(*a, **kw)
    e1.record()
    qtimes.append((e0, e1, eng.rotation_due()))
    return r


f.query_attend = timed_qa
for i in range(steps):
    eng.decode_step(ctx + i, st.queries[i], st.keys[ctx + i], st.values[ctx + i], metrics=False)
torch.cuda.synchronize()
ms = [a.elapsed_time(b) for a, b in times]
qms = [(round(a.elapsed_time(b), 3)) for a, b, _ in qtimes]
print("query_attend ms per step:", qms)
print("rotations", len(ms), "ms each", [round(x, 3) for x in ms])
print("mean rotation ms %.3f  -> %.1f us per decode step amortized" % (sum(ms[1:]) / max(1, len(ms) - 1),
                                                                    1e3 * sum(ms[1:]) / max(1, len(ms) - 1) / 16))

if os.environ.get("ICB_PROF"):
    import ctypes
    import numpy as np
    from paper_2604_10539_b200 import _native as N
    lib = N.lib()
    lib.icb_insert_profile.argtypes = [ctypes.c_void_p, ctypes.c_int]
    buf = np.zeros(8, dtype=np.uint64)
    lib.icb_insert_profile(buf.ctypes.data_as(ctypes.c_void_p), 0)
    nrot = len(ms) * eng.T
    print("per tree-rotation us: prepare %.1f search %.1f fallback %.1f finish %.1f | segments %.2f" % (
        *(buf[i] / nrot / 1.9e3 for i in range(4)), buf[4] / nrot))

    cyc = np.zeros(eng.T, dtype=np.uint64)
    fb = np.zeros(eng.T, dtype=np.uint32)
    lib.icb_insert_tree_profile.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]
    lib.icb_insert_tree_profile(cyc.ctypes.data_as(ctypes.c_void_p), fb.ctypes.data_as(ctypes.c_void_p), eng.T)
    us = cyc / len(ms) / 1.9e3
    order = np.argsort(-us)
    print("per-tree rotation us: mean %.1f  p50 %.1f  p90 %.1f  max %.1f" % (us.mean(), np.median(us),
                                                                          np.percentile(us, 90), us.max()))
    print("slowest trees (us, fallbacks/rotation):", [(int(t), round(float(us[t]), 1), round(fb[t] / len(ms), 2))
                                                      for t in order[:8]])
    print("mean fallbacks per tree-rotation %.2f; slowest-10%% trees %.2f" % (fb.mean() / len(ms),
                                                                          fb[order[:24]].mean() / len(ms)))

lib2 = __import__("paper_2604_10539_b200._native", fromlist=["lib"]).lib()
import ctypes  # noqa: E402
import numpy as np  # noqa: E402
pm = np.zeros(4, dtype=np.uint64)
lib2.icb_pdci_stats.argtypes = [ctypes.c_void_p, ctypes.c_int]
lib2.icb_pdci_stats(pm.ctypes.data_as(ctypes.c_void_p), 0)
print("warp P-DCI misses (too large, no directions, no cache, stale):", pm.tolist())
for t in (0, 1):
    i = f.info(t)
    print("tree", t, "n_dirs", i["n_dirs"])

# node sizes per level (largest nodes drive the P-DCI fallbacks)
import numpy as np  # noqa: E402
for tr in (0, eng.T // 2):
    ex = f.export(tr)
    by = {}
    for i, lv, par, own, mem in ex["nodes"]:
        by.setdefault(lv, []).append(len(mem))
    print("tree", tr, {lv: (len(v), int(np.max(v)), int(np.sum(np.array(v) > 64))) for lv, v in sorted(by.items())},
          "(level: nodes, max size, nodes > 64)")
