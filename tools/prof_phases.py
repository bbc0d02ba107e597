"""Per-phase cycle breakdown of the search kernel at C2 (ICB_PROF=1)."""
import ctypes
import os
import sys

import numpy as np
import torch

os.environ["ICB_PROF"] = "1"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2604_10539_b200 import _native as N  # noqa: E402
from paper_2604_10539_b200.engine import Engine, EngineConfig  # noqa: E402
from paper_2604_10539_b200.workload import clustered_stream  # noqa: E402

ctx = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
C2 = dict(layers=32, kv_heads=8, query_heads_per_group=4, d=128, d_prime=128, page_size=16,
          token_budget=256, promotion_ratio=0.1, sink_pages=1, window_pages=2, skip_layers=2)
st = clustered_stream(ctx, 40, 32, 8, 4, 128, 128, device="cuda")
eng = Engine(EngineConfig(**C2, kv_dtype="bf16", max_tokens=ctx + 64)).prefill(st.keys, st.values, ctx)
lib = N.lib()
lib.icb_search_profile.argtypes = [ctypes.c_void_p, ctypes.c_int]
buf = np.zeros(33, dtype=np.uint64)
for i in range(4):
    eng.decode_step(ctx + i, st.queries[i], st.keys[ctx + i], st.values[ctx + i], metrics=False)
lib.icb_search_profile(buf.ctypes.data_as(ctypes.c_void_p), 1)
for i in range(4, 12):
    eng.decode_step(ctx + i, st.queries[i], st.keys[ctx + i], st.values[ctx + i], metrics=False)
lib.icb_search_profile(buf.ctypes.data_as(ctypes.c_void_p), 1)
names = ["loop", "union", "scan+rowlist", "lift+start", "stream", "pdci+ctr", "select", "final+pages", "attention"]
print('top-B selections', buf[9], 'radix fallbacks', buf[10], 'avg boundary bin', buf[11] / max(1, buf[9]))
ns = max(1, buf[9])
print('top-B us per selection: hist %.2f scan %.2f emit %.2f sort+tail %.2f' % tuple(buf[12 + i] / ns / 1.9e3 for i in range(4)))
sc = buf[17:33]
lv_it = max(1, sc[0])
print('row lists: level iterations %d (start levels %d) | union nodes %.0f rows %.0f passes %.2f binary-search passes %.2f per level' % (
    sc[0], sc[5], sc[1] / lv_it, sc[2] / lv_it, sc[3] / lv_it, sc[4] / lv_it))
nq = 8 * eng.T
print('sub-phases us per CTA-query: union loop %.1f | sync %.1f | umask %.1f | scan nodes+stage %.1f | rows %.1f' % tuple(
    sc[8 + i] / nq / 1.9e3 for i in range(5)))
buf = buf[:9]
tot = buf.sum()
per_cta_us = buf / (8 * eng.T) / 1.9e3
for n, v, u in zip(names, buf, per_cta_us):
    print(f"{n:10s} {v / tot * 100:5.1f}%  {u:8.1f} us per CTA-query")

# per-CTA spans (the kernel ends with the slowest tree): solo vs shared SMs
cyc = np.zeros(eng.T, dtype=np.uint64)
smi = np.zeros(eng.T, dtype=np.int32)
lib.icb_search_cta_profile.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_int]
lib.icb_search_cta_profile(cyc.ctypes.data_as(ctypes.c_void_p), smi.ctypes.data_as(ctypes.c_void_p), eng.T, 1)
us = cyc / 12 / 1.9e3   # all 12 steps of the run
cnt = np.bincount(smi, minlength=148)
shared = cnt[smi] > 1
print("per-CTA us: mean %.1f p50 %.1f p90 %.1f max %.1f | solo SMs %d CTAs mean %.1f max %.1f | shared mean %.1f max %.1f" % (
    us.mean(), np.median(us), np.percentile(us, 90), us.max(), (~shared).sum(), us[~shared].mean(), us[~shared].max(),
    us[shared].mean(), us[shared].max()))
print("blocks on solo SMs:", sorted(np.flatnonzero(~shared).tolist())[:60])
