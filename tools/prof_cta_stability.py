"""Per-tree query-kernel spans across consecutive C2 steps (ICB_PROF=1): how
well the previous step's span predicts a tree's next one, and the block ->
SM map (which blocks run alone on an SM).   python tools/prof_cta_stability.py"""
import ctypes
import os
import sys

import numpy as np

os.environ["ICB_PROF"] = "1"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2604_10539_b200 import _native as N  # noqa: E402
from paper_2604_10539_b200.engine import Engine, EngineConfig  # noqa: E402
from paper_2604_10539_b200.workload import clustered_stream  # noqa: E402

C2 = dict(layers=32, kv_heads=8, query_heads_per_group=4, d=128, d_prime=128, page_size=16,
          token_budget=256, promotion_ratio=0.1, sink_pages=1, window_pages=2, skip_layers=2)
st = clustered_stream(32768, 12, 32, 8, 4, 128, 128, device="cuda")
eng = Engine(EngineConfig(**C2, kv_dtype="bf16", max_tokens=32768 + 16)).prefill(st.keys, st.values, 32768)
lib = N.lib()
lib.icb_search_cta_profile.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_int]
cyc = np.zeros(eng.T, dtype=np.uint64)
smi = np.zeros(eng.T, dtype=np.int32)
spans = []
for i in range(10):
    lib.icb_search_cta_profile(cyc.ctypes.data_as(ctypes.c_void_p), smi.ctypes.data_as(ctypes.c_void_p), eng.T, 1)
    eng.decode_step(32768 + i, st.queries[i], st.keys[32768 + i], st.values[32768 + i], metrics=False)
    lib.icb_search_cta_profile(cyc.ctypes.data_as(ctypes.c_void_p), smi.ctypes.data_as(ctypes.c_void_p), eng.T, 1)
    if i >= 2:
        spans.append(cyc.astype(np.float64) / 1.9e3)
        print("step", i, "sm map", smi[:16].tolist(), "...")
S = np.array(spans)
print("corr(step t, t+1) of per-tree spans:", [round(float(np.corrcoef(S[j], S[j + 1])[0, 1]), 3) for j in range(len(S) - 1)])
cnt = np.bincount(smi, minlength=148)
print("block -> sm:", smi.tolist())
print("solo blocks:", np.flatnonzero(cnt[smi] == 1).tolist())
