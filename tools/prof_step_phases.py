"""Per-step phase breakdown of the search kernel (ICB_PROF=1): plain steps vs
the step right after a window rotation.   python tools/prof_step_phases.py [ctx] [steps]"""
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

ctx = int(sys.argv[1]) if len(sys.argv) > 1 else 131072
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 34
C2 = dict(layers=32, kv_heads=8, query_heads_per_group=4, d=128, d_prime=128, page_size=16,
          token_budget=256, promotion_ratio=0.1, sink_pages=1, window_pages=2, skip_layers=2)
st = clustered_stream(ctx, steps, 32, 8, 4, 128, 128, device="cuda")
eng = Engine(EngineConfig(**C2, kv_dtype="bf16", max_tokens=ctx + steps + 1)).prefill(st.keys, st.values, ctx)
lib = N.lib()
lib.icb_search_profile.argtypes = [ctypes.c_void_p, ctypes.c_int]
names = ["loop", "union", "scan+rowlist", "lift+start", "stream", "pdci+ctr", "select", "final+pages", "attention"]
buf = np.zeros(25, dtype=np.uint64)
for i in range(steps):
    rot = eng.rotation_due()
    lib.icb_search_profile(buf.ctypes.data_as(ctypes.c_void_p), 1)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    eng.decode_step(ctx + i, st.queries[i], st.keys[ctx + i], st.values[ctx + i], metrics=False)
    e1.record()
    torch.cuda.synchronize()
    lib.icb_search_profile(buf.ctypes.data_as(ctypes.c_void_p), 1)
    per = buf[:9] / eng.T / 1.9e3
    info = [eng.forest.info(t) for t in (0, 1)]
    print(f"step {i:3d} rot={int(rot)} {e0.elapsed_time(e1):7.3f} ms  " +
          " ".join(f"{n}={v:.0f}" for n, v in zip(names, per)) +
          f"  radix_fb={int(buf[10])} levels={info[0]['levels']}", flush=True)
