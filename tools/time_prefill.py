"""Where Engine.prefill's time goes at C2 (device build vs host/torch work)."""
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2604_10539_b200 import forest as FM  # noqa: E402
from paper_2604_10539_b200.engine import Engine, EngineConfig  # noqa: E402
from paper_2604_10539_b200.workload import clustered_stream  # noqa: E402

ctx = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
C2 = dict(layers=32, kv_heads=8, query_heads_per_group=4, d=128, d_prime=128, page_size=16,
          token_budget=256, promotion_ratio=0.1, sink_pages=1, window_pages=2, skip_layers=2)
st = clustered_stream(ctx, 4, 32, 8, 4, 128, 128, device="cuda")
torch.cuda.synchronize()
times = {}
orig_build = FM.DeviceForest.build


def timed_build(self, *a, **kw):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = orig_build(self, *a, **kw)
    torch.cuda.synchronize()
    times["build"] = times.get("build", 0.0) + time.perf_counter() - t0
    return r


FM.DeviceForest.build = timed_build
for rep in range(2):
    times.clear()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    eng = Engine(EngineConfig(**C2, kv_dtype="bf16", max_tokens=ctx + 8, kv_offload=bool(os.environ.get("KVOFF")))).prefill(st.keys, st.values, ctx)
    torch.cuda.synchronize()
    total = time.perf_counter() - t0
    print(f"prefill {total:.3f}s  device build {times.get('build', 0):.3f}s  other {total - times.get('build', 0):.3f}s")
    del eng
    torch.cuda.empty_cache()

if os.environ.get("KPROF"):
    from torch.profiler import profile, ProfilerActivity
    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
        eng = Engine(EngineConfig(**C2, kv_dtype="bf16", max_tokens=ctx + 8, kv_offload=bool(os.environ.get("KVOFF")))).prefill(st.keys, st.values, ctx)
        torch.cuda.synchronize()
    print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=15, max_name_column_width=50))

if os.environ.get("ICB_PROF"):
    import ctypes
    import numpy as np
    from paper_2604_10539_b200 import _native as N
    buf = np.zeros(4, dtype=np.uint64)
    N.lib().icb_build_profile(ctypes.c_void_p(buf.ctypes.data), 0)
    print("parent filter: points %d, exact chains %.1f per point, window overflows %.3f%%" % (
        buf[0], buf[1] / max(1, buf[0]), 100.0 * buf[2] / max(1, buf[0])))
