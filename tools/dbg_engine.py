"""Debug helper: C2-shaped engine, prefill + a few decode steps with phase timing."""
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2604_10539_b200.engine import Engine, EngineConfig  # noqa: E402
from paper_2604_10539_b200.workload import clustered_stream  # noqa: E402

ctx = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
layers = int(sys.argv[2]) if len(sys.argv) > 2 else 32
C2 = dict(layers=layers, kv_heads=8, query_heads_per_group=4, d=128, d_prime=128, page_size=16,
          token_budget=256, promotion_ratio=0.1, sink_pages=1, window_pages=2, skip_layers=2)
st = clustered_stream(ctx, 40, C2["layers"], 8, 4, 128, 128, device="cuda")
t0 = time.time()
eng = Engine(EngineConfig(**C2, kv_dtype="bf16", max_tokens=ctx + 64)).prefill(st.keys, st.values, ctx)
torch.cuda.synchronize()
print("prefill", time.time() - t0, flush=True)
for i in range(20):
    t0 = time.time()
    rot = eng.rotation_due()
    out, m = eng.decode_step(ctx + i, st.queries[i], st.keys[ctx + i], st.values[ctx + i])
    torch.cuda.synchronize()
    print("step", i, "rot", rot, "%.2f ms" % ((time.time() - t0) * 1e3), m.pages_selected, flush=True)
