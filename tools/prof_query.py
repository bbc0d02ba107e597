"""A short C2 decode run for ncu captures of the decode kernels:
  python tools/prof_query.py [ctx] [bf16|fp32] [steps]
(the query kernel, the dense skip-layer attention, the insert kernel).
Also prints the eager step time, so the plain run is itself a check."""
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2604_10539_b200.engine import Engine, EngineConfig  # noqa: E402
from paper_2604_10539_b200.workload import clustered_stream  # noqa: E402

ctx = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
kv = sys.argv[2] if len(sys.argv) > 2 else "bf16"
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 12
C2 = dict(layers=32, kv_heads=8, query_heads_per_group=4, d=128, d_prime=128, page_size=16,
          token_budget=256, promotion_ratio=0.1, sink_pages=1, window_pages=2, skip_layers=2)
st = clustered_stream(ctx, steps, 32, 8, 4, 128, 128, device="cuda")
eng = Engine(EngineConfig(**C2, kv_dtype=kv, max_tokens=ctx + steps + 1)).prefill(st.keys, st.values, ctx)
torch.cuda.synchronize()
t0 = time.time()
for i in range(steps):
    eng.decode_step(ctx + i, st.queries[i], st.keys[ctx + i], st.values[ctx + i], metrics=False)
torch.cuda.synchronize()
eng.forest.check()
print(f"ctx {ctx} kv {kv}: {steps} steps, {(time.time() - t0) / steps * 1e3:.3f} ms/step (eager, incl. launch)")
