"""Debug helper: run one decode step's device ops one by one with syncs."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2604_10539_b200.engine import Engine, EngineConfig  # noqa: E402
from paper_2604_10539_b200.workload import clustered_stream  # noqa: E402

ctx = int(sys.argv[1]); layers = int(sys.argv[2])
C2 = dict(layers=layers, kv_heads=8, query_heads_per_group=4, d=128, d_prime=128, page_size=16,
          token_budget=256, promotion_ratio=0.1, sink_pages=1, window_pages=2, skip_layers=2)
st = clustered_stream(ctx, 40, layers, 8, 4, 128, 128, device="cuda")
eng = Engine(EngineConfig(**C2, kv_dtype="bf16", max_tokens=ctx + 64)).prefill(st.keys, st.values, ctx)
torch.cuda.synchronize()
f = eng.forest
T = eng.T
print("built", [f.info(t)["levels"] for t in range(min(T, 8))], flush=True)
qi = st.queries[0][2:].reshape(T, 4, 128).contiguous()
for step in range(3):
    if step == 0 or True:
        ids, counts, pages, npages = f.query(eng.trees_dev, qi, 256, 512, 1024)
        torch.cuda.synchronize(); print("query ok", int(npages[0]), flush=True)
    f.rotate_window(eng.trees_dev, 4, eng.rot_stats)
    torch.cuda.synchronize(); print("rotate ok", f.info(0)["n_points"], flush=True)
    f.check()
