"""Device time of rotation steps vs plain steps at C2, fused rotation
(icb_step_attend) vs separate launches: CUDA events around each eager step."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2604_10539_b200.engine import Engine, EngineConfig  # noqa: E402
from paper_2604_10539_b200.workload import clustered_stream  # noqa: E402

ctx = 32768
C2 = dict(layers=32, kv_heads=8, query_heads_per_group=4, d=128, d_prime=128, page_size=16,
          token_budget=256, promotion_ratio=0.1, sink_pages=1, window_pages=2, skip_layers=2)
steps = 96
st = clustered_stream(ctx, steps, 32, 8, 4, 128, 128, device="cuda")
for fuse in (True, False, True, False):
    eng = Engine(EngineConfig(**C2, kv_dtype="bf16", max_tokens=ctx + steps + 1, fuse_rotation=fuse)).prefill(
        st.keys, st.values, ctx)
    rot, plain = [], []
    for i in range(steps):
        r = eng.rotation_due()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        eng.decode_step(ctx + i, st.queries[i], st.keys[ctx + i], st.values[ctx + i], metrics=False)
        e1.record()
        torch.cuda.synchronize()
        if i >= 16:
            (rot if r else plain).append(e0.elapsed_time(e1))
    print(f"fuse={fuse}: rotation steps {sum(rot) / len(rot):.3f} ms (n={len(rot)}), "
          f"plain steps {sum(plain) / len(plain):.3f} ms")
    del eng
    torch.cuda.empty_cache()
