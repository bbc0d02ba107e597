"""BASELINE config 5 at full length: Llama-3.1-8B-shaped engine (32 layers, 2
dense skip, 8 kv heads, G = 4, d = 128, bf16 K/V), 8k-token prompt, 16,384
decode steps (~1,024 rotations x 16 device inserts per tree, trees growing
from 8,144 to ~24.5k points).  Decode through CUDA-graph replays with the
bench's clustered stream; reports whole-generation tokens/s, rotation cost,
final tree sizes, and checks every tree's invariants and sticky error bits.
  python tools/c5_long.py [prompt] [steps]"""
import json
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2604_10539_b200.dci import DciTree  # noqa: E402
from paper_2604_10539_b200.engine import Engine, EngineConfig  # noqa: E402
from paper_2604_10539_b200.workload import clustered_stream  # noqa: E402

n0 = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 16384
C2 = dict(layers=32, kv_heads=8, query_heads_per_group=4, d=128, d_prime=128, page_size=16,
          token_budget=256, promotion_ratio=0.1, sink_pages=1, window_pages=2, skip_layers=2)
st = clustered_stream(n0, steps, 32, 8, 4, 128, 128, device="cuda")
t0 = time.time()
eng = Engine(EngineConfig(**C2, kv_dtype="bf16", cuda_graph=True, max_tokens=n0 + steps + 1)).prefill(
    st.keys, st.values, n0)
torch.cuda.synchronize()
prefill_s = time.time() - t0
k_all, v_all = st.keys[n0:], st.values[n0:]
warm = 40
for i in range(warm):
    eng.decode_step(n0 + i, st.queries[i], k_all[i], v_all[i], metrics=False)
eng.capture_graphs()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
rot = 0
e0.record()
for i in range(warm, steps):
    rot += eng.rotation_due()
    eng.decode_step(n0 + i, st.queries[i], k_all[i], v_all[i], metrics=False)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
f = eng.forest
f.check()
info = [f.info(t) for t in range(eng.T)]
for t in range(0, eng.T, 40):
    DciTree.bound(f, t, f.scale(t), 0.1, 16, f.caps.tok_cap).check_invariants()
pts = [i["n_points"] for i in info]
print(json.dumps({"config": "C5: Llama-3.1-8B-shaped, 8k prompt + 16k decode", "prompt": n0, "decode_steps": steps,
                  "timed_steps": steps - warm, "rotations_timed": rot, "tokens_per_s": (steps - warm) / (ms / 1e3),
                  "ms_per_step": ms / (steps - warm), "prefill_s": round(prefill_s, 2),
                  "tree_points": {"min": min(pts), "max": max(pts)}, "levels_max": max(i["levels"] for i in info),
                  "indexed_tokens": len(eng.indexed_tokens), "invariants": "ok (every 40th tree)",
                  "errors": "none"}))
