"""Per-step device timeline of the C2 decode step: CUDA events around each
stage on the stream it runs on (main: rotation, append, search, paged
attention; side: dense skip-layer attention), printed relative to the step
start, averaged over steps."""
import collections
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2604_10539_b200 import engine as E  # noqa: E402
from paper_2604_10539_b200.engine import Engine, EngineConfig  # noqa: E402
from paper_2604_10539_b200.workload import clustered_stream  # noqa: E402

ctx = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
C2 = dict(layers=32, kv_heads=8, query_heads_per_group=4, d=128, d_prime=128, page_size=16,
          token_budget=256, promotion_ratio=0.1, sink_pages=1, window_pages=2, skip_layers=2)
steps = 48
GRAPH_WARM = int(os.environ.get("GRAPH_WARM", "0"))   # replay this many graph steps first
st = clustered_stream(ctx, steps + GRAPH_WARM, 32, 8, 4, 128, 128, device="cuda")
eng = Engine(EngineConfig(**C2, kv_dtype="bf16", max_tokens=ctx + steps + GRAPH_WARM + 1)).prefill(
    st.keys, st.values, ctx)
if GRAPH_WARM:
    eng.cfg.cuda_graph = True
    for i in range(GRAPH_WARM):
        eng.decode_step(ctx + i, st.queries[i], st.keys[ctx + i], st.values[ctx + i], metrics=False)
    torch.cuda.synchronize()
    eng.cfg.cuda_graph = False
    print("graphs captured:", sorted(eng._graphs))
base = GRAPH_WARM
f = eng.forest
marks = []


def ev():
    e = torch.cuda.Event(enable_timing=True)
    e.record(torch.cuda.current_stream())
    return e


def wrap(obj, name, label):
    orig = getattr(obj, name)

    def w(*a, **kw):
        e0 = ev()
        r = orig(*a, **kw)
        marks.append((label, e0, ev()))
        return r
    setattr(obj, name, w)


for nm, lab in [("rotate_window", "rotation"), ("append_window", "append"), ("query", "search"),
                ("attention", "paged_attn")]:
    wrap(f, nm, lab)
wrap(E, "dense_attention", "dense_attn(side)")
rows = collections.defaultdict(list)
for i in range(steps):
    marks.clear()
    s0 = ev()
    j = base + i
    eng.decode_step(ctx + j, st.queries[j], st.keys[ctx + j], st.values[ctx + j], metrics=False)
    s1 = ev()
    torch.cuda.synchronize()
    if i < 8:
        continue
    rows["step"].append((0.0, s0.elapsed_time(s1)))
    for lab, a, b in marks:
        rows[lab].append((s0.elapsed_time(a), s0.elapsed_time(b)))
print(f"{'stage':18s} {'start us':>9s} {'end us':>9s} {'dur us':>8s}  (mean over steps; rotation: its steps only)")
for lab, v in rows.items():
    a = sum(x for x, _ in v) / len(v) * 1e3
    b = sum(y for _, y in v) / len(v) * 1e3
    print(f"{lab:18s} {a:9.1f} {b:9.1f} {b - a:8.1f}")

