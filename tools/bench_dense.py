"""Dense skip-layer attention alone at C2 / C3 shape (16 planes x ctx rows,
bf16 K/V, G = 4): CUDA-event time per launch and HBM GB/s vs the measured
peak, for the TMA + tensor-core kernel and (ICB_DENSE_SIMT=1) the CUDA-core
kernel.   python tools/bench_dense.py [ctx ...]"""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2604_10539_b200 import dense_attention  # noqa: E402

peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
    os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0
res = []
for ctx in [int(x) for x in sys.argv[1:]] or [32768, 131072]:
    n, G, d = 16, 4, 128
    k = (torch.randn(n, ctx, d, device="cuda") / d ** 0.5).bfloat16()
    v = (torch.randn(n, ctx, d, device="cuda") / d ** 0.5).bfloat16()
    q = torch.randn(n, G, d, device="cuda") * 3
    out = torch.empty(n, G, d, device="cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for mode in ("flash", "simt"):
        if mode == "simt":
            os.environ["ICB_DENSE_SIMT"] = "1"
        else:
            os.environ.pop("ICB_DENSE_SIMT", None)
        for _ in range(3):
            dense_attention(q, k, v, ctx, out=out)
        ts = []
        for _ in range(20):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            dense_attention(q, k, v, ctx, out=out)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        ts.sort()
        ms = ts[len(ts) // 2]
        byt = 2 * n * ctx * d * 2
        res.append(dict(ctx=ctx, kernel=mode, ms=ms, bytes=byt, GBps=byt / ms / 1e6, frac=byt / ms / 1e6 / peak))
        print(json.dumps(res[-1]), flush=True)
