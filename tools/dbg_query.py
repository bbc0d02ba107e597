"""Debug helper: device query vs oracle on a golden tree for G = 1, 2, 4, 8."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from conftest import load_golden  # noqa: E402
from test_gpu_forest import _device_build, _oracle  # noqa: E402
from oracle import numerics as nm  # noqa: E402
from oracle.dci import SENTINEL  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "clu_d16"
z, meta = load_golden(f"tree_{name}.npz")
otree, _ = _oracle(z, meta)
f = _device_build(z, meta, 0)
k = meta["k"]
qs = z["queries"].astype(np.float32)
for G in (1, 2, 4, 8):
    ids, counts, pages, npages = f.query([0], qs[:G][None], k, 2 * k, 4 * k)
    torch.cuda.synchronize()
    try:
        f.check()
    except Exception as e:
        print("err", e)
    for g in range(G):
        want = otree.query(nm.lift_query32(qs[g].astype(np.float64)), SENTINEL, k, 2 * k, 4 * k)
        got = list(ids[0, g, :counts[0, g]].cpu().numpy())
        print(G, g, got == want, len(got), len(want), got[:4], want[:4], flush=True)

# no-P-DCI variant (visit cap covers every node) and evaluation counts
for cap in (4 * k, 2**40):
    e0 = f.info(0)["distance_evals"]
    o0 = otree.distance_evals
    ids, counts, _, _ = f.query([0], qs[:1][None], k, 2 * k, cap)
    want = otree.query(nm.lift_query32(qs[0].astype(np.float64)), SENTINEL, k, 2 * k, cap)
    got = list(ids[0, 0, :counts[0, 0]].cpu().numpy())
    print("cap", cap, got == want, "evals dev", f.info(0)["distance_evals"] - e0, "oracle", otree.distance_evals - o0)
