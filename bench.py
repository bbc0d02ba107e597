"""IceCache decode hot path on B200 -- the driver's benchmark.

Workload (BASELINE.json configs[1], "C2"): Llama-3.1-8B-shaped decode, 32
layers (first 2 dense "skip" layers, 30 DCI-indexed), GQA 32 q / 8 kv heads,
d = d' = 128, 32k-token context, 256-token budget (beam 512, visit cap 1024),
page size 16, bf16 page K/V (--kv fp32: fp32), fp32 lifted keys.  Synthetic
clustered q/k/v streams drawn on the device (reference workload distribution,
random init).  --ctx 131072 is C3 (with --kv-offload: K/V in pinned host
memory); --seqs-per-gpu S batches S sequences per GPU (C4 at S = 64 / N).

A "step" = one decode token through every layer: window rotation (every 16
tokens, 16 device inserts per tree), window append, DCI search for 32 query
heads per layer + GQA page union, sparse paged attention, dense attention of
the skip layers.  Metric: decode tokens/s.

Timing: W eager warm-up steps (they include a rotation), both step variants
captured as CUDA graphs, then EXACTLY K graph-replayed steps between CUDA
events on the launching stream (value); per-step events give the per-rotation-
period distribution.  Then K' >= 32 eager steps with CUDA events around each
search + attention launch give the dominant kernel's duration (roofline) and
the eager tokens/s; then the public-API e2e leg (pinned host I/O).

  python bench.py [--gpus N --steps K --warmup W] [--impl reference] [--check]

One process per GPU (torchrun for N > 1): rank r decodes sequences
dist.plan_rank(total, N, r) (sequence-parallel, no collective), value =
tokens of all ranks / max rank time.  `--impl reference` times the
UNMODIFIED reference package (pip-installed into baseline/_ref) on the host
cores on a bounded sample of the same workload.  `--check` diffs the bench
engine's selections on a C2-shaped slice drawn with the NumPy generator
against the reference's golden run.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

E2E_STEPS = 64
E2E_SEGMENTS = 3   # e2e throughput = median of the segments (one host stall cannot dominate)
E2E_WARM = 4       # untimed steps through the host-I/O path first (copy streams, staging buffers)
METRIC = "decode tokens/s (TPOT) at 32k ctx, 256-token budget; DCI top-k query µs/head"
C2 = dict(layers=32, kv_heads=8, query_heads_per_group=4, d=128, d_prime=128, page_size=16,
          token_budget=256, promotion_ratio=0.1, sink_pages=1, window_pages=2, skip_layers=2)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=256)
    ap.add_argument("--warmup", type=int, default=16)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--ctx", type=int, default=32768)
    ap.add_argument("--kv", default="bf16", choices=["bf16", "fp32"])
    ap.add_argument("--layer-serial", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="e2e leg without CUDA graphs")
    ap.add_argument("--fuse-rotation", action="store_true",
                    help="rotation steps as one icb_step_attend launch (A/B; off by default)")
    ap.add_argument("--reuse-stride", type=int, default=0,
                    help="selection reuse (anchor layers, engine.py:321-363); 0 = the reference default (off)")
    ap.add_argument("--kv-offload", action="store_true",
                    help="BASELINE config 3: page K/V in pinned host memory, per-step HBM page pool")
    ap.add_argument("--seqs-per-gpu", type=int, default=1,
                    help="BASELINE config 4: S independent sequences per GPU, decoded in lockstep in the same "
                         "launches (their trees side by side: kv_heads x S)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--check", action="store_true",
                    help="diff the bench engine's selections on a C2-shaped slice against the reference golden")
    ap.add_argument("--seed", type=int, default=0)
    return ap.parse_args()


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """SM clock and throttle reasons polled through NVML every 5 ms while the
    timed region runs (nvidia-smi's own loop is too coarse for a ~100 ms
    region); falls back to nvidia-smi -lms when NVML is unavailable."""

    REASONS = {"hw_slowdown": "nvmlClocksEventReasonHwSlowdown",
               "hw_thermal_slowdown": "nvmlClocksEventReasonHwThermalSlowdown",
               "hw_power_brake_slowdown": "nvmlClocksEventReasonHwPowerBrakeSlowdown",
               "sw_thermal_slowdown": "nvmlClocksEventReasonSwThermalSlowdown",
               "sw_power_cap": "nvmlClocksEventReasonSwPowerCap"}

    def __init__(self, index=0, period_s=0.005):
        self.index = index
        self.period = period_s
        self.sm, self.mx, self.reasons = [], 0.0, set()
        self.stop = threading.Event()
        self.t = None

    def __enter__(self):
        try:
            import pynvml as nv
            nv.nvmlInit()
            h = nv.nvmlDeviceGetHandleByIndex(self.index)
            self.mx = float(nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM))
            bits = {k: getattr(nv, v) for k, v in self.REASONS.items() if hasattr(nv, v)}

            def poll():
                while True:
                    try:
                        self.sm.append(float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)))
                        r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                        self.reasons |= {k for k, b in bits.items() if r & b}
                    except Exception:
                        pass
                    if self.stop.wait(self.period):
                        return
            self.t = threading.Thread(target=poll, daemon=True)
            self.t.start()
        except Exception:
            self.t = None
        return self

    def __exit__(self, *a):
        self.stop.set()
        if self.t:
            self.t.join(timeout=2)

    def summary(self):
        return {"sm_mhz": statistics.median(self.sm) if self.sm else None, "sm_max_mhz": self.mx or None,
                "reasons": sorted(self.reasons), "samples": len(self.sm), "source": "nvml 5 ms poll"}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


# ------------------------------------------------------------------ our arm
def workload_label(args):
    name = {32768: "C2", 131072: "C3"}.get(args.ctx, "C2-shaped")
    if args.seqs_per_gpu > 1:
        name = f"C4 slice ({args.seqs_per_gpu} sequences per GPU)"
    kv = "K/V in pinned host memory + per-step HBM page pool" if args.kv_offload else "K/V in HBM"
    return (f"{name}: Llama-3.1-8B-shaped decode, 32 layers (2 dense skip + 30 DCI-indexed), GQA 32q/8kv, "
            f"d=128, {args.ctx // 1024}k ctx, budget 256, page 16, {args.kv} KV, {kv}")


def traffic_key(args):
    return f"ctx{args.ctx}_{args.kv}_s{args.seqs_per_gpu}" + ("_offload" if args.kv_offload else "") + \
        (f"_reuse{args.reuse_stride}" if args.reuse_stride else "")


def run_ours(args, rank, world):
    import numpy as np
    import torch

    from paper_2604_10539_b200.dist import max_over_ranks, plan_rank
    from paper_2604_10539_b200.engine import Engine, EngineConfig
    from paper_2604_10539_b200.workload import clustered_stream

    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", 0)))
    torch.cuda.set_device(dev)
    K, W = args.steps, args.warmup
    if W < 3:
        raise SystemExit("--warmup must be >= 3")
    KT = max(32, K)                      # eager kernel-timing segment
    n0 = args.ctx
    total_steps = W + K + KT + E2E_WARM + E2E_SEGMENTS * E2E_STEPS + 1
    plan = plan_rank(args.seqs_per_gpu * world, world, rank, args.seed)
    S = plan.per_gpu
    # S sequences of equal length: per (layer, kv head) trees are independent and
    # rotate in lockstep, so the batch is the model with kv_heads x S
    cS = dict(C2, kv_heads=C2["kv_heads"] * S)
    # several sequences per GPU: the prompt stream in bf16 (its K/V plus the forest
    # must fit HBM together; the engine converts it per chunk of layers)
    stream = clustered_stream(n0, total_steps, cS["layers"], cS["kv_heads"], cS["query_heads_per_group"],
                              cS["d"], cS["d_prime"], seed=plan.seed, device=dev,
                              dtype=torch.bfloat16 if S > 1 else torch.float32)
    cfg = EngineConfig(**cS, seed=plan.seed, kv_dtype=args.kv, max_tokens=n0 + total_steps + 1,
                       layer_serial=args.layer_serial, cuda_graph=False, reuse_stride=args.reuse_stride,
                       fuse_rotation=args.fuse_rotation, kv_offload=args.kv_offload)
    t0 = time.time()
    eng = Engine(cfg, device=dev).prefill(stream.keys, stream.values, n0)
    torch.cuda.synchronize()
    prefill_s = time.time() - t0
    q_all = stream.queries
    k_all = stream.keys[n0:]
    v_all = stream.values[n0:]
    cur = torch.cuda.current_stream()
    f = eng.forest
    fused_rot = eng.cfg.fuse_rotation and args.reuse_stride < 2
    base_launches = 4 if args.reuse_stride < 2 else 6

    def step(i):
        rot = eng.rotation_due()
        eng.decode_step(n0 + i, q_all[i], k_all[i], v_all[i], metrics=False)
        # library kernels per step: window append, search + paged attention
        # (reuse: anchor search, pages_from_tokens, paged attention), dense
        # append, dense attention, + the rotation insert kernel; a fused
        # rotation step is one launch for rotation + append + search + attention
        return rot, (3 if (rot and fused_rot) else base_launches + (1 if rot else 0))

    # ---- warm-up (eager: first use of every kernel and scratch, incl. a rotation)
    seen = set()
    for i in range(W):
        seen.add(step(i)[0])
    j = W
    while seen != {False, True}:          # only when the prompt length makes step 0 plain
        seen.add(step(j)[0])
        j += 1
    if not args.no_graph:
        eng.cfg.cuda_graph = True
        eng.capture_graphs()
    torch.cuda.synchronize()

    # ---- timed region: exactly K steps (graph replays unless --no-graph)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(K + 1)]
    launches = 0
    rot_steps = []
    info0 = [f.info(t) for t in range(eng.T)]
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    with ClockSampler(dev.index) as clk:
        ev[0].record(cur)
        for k in range(K):
            r, nl = step(j + k)
            launches += nl
            if r:
                rot_steps.append(k)
            ev[k + 1].record(cur)
        torch.cuda.synchronize()
    ms = ev[0].elapsed_time(ev[K])
    step_ms = [ev[k].elapsed_time(ev[k + 1]) for k in range(K)]
    j += K
    ms_max = max_over_ranks(ms, dev)
    tokens_per_s = world * S * K / (ms_max / 1e3)
    info_t = [f.info(t) for t in range(eng.T)]
    # whole 16-step rotation periods inside the timed region
    periods = []
    for a, b in zip(rot_steps, rot_steps[1:]):
        periods.append(S * (b - a) / (sum(step_ms[a:b]) / 1e3))

    # ---- kernel timing: eager steps, CUDA events around the search + attention launch
    eng.cfg.cuda_graph = False
    ev_q0 = [torch.cuda.Event(enable_timing=True) for _ in range(KT)]
    ev_q1 = [torch.cuda.Event(enable_timing=True) for _ in range(KT)]
    timing = {"i": None}
    orig_qa, orig_q, orig_a = f.query_attend, f.query, f.attention

    def around(fn, first, last):
        def wrapped(*a, **kw):
            i = timing["i"]
            if i is not None and first:
                ev_q0[i].record(cur)
            r = fn(*a, **kw)
            if i is not None and last:
                ev_q1[i].record(cur)
            return r
        return wrapped

    if args.reuse_stride >= 2:
        f.query, f.attention = around(orig_q, True, False), around(orig_a, False, True)
    else:
        f.query_attend = around(orig_qa, True, True)
    stats0 = eng.stats.sum(0).cpu().numpy().copy()
    pool0 = f.pool_stats()[:, 0].sum() if args.kv_offload else 0
    info1 = [f.info(t) for t in range(eng.T)]
    fixed_tok = 0
    kt_rot = set()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(cur)
    for i in range(KT):
        timing["i"] = i
        r, _ = step(j + i)
        if r:
            kt_rot.add(i)
        fixed_tok += eng.T * (C2["page_size"] * C2["sink_pages"] + sum(eng._win_fills))
    timing["i"] = None
    e1.record(cur)
    torch.cuda.synchronize()
    eager_ms = e0.elapsed_time(e1)
    j += KT
    f.query_attend, f.query, f.attention = orig_qa, orig_q, orig_a
    info2 = [f.info(t) for t in range(eng.T)]
    stats1 = eng.stats.sum(0).cpu().numpy().copy()
    pool1 = f.pool_stats()[:, 0].sum() if args.kv_offload else 0
    f.check()
    # a fused rotation step's launch also carries that step's inserts: not a roofline sample
    samples = [i for i in range(KT) if not (fused_rot and i in kt_rot)]
    launch_ms = [ev_q0[i].elapsed_time(ev_q1[i]) for i in samples]
    # algorithmic bytes of the launch: search 4(d+1) U + 4 E, attention
    # 2 d b_kv per attended token (sink, window, selected pages)
    rows = sum(b["rows_read"] - a["rows_read"] for a, b in zip(info1, info2))
    rere = sum(b["owner_rereads"] - a["owner_rereads"] for a, b in zip(info1, info2))
    evals = sum(b["distance_evals"] - a["distance_evals"] for a, b in zip(info1, info2))
    U = rows - rere
    search_bytes = (4 * (C2["d"] + 1) * U + 4 * evals) / KT
    kv_b = 2 if args.kv == "bf16" else 4
    attn_tokens = (float(stats1[1] - stats0[1]) + fixed_tok) / KT
    attn_bytes = attn_tokens * (C2["d"] + C2["d_prime"]) * kv_b
    launch_bytes = search_bytes + (attn_bytes if args.reuse_stride < 2 else 0.0)
    launch_s = statistics.median(launch_ms) / 1e3
    peak, peak_kind = peaks()
    achieved = launch_bytes / launch_s / 1e9
    heads = eng.T * C2["query_heads_per_group"]
    # the timed region's own counters agree with the kernel-timing segment's
    evals_timed = sum(b["distance_evals"] - a["distance_evals"] for a, b in zip(info0, info_t)) / K

    # ---- e2e: the next steps through the public API with host (pinned) inputs/outputs
    eng.cfg.cuda_graph = not args.no_graph
    e2e_val = run_e2e(eng, stream, n0, j, E2E_STEPS, dev, world, E2E_SEGMENTS, seqs=S)

    traffic, traffic_src = read_ncu_traffic(traffic_key(args))
    offload = None
    if args.kv_offload:
        offload = offload_report(args, dev, float(pool1 - pool0) / KT, eager_ms / KT)
    res = {
        "metric": METRIC, "value": tokens_per_s, "unit": "tokens/s", "n_gpus": world, "steps": K, "warmup": W,
        "ms_per_step": ms_max / K, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "fp32 search keys / bf16 KV / fp32 accum" if args.kv == "bf16" else "fp32",
        "data": "synthetic clustered q/k/v (reference workload distribution), random init, drawn on device" +
                (" (prompt K/V bf16-representable: the multi-sequence stream is held in bf16)" if S > 1 else ""),
        "config": {"workload": workload_label(args), "context": n0, "budget": 256, "beam": 512, "visit_cap": 1024,
                   "page_size": 16, "layers": 32, "kv_heads": 8, "q_heads": 32, "kv_dtype": args.kv,
                   "sequences_per_gpu": S, "sequences": list(plan.sequences), "global_batch": S * world,
                   "parallelism": f"sequence-parallel x{world} (no collective)",
                   "layer_mode": "layer-serial" if args.layer_serial else "layers batched per step",
                   "step_execution": "eager launches" if args.no_graph else
                   "CUDA-graph replays (plain / rotating step variants captured before the timed region)",
                   "rotations_in_timed_region": len(rot_steps), "reuse_stride": args.reuse_stride,
                   "l2": "per-step working set ~1.4 GB > 126 MB L2; no flush",
                   "prefill_s": round(prefill_s, 2),
                   "kv": "pinned host + per-step HBM page pool (config 3)" if args.kv_offload else "HBM resident"},
        "step_ms": {"median": statistics.median(step_ms), "mean": statistics.mean(step_ms),
                    "max": max(step_ms), "rotation_step_median": statistics.median([step_ms[k] for k in rot_steps])
                    if rot_steps else None},
        "period_tokens_per_s": {"median": statistics.median(periods) if periods else None,
                                "n_periods": len(periods),
                                "note": "tokens/s over each whole 16-step rotation period of the timed region"},
        "eager_tokens_per_s": world * S * KT / (max_over_ranks(eager_ms, dev) / 1e3),
        "roofline": {"bound": "hbm", "kernel": "query_kernel (DCI search + top-k + page union + fused sparse "
                                               "attention)" if args.reuse_stride < 2 else "query_kernel (anchors) "
                                                                                         "+ attn_kernel",
                     "achieved": achieved, "peak": peak, "peak_kind": peak_kind, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic, "traffic_source": traffic_src,
                     "alg_bytes_per_launch": launch_bytes, "alg_bytes_search": search_bytes,
                     "alg_bytes_attention": attn_bytes, "launch_ms": launch_s * 1e3,
                     "launch_ms_mean": statistics.mean(launch_ms),
                     "launch_timing": f"median of {len(launch_ms)} launches: CUDA events around each search + "
                                      "attention launch on its stream, eager steps right after the timed region",
                     "unique_rows_per_step": U / KT, "evals_per_step": evals / KT,
                     "evals_per_step_timed_region": evals_timed},
        "dci_topk_us_per_head": launch_s * 1e6 / heads,
        "attended_tokens_per_step": attn_tokens,
        "gpu_launches": launches,
        **({"kv_offload": offload} if offload else {}),
        "clocks": clk.summary(),
        "e2e": e2e_val,
    }
    return res


def offload_report(args, dev, gathered, step_ms):
    """Host-link use of the page gather vs a plain pinned H2D copy on this box."""
    import torch
    hb = torch.empty(256 << 20, dtype=torch.uint8).pin_memory()
    db = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    for _ in range(2):
        db.copy_(hb, non_blocking=True)
    c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    c0.record()
    for _ in range(4):
        db.copy_(hb, non_blocking=True)
    c1.record()
    torch.cuda.synchronize()
    h2d_peak = 4 * hb.numel() / (c0.elapsed_time(c1) / 1e3) / 1e9
    del hb, db
    link = gathered / (step_ms / 1e3) / 1e9
    return {"gathered_bytes_per_step": gathered, "host_link_GBps": link, "pinned_h2d_peak_GBps": h2d_peak,
            "link_frac": link / h2d_peak,
            "mechanism": "K/V of all pages in pinned device-mapped host memory; each tree's CTA gathers the step's "
                         "missing pages (filled rows, 16-B loads) into its HBM pool after its search, overlapping "
                         "other trees' searches; resident pages are kept"}


def run_e2e(eng, stream, n0, start, K2, dev, world, segments=1, seqs=1):
    """Same metric through Engine.decode_step with pinned host inputs (H2D)
    and the step's outputs read back to pinned host memory (D2H) inside the
    timed region; whole-job tokens over the slowest rank's wall time.  The
    value is the median over `segments` consecutive K2-step segments (Python's
    cyclic GC is paused while timing, as a serving loop would)."""
    import gc

    import torch

    from paper_2604_10539_b200.dist import max_over_ranks
    n = K2 * segments + E2E_WARM
    qh = stream.queries[start:start + n].float().cpu().pin_memory()
    kh = stream.keys[n0 + start:n0 + start + n].float().cpu().pin_memory()
    vh = stream.values[n0 + start:n0 + start + n].float().cpu().pin_memory()
    outh = torch.empty((n,) + (qh.shape[1], qh.shape[2], stream.values.shape[-1]), dtype=torch.float32).pin_memory()
    if eng.steps_done != start:
        return None
    vals = []
    for i in range(E2E_WARM):   # untimed: first use of the host-I/O path
        eng.decode_step(n0 + start + i, qh[i], kh[i], vh[i], metrics=False, out=outh[i])
    torch.cuda.synchronize()
    gc.disable()
    try:
        for sgm in range(segments):
            torch.cuda.synchronize()
            if world > 1:
                torch.distributed.barrier()
            t0 = time.perf_counter()
            for i in range(E2E_WARM + sgm * K2, E2E_WARM + (sgm + 1) * K2):
                # host (pinned) inputs in, host output back: the engine stages both
                # through its copy streams (the D2H is complete at the synchronize)
                eng.decode_step(n0 + start + i, qh[i], kh[i], vh[i], metrics=False, out=outh[i])
            torch.cuda.synchronize()
            dt = max_over_ranks(time.perf_counter() - t0, dev)
            vals.append(world * seqs * K2 / dt)
    finally:
        gc.enable()
    h2d = (qh[0].numel() + kh[0].numel() + vh[0].numel()) * 4
    d2h = outh[0].numel() * 4
    return {"value": statistics.median(vals), "unit": "tokens/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
            "steps": K2 * segments, "untimed_warmup_steps": E2E_WARM, "segments": [round(v, 1) for v in vals],
            "path": "Engine.decode_step (public API) -> C ABI; pinned host q/k/v in, pinned host outputs back"}


def read_ncu_traffic(key):
    """DRAM bytes per launch of the dominant kernel from the ncu capture of the
    same configuration (profiles/search_traffic.json, keyed by config)."""
    p = os.path.join(ROOT, "profiles", "search_traffic.json")
    try:
        with open(p) as fh:
            ent = json.load(fh).get(key)
        if ent:
            return ent["dram_bytes_per_launch"], ent.get("source", "ncu")
    except Exception:
        pass
    return None, f"no ncu capture of config {key}"


# ------------------------------------------------------------------ CPU legs
REF_PATH = os.path.join(ROOT, "baseline", "_ref")


def import_reference():
    """The UNMODIFIED reference package, pip-installed into baseline/_ref."""
    if not os.path.isdir(os.path.join(REF_PATH, "icecache")):
        raise RuntimeError("baseline/_ref is missing: run __graft_entry__.build() (pip install --target baseline/_ref)")
    if REF_PATH not in sys.path:
        sys.path.insert(0, REF_PATH)
    import icecache
    return icecache


def ref_sample(rank, steps, warm, ctx, seed, barrier=None, out=None):
    """One process's bounded sample of the C2 step on the unmodified reference:
    a 1-layer, 1-kv-head, G = 4 Engine (one indexed (layer, kv head) group,
    skip_layers = 0) over a 32k prompt drawn by the reference's own
    generate_workload, plus one dense skip-layer head (the reference's
    full_attention over the whole context, what its engine runs for layers <
    skip_layers).  Per step: one group decode_step (rotation when due, G
    searches, union, backload, sparse attention, evict) and one dense head."""
    import numpy as np
    ic = import_reference()
    spec = ic.WorkloadSpec(kind="clustered", n_tokens=ctx + warm + steps + 1, d=128, d_prime=128, clusters=32,
                           layers=1, kv_heads=1, query_heads_per_group=4, seed=seed)
    wl = ic.generate_workload(spec)
    cfg = ic.EngineConfig(layers=1, kv_heads=1, query_heads_per_group=4, d=128, d_prime=128, page_size=16,
                          token_budget=256, promotion_ratio=0.1, skip_layers=0, seed=seed)
    t0 = time.perf_counter()
    eng = ic.Engine(cfg).prefill(wl, ctx)
    build_s = time.perf_counter() - t0
    kd, vd = wl.keys[: ctx + 1, 0, 0], wl.values[: ctx + 1, 0, 0]
    group_s, dense_s, q_us, step_s = [], [], [], []
    orig = eng._select_tokens

    def timed_select(*a, **kw):
        tq = time.perf_counter()
        r = orig(*a, **kw)
        q_us.append((time.perf_counter() - tq) * 1e6)
        return r
    eng._select_tokens = timed_select
    for t in range(warm + steps):
        if barrier is not None:
            barrier.wait()
        ts = time.perf_counter()
        eng.decode_step(wl.decode_step(ctx, t))
        tg = time.perf_counter()
        ic.full_attention(wl.queries[ctx + t, 0, 0], kd, vd)
        te = time.perf_counter()
        if t >= warm:
            group_s.append(tg - ts)
            dense_s.append(te - tg)
            step_s.append(te - ts)
    res = dict(group_s=group_s, dense_s=dense_s, step_s=step_s, query_us=q_us[4 * warm:], build_s=build_s)
    if out is not None:
        out.put((rank, res))
    return res


def ref_value(group_s, dense_s, procs):
    """tokens/s of the full C2 step (240 indexed groups + 64 dense q heads)
    spread over `procs` host processes, from per-group / per-dense-head times."""
    per_token = (240 * statistics.median(group_s) + 64 * statistics.median(dense_s)) / procs
    return 1.0 / per_token


def cpu_baseline_leg(ctx):
    """Rank 0, N = 1: the reference on one host core, bounded sample."""
    r = ref_sample(0, 4, 1, ctx, 0)
    return {"value": ref_value(r["group_s"], r["dense_s"], 1), "unit": "tokens/s", "cores": 1, "kind": "reference",
            "sample": f"unmodified reference (baseline/_ref icecache) Engine, one {ctx // 1024}k (layer, kv head) "
                      f"G=4 group: prefill {r['build_s']:.1f}s, 4 decode steps timed + 4 dense skip-layer heads; "
                      f"x240 groups + 64 dense heads per token; DciTree.query "
                      f"{statistics.median(r['query_us']):.0f} us/head"}


def run_reference(args):
    """--impl reference: the unmodified reference package on all host cores,
    one process per core, each its own (layer, kv head) group; each step =
    every process's group decode step + one dense head, in lockstep."""
    import multiprocessing as mp
    ncores = len(os.sched_getaffinity(0))
    nproc = max(1, min(ncores, 16))
    # one BLAS thread per process: the processes are the parallelism
    for var in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS", "MKL_NUM_THREADS"):
        os.environ[var] = "1"
    ctx = mp.get_context("fork")
    bar = ctx.Barrier(nproc)
    q = ctx.Queue()
    t0 = time.time()
    procs = [ctx.Process(target=ref_sample, args=(r, args.steps, args.warmup, args.ctx, args.seed + r, bar, q))
             for r in range(nproc)]
    for p in procs:
        p.start()
    res = dict(q.get() for _ in procs)
    for p in procs:
        p.join()
    wall = time.time() - t0
    group = [x for r in res.values() for x in r["group_s"]]
    dense = [x for r in res.values() for x in r["dense_s"]]
    steps = [max(res[r]["step_s"][i] for r in res) for i in range(args.steps)]
    value = ref_value(group, dense, nproc)
    frac = (nproc / 240.0)
    return {"impl": "reference", "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": 0,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": statistics.mean(steps) * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "fp64 (NumPy)",
            "data": "synthetic clustered (the reference's generate_workload)",
            "config": {"workload": f"C2 sample: {nproc} processes x one {args.ctx // 1024}k (layer, kv head) G=4 "
                                   "group + one dense head per step", "context": args.ctx, "budget": 256,
                       "sample_fraction_of_token": f"{nproc}/240 indexed groups + {nproc}/64 dense heads per step",
                       "value_from": "per-group and per-dense-head median step times, (240 t_group + 64 t_dense) "
                                     "/ processes per token"},
            "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": nproc, "kind": "reference",
                             "sample": f"unmodified reference (baseline/_ref) Engine + full_attention, {nproc} "
                                       f"processes, {args.steps} timed steps each, wall {wall:.1f}s incl. prefill"},
            "dci_topk_us_per_head": statistics.median([x for r in res.values() for x in r["query_us"]]),
            "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


# ------------------------------------------------------------------ --check
def run_check(args):
    """The bench's engine configuration (bf16 KV, CUDA graphs) on a C2-shaped
    slice drawn with the NumPy generator (reference draws), against the
    reference's golden run tests/golden/engine_c2_s0.npz: every step metric and
    every query head's ranked token list."""
    import numpy as np
    import torch

    from paper_2604_10539_b200.engine import Engine, EngineConfig
    from paper_2604_10539_b200.workload import WorkloadSpec, generate_workload
    z = np.load(os.path.join(ROOT, "tests", "golden", "engine_c2_s0.npz"))
    meta = json.loads(str(z["meta"]))
    sk, ck = meta["spec"], meta["cfg"]
    wl = generate_workload(WorkloadSpec(kind="clustered", **sk))
    for a in (wl.keys, wl.values, wl.queries):
        a[:] = a.astype(np.float32).astype(np.float64)
    n0, steps = meta["n_prefill"], meta["steps"]
    cfg = EngineConfig(layers=sk["layers"], kv_heads=sk["kv_heads"], query_heads_per_group=sk["query_heads_per_group"],
                       d=sk["d"], d_prime=sk["d_prime"], seed=sk["seed"], kv_dtype=args.kv, cuda_graph=True,
                       max_tokens=n0 + steps + 1, **ck)
    dev = torch.device("cuda", 0)
    eng = Engine(cfg, device=dev).prefill(wl.keys, wl.values, n0)
    q = torch.as_tensor(wl.queries, dtype=torch.float32, device=dev)
    k = torch.as_tensor(wl.keys, dtype=torch.float32, device=dev)
    v = torch.as_tensor(wl.values, dtype=torch.float32, device=dev)
    G, H = cfg.query_heads_per_group, cfg.kv_heads
    lists = exact = 0
    set_equal = 0
    for t in range(steps):
        tok = n0 + t
        eng.decode_step(tok, q[tok], k[tok], v[tok], metrics=False)
        ids, counts, _, _ = eng.selected()
        for i, (layer, h) in enumerate(meta["calls"]):
            tr, g = (layer - cfg.skip_layers) * H + h, i % G
            got = [int(x) for x in ids[tr, g, :counts[tr, g]]]
            want = [int(x) for x in z["tokens"][t, i] if x >= 0]
            lists += 1
            exact += got == want
            set_equal += set(got) == set(want)
    out = {"check": "c2_slice_vs_reference_golden", "kv": args.kv, "graphs": True, "lists": lists,
           "ranked_identical": exact, "sets_identical": set_equal,
           "ok": set_equal == lists}
    return out


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if args.check:
        if rank == 0:
            print(json.dumps(run_check(args)), flush=True)
        return
    if args.impl == "reference":
        if rank == 0:
            print(json.dumps(run_reference(args)), flush=True)
        return
    if world > 1:
        # NCCL's init lines (nranks, NVLS / P2P transport) go to the log, so a
        # scaling run shows every rank joined the communicator
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        import torch
        dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", 0)))
        torch.cuda.set_device(dev)
        torch.distributed.init_process_group("nccl", device_id=dev)
    res = run_ours(args, rank, world)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        res["cpu_baseline"] = cpu_baseline_leg(32768)
    if rank == 0:
        print(json.dumps(res), flush=True)
    if world > 1:
        import torch
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
