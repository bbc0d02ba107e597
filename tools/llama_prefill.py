"""Prefill pipelining with a model forward in the loop (SURVEY §8(f) ranks 2
and 4): a Llama-3.1-8B-shaped LlamaModel (transformers, random init, bf16 --
no checkpoint is reachable) runs the prompt forward; its post-RoPE K/V of
every layer go to the engine, and its q/k/v of the next tokens drive decode
steps.

  serial     forward over the prompt, then Engine.prefill(all layers' K/V)
  pipelined  Engine.prefill_layers: each layer's K/V handed over from inside
             the forward (an attention hook); that layer's trees build on the
             engine's stream while the model computes the next layers

Prints one JSON line: forward-only, serial and pipelined time to first token
(prefill), the build's share, and the engine's decode TPOT on the model's
q/k/v.   python tools/llama_prefill.py [n_prompt] [decode_steps]
"""
import json
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2604_10539_b200.engine import Engine, EngineConfig  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
D = int(sys.argv[2]) if len(sys.argv) > 2 else 64
GROUP = int(sys.argv[3]) if len(sys.argv) > 3 else 4
from transformers import AttentionInterface, LlamaConfig, LlamaModel  # noqa: E402
from transformers.integrations.sdpa_attention import sdpa_attention_forward  # noqa: E402

state = {"mode": None, "k": {}, "v": {}, "q": {}, "pf": None}


def hook(module, query, key, value, attention_mask, **kw):
    layer = module.layer_idx
    if state["mode"] == "serial":
        state["k"][layer] = key[0].permute(1, 0, 2).contiguous()        # [S, H, D] post-RoPE
        state["v"][layer] = value[0].permute(1, 0, 2).contiguous()
        state["q"][layer] = query[0, :, n:].permute(1, 0, 2).contiguous()   # decode positions' queries
    elif state["mode"] == "pipelined":
        state["pf"].layer(layer, key[0].permute(1, 0, 2), value[0].permute(1, 0, 2))
    return sdpa_attention_forward(module, query, key, value, attention_mask, **kw)


AttentionInterface.register("icecache_hook", hook)
cfg = LlamaConfig(vocab_size=128256, hidden_size=4096, intermediate_size=14336, num_hidden_layers=32,
                  num_attention_heads=32, num_key_value_heads=8, head_dim=128, max_position_embeddings=n + D + 16,
                  rope_theta=500000.0, attn_implementation="icecache_hook")
torch.manual_seed(0)
t0 = time.time()
with torch.device("cuda"):
    model = LlamaModel(cfg).to(torch.bfloat16).eval()
init_s = time.time() - t0
ids = torch.randint(0, cfg.vocab_size, (1, n + D), device="cuda", generator=torch.Generator("cuda").manual_seed(1))
ecfg = dict(layers=32, kv_heads=8, query_heads_per_group=4, d=128, d_prime=128, page_size=16, token_budget=256,
            skip_layers=2, kv_dtype="bf16", max_tokens=n + D + 1)


def timed(fn):
    torch.cuda.synchronize()
    t = time.perf_counter()
    r = fn()
    torch.cuda.synchronize()
    return r, time.perf_counter() - t


with torch.no_grad():
    state["mode"] = None
    _, fwd_warm = timed(lambda: model(input_ids=ids[:, :n], use_cache=False))     # warm-up (kernels, allocator)
    _, fwd_s = timed(lambda: model(input_ids=ids[:, :n], use_cache=False))
    # serial: forward (prompt + decode positions, capturing q/k/v), then the whole prefill
    state["mode"] = "serial"
    _, fwd_cap_s = timed(lambda: model(input_ids=ids, use_cache=False))
    keys = torch.stack([state["k"][l] for l in range(32)], 1)        # [n + D, L, H, d]
    values = torch.stack([state["v"][l] for l in range(32)], 1)
    queries = torch.stack([state["q"][l] for l in range(32)], 1)     # [D, L, Hq, d]
    state["k"].clear(); state["v"].clear(); state["q"].clear()
    warm = Engine(EngineConfig(**dict(ecfg, max_tokens=4096 + 8))).prefill(keys[:4096], values[:4096], 4096)
    del warm                                                          # first use of every build kernel
    eng, build_s = timed(lambda: Engine(EngineConfig(**ecfg)).prefill(keys, values, n))
    # pipelined: the trees of each layer build while the model runs the next layers
    state["mode"] = "pipelined"
    eng2 = Engine(EngineConfig(**ecfg))

    def pipelined():
        state["pf"] = eng2.prefill_layers(n, group=GROUP)
        model(input_ids=ids[:, :n], use_cache=False)
        return state["pf"].finish()
    _, pipe_s = timed(pipelined)
    state["mode"] = None
    same = all(eng.forest.export(t)["nodes"] == eng2.forest.export(t)["nodes"] for t in range(0, eng.T, 37))
    # decode on the model's q/k/v (the engine's part of TPOT)
    k_dec, v_dec = keys[n:].float(), values[n:].float()
    for i in range(4):
        eng.decode_step(n + i, queries[i].float(), k_dec[i], v_dec[i], metrics=False)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(4, D):
        eng.decode_step(n + i, queries[i].float(), k_dec[i], v_dec[i], metrics=False)
    e1.record()
    torch.cuda.synchronize()
    tpot = e0.elapsed_time(e1) / (D - 4)
print(json.dumps({
    "model": "Llama-3.1-8B-shaped LlamaModel, random init, bf16 (transformers)", "prompt": n,
    "layers_per_build": GROUP,
    "forward_s": round(fwd_s, 3), "serial_prefill_s": round(fwd_s + build_s, 3),
    "serial_build_s": round(build_s, 3), "pipelined_prefill_s": round(pipe_s, 3),
    "build_hidden_frac": round(1 - (pipe_s - fwd_s) / max(build_s, 1e-9), 3),
    "trees_identical_serial_vs_pipelined": same, "model_init_s": round(init_s, 1),
    "engine_decode_ms_per_token_on_model_qkv": round(tpot, 4), "decode_steps_timed": D - 4}))
