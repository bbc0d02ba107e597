"""q/k/v of a Llama forward as an ICET trace (the reference's trace format,
workload.py:170-224), for engine runs on model-produced embeddings.

A Llama (transformers' LlamaForCausalLM, random init from a fixed seed -- no
checkpoints are reachable here) runs one causal forward over random token
ids; an attention hook records every layer's post-RoPE queries, keys and
values, which is exactly what a decode step hands the KV cache at each
position.  The trace stores each GQA group's first-head query (the format's
rule), so reference and device engines replay identical inputs.

  python tools/llama_trace.py OUT.icet [n_tokens] [layers] [hidden] [heads] [kv_heads] [head_dim]
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def capture_qkv(n_tokens=700, layers=3, hidden=256, heads=8, kv_heads=2, head_dim=32, seed=0, device="cpu",
                dtype=torch.float32):
    from transformers import AttentionInterface, LlamaConfig, LlamaForCausalLM
    from transformers.integrations.sdpa_attention import sdpa_attention_forward
    rec = {}

    def capture(module, query, key, value, attention_mask, **kw):
        # query [B, Hq, S, D], key / value [B, Hkv, S, D], post-RoPE
        rec[module.layer_idx] = (query[0].permute(1, 0, 2).float().cpu(), key[0].permute(1, 0, 2).float().cpu(),
                                 value[0].permute(1, 0, 2).float().cpu())
        return sdpa_attention_forward(module, query, key, value, attention_mask, **kw)

    AttentionInterface.register("icet_capture", capture)
    torch.manual_seed(seed)
    cfg = LlamaConfig(vocab_size=2000, hidden_size=hidden, intermediate_size=2 * hidden, num_hidden_layers=layers,
                      num_attention_heads=heads, num_key_value_heads=kv_heads, head_dim=head_dim,
                      max_position_embeddings=max(4096, n_tokens), attn_implementation="icet_capture")
    with torch.device(device):
        model = LlamaForCausalLM(cfg).to(dtype).eval()
    ids = torch.randint(0, cfg.vocab_size, (1, n_tokens), generator=torch.Generator().manual_seed(seed + 1))
    with torch.no_grad():
        model(input_ids=ids.to(device), use_cache=False)
    q = np.stack([rec[l][0].numpy() for l in range(layers)], axis=1)   # [n, L, Hq, D]
    k = np.stack([rec[l][1].numpy() for l in range(layers)], axis=1)   # [n, L, H, D]
    v = np.stack([rec[l][2].numpy() for l in range(layers)], axis=1)
    return q, k, v


if __name__ == "__main__":
    from paper_2604_10539_b200.trace import save_trace
    out = sys.argv[1]
    args = [int(x) for x in sys.argv[2:]]
    names = ["n_tokens", "layers", "hidden", "heads", "kv_heads", "head_dim"]
    kw = dict(zip(names, args))
    q, k, v = capture_qkv(**kw)
    G = q.shape[2] // k.shape[2]
    save_trace(k, v, q, G, out)
    print(out, k.shape, q.shape, os.path.getsize(out), "bytes")
