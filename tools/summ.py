"""One-line summary of a bench.py JSON line (stdin)."""
import json
import sys

for line in sys.stdin:
    line = line.strip()
    if not line.startswith('{'):
        continue
    d = json.loads(line)
    r = d.get("roofline", {})
    a = d.get("attention_ms_per_step", 0)
    a = f"{a:.3f} ms" if isinstance(a, float) else a
    print("value %.1f tok/s | ms/step %.3f | search %.3f ms frac %.3f | attn %s | e2e %s | launches %s | clocks %s"
          % (d["value"], d["ms_per_step"], r.get("launch_ms", 0), r.get("frac", 0), a,
             (d.get("e2e") or {}).get("value"), d.get("gpu_launches"), d.get("clocks")))
