import json,sys
for line in sys.stdin:
    line=line.strip()
    if not line.startswith('{'): continue
    d=json.loads(line)
    r=d.get("roofline",{})
    print("value %.1f tok/s | ms/step %.3f | search %.3f ms frac %.3f | attn %.3f ms | e2e %s | launches %s | clocks %s" % (d["value"], d["ms_per_step"], r.get("launch_ms",0), r.get("frac",0), d.get("attention_ms_per_step",0), (d.get("e2e") or {}).get("value"), d.get("gpu_launches"), d.get("clocks")))
