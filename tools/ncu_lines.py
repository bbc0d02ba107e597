"""Top CUDA source lines of an ncu report by warp-stall samples:
  python tools/ncu_lines.py REPORT.ncu-rep [N]
(ncu --page source --print-source cuda,sass; CUDA-line aggregate rows)."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows, f, hdr = [], None, None
for rec in csv.reader(io.StringIO(raw)):
    if not rec:
        continue
    if rec[0] == "File Path":
        f = rec[1].split("/")[-1]
        continue
    if rec[0] == "Line No":
        hdr = rec
        continue
    if hdr is None or len(rec) < 5 or rec[2] != "-":
        continue
    d = dict(zip(hdr[2:], rec[2:]))
    try:
        s = int(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
    except ValueError:
        continue
    stalls = {k[6:]: int(v) for k, v in zip(hdr[2:], rec[2:]) if k.startswith("stall_") and "Not Issued" not in k
              and v.isdigit() and int(v) > 0}
    rows.append((s, f, rec[0], rec[1].strip()[:90], stalls))
tot = sum(r[0] for r in rows) or 1
rows.sort(reverse=True)
for s, f, ln, src, st in rows[:top]:
    big = sorted(st.items(), key=lambda kv: -kv[1])[:3]
    print(f"{100 * s / tot:5.1f}% {f}:{ln:5s} {src:90s} {big}")
