"""Summarize an `ncu --metrics gpu__time_duration.sum --csv` launch list into
a per-kernel table (share of device time, launches, mean duration)."""
import collections
import csv
import sys

src, dst = sys.argv[1], sys.argv[2]
cmd = sys.argv[3] if len(sys.argv) > 3 else None
rows = list(csv.reader(open(src)))
hdr = None
agg = collections.defaultdict(list)
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        ki, vi, ui = r.index("Kernel Name"), r.index("Metric Value"), r.index("Metric Unit")
        mi = r.index("Metric Name") if "Metric Name" in r else None
        continue
    if hdr and len(r) > vi:
        if mi is not None and r[mi] != "gpu__time_duration.sum":
            continue
        try:
            val = float(r[vi].replace(",", ""))
        except ValueError:
            continue
        scale = {"ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "nsecond": 1e-3}.get(r[ui], 1e-3)
        agg[r[ki].split("(")[0][:70]].append(val * scale)
tot = sum(sum(v) for v in agg.values())
with open(dst, "w") as fh:
    fh.write(f"# ncu launch list summary ({src})\n\n")
    if cmd:
        fh.write(f"Command: `{cmd}`\n\n")
    fh.write("Cold-cache, serialized per-launch device times (compare shares, not absolutes).\n\n")
    fh.write("| share | launches | mean us | kernel |\n|---:|---:|---:|---|\n")
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        fh.write(f"| {sum(v) / tot * 100:.1f}% | {len(v)} | {sum(v) / len(v):.1f} | `{k}` |\n")
print(open(dst).read()[:3000])
