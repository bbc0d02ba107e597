"""Summarize one kernel of an `ncu --set full` report into profiles/.

  python tools/ncu_summary.py REPORT.ncu-rep KERNEL_REGEX OUT.json [--traffic profiles/search_traffic.json]

Writes the headline metrics (duration, DRAM bytes, throughputs, occupancy
limits, stall breakdown) of the first launch whose name matches KERNEL_REGEX;
with --traffic also the per-launch DRAM traffic that bench.py reports as
roofline.traffic.
"""
import csv
import io
import json
import re
import subprocess
import sys

METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
           "dram__throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__throughput.avg.pct_of_peak_sustained_elapsed",
           "smsp__issue_active.avg.pct_of_peak_sustained_active",
           "sm__warps_active.avg.pct_of_peak_sustained_active",
           "lts__t_sector_hit_rate.pct", "launch__grid_size", "launch__block_size",
           "launch__registers_per_thread", "launch__occupancy_limit_registers",
           "launch__occupancy_limit_shared_mem", "smsp__inst_executed.sum"]
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def main():
    rep, pat, out = sys.argv[1], sys.argv[2], sys.argv[3]
    traffic = sys.argv[sys.argv.index("--traffic") + 1] if "--traffic" in sys.argv else None
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    rx = re.compile(pat)
    kcol = hdr.index("Kernel Name")
    row = next(r for r in rows[2:] if rx.search(r[kcol]))
    res = {"kernel": row[kcol][:120], "report": rep}
    for m in METRICS:
        if m in hdr:
            i = hdr.index(m)
            res[m] = [row[i], units[i]]
    stalls = []
    for i, h in enumerate(hdr):
        if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("_not_issued"):
            try:
                stalls.append((h.replace("smsp__pcsamp_warps_issue_stalled_", ""), float(row[i].replace(",", ""))))
            except ValueError:
                pass
    tot = sum(v for _, v in stalls) or 1.0
    res["stall_top"] = [(k, round(100 * v / tot, 1)) for k, v in sorted(stalls, key=lambda kv: -kv[1])[:8]]

    def nbytes(m):
        v, u = res[m]
        return float(v.replace(",", "")) * UNIT.get(u, 1)
    res["dram_bytes_per_launch"] = nbytes("dram__bytes_read.sum") + nbytes("dram__bytes_write.sum")
    with open(out, "w") as fh:
        json.dump(res, fh, indent=1)
    if traffic:
        with open(traffic, "w") as fh:
            json.dump({"kernel": res["kernel"], "source": out,
                       "dram_bytes_per_launch": res["dram_bytes_per_launch"],
                       "note": "ncu --set full, one launch inside bench.py at C2 (240 trees)"}, fh, indent=1)
    print(json.dumps(res, indent=1)[:2500])


if __name__ == "__main__":
    main()
