"""Record the dominant kernel's DRAM bytes per launch from an ncu --set full
report under a bench configuration key in profiles/search_traffic.json
(bench.py reads it as roofline.traffic):
  python tools/ncu_traffic.py REPORT.ncu-rep KEY "source description" [KERNEL_REGEX]"""
import csv
import io
import json
import os
import re
import subprocess
import sys

UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
rep, key, src = sys.argv[1], sys.argv[2], sys.argv[3]
pat = re.compile(sys.argv[4] if len(sys.argv) > 4 else "query_kernel")
rows = list(csv.reader(io.StringIO(subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"],
                                                  capture_output=True, text=True).stdout)))
hdr, units = rows[0], rows[1]
row = next(r for r in rows[2:] if pat.search(r[hdr.index("Kernel Name")]))


def val(m):
    i = hdr.index(m)
    return float(row[i].replace(",", "")) * UNIT.get(units[i], 1)


path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "search_traffic.json")
db = json.load(open(path)) if os.path.exists(path) else {}
dur_i = hdr.index("gpu__time_duration.sum")
db[key] = {"kernel": row[hdr.index("Kernel Name")][:100],
           "dram_bytes_per_launch": val("dram__bytes_read.sum") + val("dram__bytes_write.sum"),
           "dram_read": val("dram__bytes_read.sum"), "dram_write": val("dram__bytes_write.sum"),
           "source": src, "launch_us_cold": float(row[dur_i].replace(",", "")) * (1e3 if units[dur_i] == "ms" else 1)}
json.dump(db, open(path, "w"), indent=1)
print(key, json.dumps(db[key]))
