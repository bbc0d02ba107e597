"""Per-kernel SASS instruction classes of the built library (the Blackwell
evidence table of profiles/): tensor-core (HMMA, UTC*MMA), TMA (UTMALDG,
UBLKCP), async copies (LDGSTS), mbarrier (SYNCS), tensor memory (LDTM/STTM).
  python tools/sass_summary.py [lib.so] > profiles/r02_sass_evidence.md"""
import collections
import re
import subprocess
import sys

lib = sys.argv[1] if len(sys.argv) > 1 else "paper_2604_10539_b200/libicecache_b200.so"
sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
CLASSES = ["UTCHMMA", "UTCIMMA", "UTCQMMA", "UTCMMA", "LDTM", "STTM", "HMMA", "UTMALDG", "UBLKCP", "LDGSTS", "SYNCS",
           "LDSM", "DFMA", "FFMA2", "FFMA", "SHFL", "REDUX"]
cur = None
counts = collections.OrderedDict()
names = subprocess.run(["c++filt"], input="\n".join(re.findall(r"Function : (\S+)", sass)), capture_output=True,
                       text=True).stdout.splitlines()
mangled = re.findall(r"Function : (\S+)", sass)
demangle = dict(zip(mangled, names))
for line in sass.splitlines():
    m = re.search(r"Function : (\S+)", line)
    if m:
        cur = demangle.get(m.group(1), m.group(1))
        counts[cur] = collections.Counter()
        continue
    if cur is None:
        continue
    ins = re.search(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(\.[A-Z0-9_.]+)?", line)
    if ins:
        op = ins.group(1)
        for c in CLASSES:
            if op.startswith(c):
                counts[cur][c] += 1
                break
print("| kernel | " + " | ".join(CLASSES) + " |")
print("|---|" + "---|" * len(CLASSES))
for k, c in counts.items():
    short = re.sub(r"\(.*", "", k)[:70]
    if not any(c.values()):
        continue
    print(f"| `{short}` | " + " | ".join(str(c[x]) if c[x] else "" for x in CLASSES) + " |")
