"""Per-kernel share of device time from an ncu --metrics gpu__time_duration.sum --csv launch list."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hdr]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
d = defaultdict(list)
for r in rows[hdr + 1:]:
    if len(r) > vi:
        scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "nsecond": 1e-6, "ms": 1.0, "msecond": 1.0}.get(r[ui], 1e-6)
        d[r[ki].split("(")[0][:48]].append(float(r[vi].replace(",", "")) * scale)
tot = sum(sum(v) for v in d.values())
print(f"{'kernel':50s} {'launches':>8s} {'mean ms':>9s} {'share':>6s}")
for k, v in sorted(d.items(), key=lambda kv: -sum(kv[1])):
    print(f"{k:50s} {len(v):8d} {sum(v) / len(v):9.3f} {sum(v) / tot:6.3f}")
