"""Per-kernel share of device time from an ncu --metrics gpu__time_duration.sum[,dram__bytes_*] --csv launch
list (other metrics, when present, are averaged per kernel as well)."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hdr]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
ni = h.index("Metric Name") if "Metric Name" in h else None
d = defaultdict(list)
other = defaultdict(lambda: defaultdict(list))
TS = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "nsecond": 1e-6, "ms": 1.0, "msecond": 1.0}
BS = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
for r in rows[hdr + 1:]:
    if len(r) <= vi:
        continue
    name = r[ki].split("(")[0][:48]
    metric = r[ni] if ni is not None else "gpu__time_duration.sum"
    val = float(r[vi].replace(",", ""))
    if metric == "gpu__time_duration.sum":
        d[name].append(val * TS.get(r[ui], 1e-6))
    else:
        other[name][metric].append(val * BS.get(r[ui], 1.0))
tot = sum(sum(v) for v in d.values())
extra = sorted({m for o in other.values() for m in o})
print(f"{'kernel':50s} {'launches':>8s} {'mean ms':>9s} {'share':>6s}" + "".join(f" {m[:22]:>24s}" for m in extra))
for k, v in sorted(d.items(), key=lambda kv: -sum(kv[1])):
    print(f"{k:50s} {len(v):8d} {sum(v) / len(v):9.3f} {sum(v) / tot:6.3f}" +
          "".join(f" {sum(other[k][m]) / max(len(other[k][m]), 1) / 1e9:21.3f} GB" for m in extra))
