"""Opcode mix and stall hot spots from `ncu --page source --csv --print-source sass` output."""
import csv
import re
import sys
from collections import Counter, defaultdict

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
ia, isrc = h.index("Address"), h.index("Source")
iex = h.index("Instructions Executed")
ith = h.index("Thread Instructions Executed")
ismp = h.index("Warp Stall Sampling (All Samples)")
mix, thr, smp = Counter(), Counter(), Counter()
tot = 0
for r in rows[2:]:
    if len(r) <= ith:
        continue
    src = r[isrc].strip()
    m = re.match(r"(@!?U?P\w+\s+)?([A-Z0-9_]+)(\.[A-Z0-9_.]+)?", src)
    if not m:
        continue
    op = m.group(2)
    n = int(float(r[iex] or 0))
    mix[op] += n
    thr[op] += int(float(r[ith] or 0))
    smp[op] += int(float(r[ismp] or 0))
    tot += n
cells = float(sys.argv[2]) if len(sys.argv) > 2 else None
print(f"total warp instructions {tot:.4g}")
for op, n in mix.most_common(40):
    extra = f" thread-inst/cell {thr[op] / cells:8.1f}" if cells else ""
    print(f"{op:10s} {n:14d} {100 * n / tot:6.2f}%  stall-samples {smp[op]:8d}{extra}")
