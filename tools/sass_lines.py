"""Attribute ncu per-instruction executed counts (source page, SASS csv) to CUDA source lines
using nvdisasm -g line info of the same cubin.
usage: sass_lines.py <libmhd.so> <mangled kernel name> <ncu sass csv> [top]"""
import csv
import os
import re
import subprocess
import sys
import tempfile
from collections import Counter, defaultdict

so, kern, csvp = sys.argv[1:4]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
d = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(so)], cwd=d, capture_output=True)
txt = ""
for f in sorted(os.listdir(d)):
    if f.endswith(".cubin"):
        t = subprocess.run(["nvdisasm", "-g", os.path.join(d, f)], capture_output=True, text=True).stdout
        if kern + ":" in t:
            txt = t
            break
lines = txt.splitlines()
start = [i for i, l in enumerate(lines) if l.strip().startswith(kern + ":")][0]
insts, cur = [], None
for l in lines[start + 1:]:
    if l.strip().startswith(".section") or (re.match(r"^(\.text\.)?_Z\w+:\s*$", l) and kern not in l):
        break
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        cur = (m.group(1).split("/")[-1], int(m.group(2)))
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(@!?U?P\w+\s+)?([A-Z0-9_]+)", l)
    if m:
        insts.append((m.group(3), cur))
rows = list(csv.reader(open(csvp)))
h = rows[1]
iex = h.index("Instructions Executed")
ismp = h.index("Warp Stall Sampling (All Samples)")
dyn = [(int(float(r[iex] or 0)), int(float(r[ismp] or 0))) for r in rows[2:] if len(r) > iex]
assert len(dyn) == len(insts), (len(dyn), len(insts))
byline, byop, bysmp = Counter(), defaultdict(Counter), Counter()
for (op, loc), (n, s) in zip(insts, dyn):
    byline[loc] += n
    byop[loc][op] += n
    bysmp[loc] += s
tot = sum(n for n, _ in dyn)
tots = sum(s for _, s in dyn)
srcs = {}
for loc, c in byline.most_common(top):
    if loc is None:
        continue
    f, ln = loc
    if f not in srcs:
        for cand in ("paper_2510_24175_b200/csrc/" + f,):
            if os.path.exists(cand):
                srcs[f] = open(cand).read().splitlines()
    s = srcs.get(f, [""] * (ln + 1))[ln - 1].strip()[:72] if f in srcs else ""
    ops = ", ".join(f"{o}:{100 * v / max(c, 1):.0f}%" for o, v in byop[loc].most_common(3))
    print(f"{100 * c / tot:5.1f}% stall {100 * bysmp[loc] / max(tots, 1):5.1f}% {f}:{ln:<4d} {s:72s} [{ops}]")
