#!/usr/bin/env python
"""Parallel efficiency from bench.py lines: E(N) = value(N) / (N value(1)) —
the same number the driver computes from its per-N runs.

  python tools/scaling_report.py b1.jsonl b2.jsonl b4.jsonl b8.jsonl
"""
import json
import sys


def main(paths):
    lines = []
    for p in paths:
        for l in open(p):
            l = l.strip()
            if l.startswith("{"):
                d = json.loads(l)
                if "value" in d and d.get("impl") != "reference":
                    lines.append(d)
    by_n = {d["n_gpus"]: d for d in lines}
    if 1 not in by_n:
        sys.exit("need the N = 1 line")
    v1 = by_n[1]["value"]
    for n in sorted(by_n):
        d = by_n[n]
        print(f"N={n}  {d['scaling']:6s}  {d['value']:.4g} zone-updates/s  {d['ms_per_step']:.3f} ms/step  "
              f"E={d['value'] / (n * v1):.3f}  ({d['config'].get('workload')})")


if __name__ == "__main__":
    main(sys.argv[1:])
