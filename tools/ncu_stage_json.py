#!/usr/bin/env python
"""Per-stage ncu summary of the fused stage kernel for bench.py's roofline (profiles/ncu_stage_<scheme>_<wl><n>.json):
  ncu_stage_json.py <stage.ncu-rep (stage 1, stage 2 launches)> <dt.ncu-rep> <out.json> <cells>
Each entry: duration under ncu, DRAM bytes per launch and per cell, FP64-pipe / issue / warps active,
registers, instructions per cell."""
import csv
import json
import os
import subprocess
import sys

MULT = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "ms": 1e-3, "us": 1e-6, "ns": 1e-9, "s": 1.0}


def rows(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(out.splitlines()))
    return r[0], r[1], r[2:]


def summary(h, u, v, cells, path, what):
    def g(k):
        x = float(v[h.index(k)].replace(",", ""))
        return x * MULT.get(u[h.index(k)], 1.0)
    rd, wr = g("dram__bytes_read.sum"), g("dram__bytes_write.sum")
    return {"report": os.path.basename(path), "kernel": v[h.index("Kernel Name")], "launch": what,
            "duration_s_under_ncu": g("gpu__time_duration.sum"), "dram_bytes_read": rd, "dram_bytes_write": wr,
            "dram_bytes_per_launch": rd + wr, "dram_bytes_per_cell": (rd + wr) / cells,
            "fp64_pipe_active_pct": g("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
            "issue_active_pct": g("smsp__issue_active.avg.pct_of_peak_sustained_active"),
            "warps_active_pct": g("sm__warps_active.avg.pct_of_peak_sustained_active"),
            "registers_per_thread": g("launch__registers_per_thread"),
            "thread_instructions_per_cell": g("smsp__inst_executed.sum") * 32 / cells}


def main(stage_rep, dt_rep, out, cells):
    cells = float(cells)
    h, u, vs = rows(stage_rep)
    d = {}
    for i, v in enumerate(vs[:3]):
        d[f"stage{i + 1}"] = summary(h, u, v, cells, stage_rep, f"RK stage {i + 1} of the 4th step (after 3 warm-up steps)")
    if dt_rep and os.path.exists(dt_rep):
        h, u, vs = rows(dt_rep)
        d["dt"] = summary(h, u, vs[0], cells, dt_rep, "dt pass of the 4th step")
    json.dump(d, open(out, "w"), indent=1)
    print(json.dumps(d, indent=1))


if __name__ == "__main__":
    main(*sys.argv[1:5])
