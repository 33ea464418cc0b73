"""Summarise an ncu report (raw page) into the metrics DESIGN.md tracks; usage: ncu_summary.py rep.ncu-rep"""
import csv
import os
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__registers_per_thread",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem", "launch__grid_size",
        "launch__block_size", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "smsp__thread_inst_executed_per_inst_executed.ratio",
        "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum", "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum",
        "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum", "sass__inst_executed_local_loads",
        "sass__inst_executed_local_stores", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum", "sm__cycles_elapsed.avg.per_second"]


def to_json(path, out_json, cells, which="stage 1 (7th stage launch: after 3 warm-up steps)"):
    """one-kernel summary used by bench.py's roofline.traffic (profiles/ncu_stage_summary.json)"""
    import json
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, u, v = rows[0], rows[1], rows[2]

    def g(k, scale=1.0):
        x = float(v[h.index(k)].replace(",", ""))
        unit = u[h.index(k)]
        mult = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "ms": 1e-3, "us": 1e-6, "ns": 1e-9}.get(unit, 1.0)
        return x * mult * scale
    d = {"report": os.path.basename(path), "kernel": v[h.index("Kernel Name")],
         "duration_s_under_ncu": g("gpu__time_duration.sum"),
         "dram_bytes_per_launch": g("dram__bytes_read.sum") + g("dram__bytes_write.sum"),
         "dram_bytes_per_cell": (g("dram__bytes_read.sum") + g("dram__bytes_write.sum")) / cells,
         "fp64_pipe_active_pct": g("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
         "issue_active_pct": g("smsp__issue_active.avg.pct_of_peak_sustained_active"),
         "warps_active_pct": g("sm__warps_active.avg.pct_of_peak_sustained_active"),
         "registers_per_thread": g("launch__registers_per_thread"),
         "warp_instructions": g("smsp__inst_executed.sum"),
         "thread_instructions_per_cell": g("smsp__inst_executed.sum") * 32 / cells,
         "stage_of_launch": which}
    json.dump(d, open(out_json, "w"), indent=1)
    print(json.dumps(d, indent=1))


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, u = rows[0], rows[1]
    for v in rows[2:]:
        name = v[h.index("Kernel Name")] if "Kernel Name" in h else "?"
        print("kernel:", name[:100])
        for k in KEYS:
            if k in h:
                print(f"  {k} = {v[h.index(k)]} {u[h.index(k)]}")
        st = [(k, float(v[i])) for i, k in enumerate(h) if k.startswith("smsp__average_warps_issue_stalled_")
              and k.endswith("_per_issue_active.ratio") and v[i] not in ("", "n/a")]
        st.sort(key=lambda t: -t[1])
        print("  stalls per issued instruction:",
              ", ".join(f"{k[len('smsp__average_warps_issue_stalled_'):-len('_per_issue_active.ratio')]}={x:.2f}"
                        for k, x in st[:8]))


if __name__ == "__main__":
    if sys.argv[1] == "--json":
        to_json(sys.argv[2], sys.argv[3], float(sys.argv[4]), *sys.argv[5:6])
    else:
        for p in sys.argv[1:]:
            main(p)
