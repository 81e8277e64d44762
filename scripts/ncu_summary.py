#!/usr/bin/env python
"""Summarise an ncu --set full report (and optionally a launch-list CSV) into
profiles/<name>.md + .json.

  python scripts/ncu_summary.py gpurun_out/scan_deep100m.ncu-rep profiles/r1_scan_deep100m \
      [--launches gpurun_out/launches_deep100m.csv] [--algo-bytes N]
"""
import argparse
import csv
import io
import json
import subprocess
import sys

METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__shared_mem_per_block_dynamic", "launch__grid_size", "launch__block_size",
    "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_registers", "smsp__inst_executed.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "lts__t_sector_hit_rate.pct", "sm__cycles_elapsed.avg.per_second", "lts__t_bytes.sum",
    "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
    "l1tex__throughput.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
]
STALLS = ["long_scoreboard", "short_scoreboard", "barrier", "wait", "mio_throttle", "lg_throttle", "math_pipe_throttle",
          "not_selected", "selected", "no_instructions", "branch_resolving", "dispatch_stall"]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    kernels = []
    for vals in rows[2:]:
        d = {h: (v, u) for h, u, v in zip(hdr, units, vals)}
        kernels.append(d)
    return kernels


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("out")
    ap.add_argument("--launches")
    ap.add_argument("--algo-bytes", type=float, default=None)
    ap.add_argument("--note", default="")
    a = ap.parse_args()
    ks = raw(a.rep)
    summary = {"report": a.rep, "note": a.note, "kernels": []}
    md = [f"# ncu summary: {a.rep}", "", a.note, ""]
    for d in ks:
        name = d.get("Kernel Name", ("?", ""))[0]
        m = {k: d[k][0] + (" " + d[k][1] if d[k][1] else "") for k in METRICS if k in d}
        stalls = {}
        for s in STALLS:
            k = f"smsp__pcsamp_warps_issue_stalled_{s}"
            if k in d:
                stalls[s] = d[k][0]
        ent = {"kernel": name, "metrics": m, "stall_samples": stalls}
        try:
            rd = float(d["dram__bytes_read.sum"][0]) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[
                d["dram__bytes_read.sum"][1]]
            wr = float(d["dram__bytes_write.sum"][0]) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[
                d["dram__bytes_write.sum"][1]]
            ent["dram_bytes_per_launch"] = rd + wr
            if a.algo_bytes:
                ent["algorithmic_bytes_per_launch"] = a.algo_bytes
                ent["dram_over_algorithmic"] = (rd + wr) / a.algo_bytes
        except Exception:
            pass
        summary["kernels"].append(ent)
        md += [f"## {name}", "", "| metric | value |", "|---|---|"]
        md += [f"| {k} | {v} |" for k, v in m.items()]
        if "dram_bytes_per_launch" in ent:
            md.append(f"| dram bytes (read+write) per launch | {ent['dram_bytes_per_launch']:.4g} |")
        if a.algo_bytes:
            md.append(f"| algorithmic bytes per launch | {a.algo_bytes:.4g} |")
        md += ["", "stall samples: " + ", ".join(f"{k}={v}" for k, v in stalls.items()), ""]
    if a.launches:
        rows = [r for r in csv.reader(open(a.launches)) if len(r) > 5]
        hdr = rows[0]
        iname, ival = hdr.index("Kernel Name"), hdr.index("Metric Value")
        launches = [(r[iname], float(r[ival])) for r in rows[1:]]
        tot = sum(v for _, v in launches)
        summary["launches"] = [{"kernel": k, "ns": v, "share": v / tot} for k, v in launches]
        md += ["## launch list (ncu gpu__time_duration, cold-cache, serialised: compare shares)", "",
               "| kernel | ns | share |", "|---|---|---|"]
        md += [f"| {k[:90]} | {v:.0f} | {v / tot:.3f} |" for k, v in launches]
    json.dump(summary, open(a.out + ".json", "w"), indent=1)
    open(a.out + ".md", "w").write("\n".join(md) + "\n")
    print("wrote", a.out + ".md/.json")


if __name__ == "__main__":
    sys.exit(main())
