"""Summarise a K2 `ncu --set full` report (raw page) into profiles/ncu_k2_summary.json, which
bench.py reads for roofline.traffic (DRAM bytes of one simulate call = all its K2 launches: one per
K2 mode present, e.g. FRESH (chain summariser) + LEAN (ensembling / routing) at C5).

  python scripts/ncu_summary.py report.ncu-rep[,more.ncu-rep] out.json workload "command"

Several reports may be given (comma-separated): per kernel the first row with all counters wins
(ncu sometimes returns nan counters for the second of two long launches in one capture).
"""
import csv
import io
import json
import subprocess
import sys

rep, out, workload, command = sys.argv[1], sys.argv[2], sys.argv[3], sys.argv[4]
MULT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ms": 1, "us": 1e-3, "ns": 1e-6, "s": 1e3,
        "msecond": 1, "usecond": 1e-3, "nsecond": 1e-6}


def kernel(h, u, v):
    get = {n: (v[i], u[i]) for i, n in enumerate(h)}

    def val(name):
        x, unit = get[name]
        return float(x.replace(",", "")) * MULT.get(unit, 1)

    def opt(name):   # a counter ncu could not collect in this pass reads as nan
        x = val(name)
        return None if x != x else int(x)

    rd, wr = opt("dram__bytes_read.sum"), opt("dram__bytes_write.sum")
    return {
        "kernel": get["Kernel Name"][0],
        "gpu_time_ms": val("gpu__time_duration.sum"),
        "dram_bytes_read": rd, "dram_bytes_write": wr,
        "smsp_inst_executed": opt("smsp__inst_executed.sum"),
        "issue_active_pct": val("smsp__issue_active.avg.pct_of_peak_sustained_active"),
        "warps_active_pct": val("sm__warps_active.avg.pct_of_peak_sustained_active"),
        "fp64_pipe_pct": val("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
        "tensor_pipe_pct": val("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"),
        "registers_per_thread": int(val("launch__registers_per_thread")),
        "stall_per_issue": {k: round(val(f"smsp__average_warps_issue_stalled_{k}_per_issue_active.ratio"), 3)
                            for k in ("wait", "short_scoreboard", "branch_resolving", "not_selected",
                                      "no_instruction", "long_scoreboard", "math_pipe_throttle")},
    }


by_name = {}
for r in rep.split(","):
    raw = subprocess.run(["ncu", "-i", r, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, u = rows[0], rows[1]
    for v in rows[2:]:
        if len(v) != len(h) or "k_simulate" not in v[h.index("Kernel Name")]:
            continue
        k = kernel(h, u, v)
        if k["dram_bytes_read"] is None or k["smsp_inst_executed"] is None:
            by_name.setdefault(k["kernel"], k)
        elif by_name.get(k["kernel"]) is None or by_name[k["kernel"]]["dram_bytes_read"] is None:
            by_name[k["kernel"]] = k
ks = list(by_name.values())
tot_ms = sum(k["gpu_time_ms"] for k in ks)
summary = {
    "workload": workload, "kernel": "k_simulate (K2, all launches of one simulate call)", "command": command,
    "launches": ks,
    "gpu_time_ms": tot_ms,
    "dram_bytes_per_launch": (None if any(k["dram_bytes_read"] is None or k["dram_bytes_write"] is None for k in ks)
                              else sum(k["dram_bytes_read"] + k["dram_bytes_write"] for k in ks)),
    "smsp_inst_executed": sum(k["smsp_inst_executed"] for k in ks),
    # time-weighted over the launches
    "issue_active_pct": sum(k["issue_active_pct"] * k["gpu_time_ms"] for k in ks) / tot_ms,
    "warps_active_pct": sum(k["warps_active_pct"] * k["gpu_time_ms"] for k in ks) / tot_ms,
    "fp64_pipe_pct": sum(k["fp64_pipe_pct"] * k["gpu_time_ms"] for k in ks) / tot_ms,
    "tensor_pipe_pct": max(k["tensor_pipe_pct"] for k in ks),
}
json.dump(summary, open(out, "w"), indent=1)
print(json.dumps(summary))
