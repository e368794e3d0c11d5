"""Summarise one K2 `ncu --set full` report (raw page) into profiles/ncu_k2_summary.json,
which bench.py reads for roofline.traffic (dram bytes per launch)."""
import csv
import io
import json
import subprocess
import sys

rep, out, workload, command = sys.argv[1], sys.argv[2], sys.argv[3], sys.argv[4]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, u, v = rows[0], rows[1], rows[2]
get = {n: (v[i], u[i]) for i, n in enumerate(h)}


def val(name, scale=1.0):
    x, unit = get[name]
    x = x.replace(",", "")
    mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ms": 1, "us": 1e-3, "s": 1e3}.get(unit, 1)
    return float(x) * mult * scale


rd, wr = val("dram__bytes_read.sum"), val("dram__bytes_write.sum")
summary = {
    "workload": workload, "kernel": "k_simulate<16, true> (K2)", "command": command,
    "gpu_time_ms": val("gpu__time_duration.sum"),
    "dram_bytes_read": int(rd), "dram_bytes_write": int(wr), "dram_bytes_per_launch": int(rd + wr),
    "smsp_inst_executed": int(val("smsp__inst_executed.sum")),
    "issue_active_pct": val("smsp__issue_active.avg.pct_of_peak_sustained_active"),
    "warps_active_pct": val("sm__warps_active.avg.pct_of_peak_sustained_active"),
    "fp64_pipe_pct": val("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
    "tensor_pipe_pct": val("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"),
    "registers_per_thread": int(val("launch__registers_per_thread")),
    "stall_per_issue": {k: round(val(f"smsp__average_warps_issue_stalled_{k}_per_issue_active.ratio"), 3)
                        for k in ("wait", "short_scoreboard", "branch_resolving", "not_selected", "no_instruction",
                                  "long_scoreboard", "math_pipe_throttle")},
}
json.dump(summary, open(out, "w"), indent=1)
print(json.dumps(summary))
