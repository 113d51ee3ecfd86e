"""Extract the judged metrics of every kernel in an ncu --set full report to JSON.
usage: python tools/ncu_full_json.py <report.ncu-rep> > out.json"""
import csv
import io
import json
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "dram__bytes_read.sum",
        "dram__bytes_write.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__warps_eligible.avg.per_cycle_active"]
raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
out = []
for r in rows[2:]:
    d = dict(zip(hdr, r))
    u = dict(zip(hdr, units))
    rec = {"kernel": d["Kernel Name"]}
    for k in KEYS:
        if k in d:
            rec[k] = f"{d[k]} {u.get(k, '')}".strip()
    stalls = {}
    for k, v in d.items():
        if k.startswith("smsp__average_warp_latency_issue_stalled_") or not k.startswith("smsp__pcsamp_warps_issue_stalled_"):
            continue
        if k.endswith("_not_issued"):
            continue
        try:
            stalls[k.replace("smsp__pcsamp_warps_issue_stalled_", "")] = float(v.replace(",", ""))
        except ValueError:
            pass
    tot = sum(stalls.values())
    if tot > 0:
        top = sorted(stalls.items(), key=lambda x: -x[1])[:6]
        rec["top_stalls"] = {k: round(v / tot, 3) for k, v in top}
    out.append(rec)
json.dump(out, sys.stdout, indent=1)
