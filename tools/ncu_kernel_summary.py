"""One-kernel summary of an ncu --set full report (raw page): duration, SOL %, occupancy, pipes,
stall reasons.  usage: ncu_kernel_summary.py REPORT.ncu-rep [NOTE]"""
import csv, io, json, subprocess, sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, vals = rows[0], rows[1], rows[2]
d = dict(zip(hdr, vals))
u = dict(zip(hdr, units))
keys = {
    "kernel": "Kernel Name", "grid": "launch__grid_size", "block": "launch__block_size",
    "duration": "gpu__time_duration.sum", "registers": "launch__registers_per_thread",
    "sm_throughput_pct": "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "dram_throughput_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "l2_hit_pct": "lts__t_sector_hit_rate.pct",
    "achieved_occupancy_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "fp64_pipe_pct": "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "issue_active_pct": "sm__inst_issued.avg.pct_of_peak_sustained_active",
    "dram_bytes_read": "dram__bytes_read.sum", "dram_bytes_write": "dram__bytes_write.sum",
}
out = {}
for k, m in keys.items():
    if m in d:
        out[k] = d[m] + (f" {u[m]}" if u.get(m) else "")
stalls = {}
for name, v in d.items():
    if name.startswith("smsp__average_warps_issue_stalled_") and name.endswith("_per_issue_active.ratio"):
        try:
            f = float(v)
        except ValueError:
            continue
        if f >= 0.05:
            stalls[name[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]] = round(f, 3)
out["stalls_per_issue"] = dict(sorted(stalls.items(), key=lambda x: -x[1]))
if len(sys.argv) > 2:
    out["note"] = sys.argv[2]
print(json.dumps(out, indent=1))
