"""Summarise one `ncu --set full` capture of a Schur-update launch (raw CSV page) into the JSON
that bench.py reads for roofline.traffic.  usage: ncu_summary.py RAW.csv K NDIAG COMMAND NCU_CMD OUT.json"""
import csv, json, sys

raw, K, ndiag, command, ncu_cmd, out = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), sys.argv[4], sys.argv[5], sys.argv[6]
rows = list(csv.reader(open(raw)))
hdr, units, vals = rows[0], rows[1], rows[2]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3}


def get(name, to=None):
    i = hdr.index(name)
    v = float(vals[i].replace(",", ""))
    return v * scale.get(units[i], 1.0) if to else v


grid = int(get("launch__grid_size"))
dur = get("gpu__time_duration.sum", "ms")
rd, wr = get("dram__bytes_read.sum", "B"), get("dram__bytes_write.sum", "B")
T = 128
flops = (grid - ndiag) * 2.0 * T * T * K + ndiag * T * (T + 1.0) * K
# minimum bytes: every output tile read + written once, and the A/B panel tiles read once
panel_rows = ndiag  # distinct rows/cols of the set (square trailing block)
alg_bytes = grid * 2 * T * T * 8 + panel_rows * (K // T) * T * T * 8
json.dump({
    "kernel": "gemm_kernel<MODE_UPDATE> (trailing 'rest' Schur update, first outer step)",
    "command": command, "ncu": ncu_cmd, "grid": grid, "tiles_diagonal": ndiag, "K": K,
    "duration_ms": dur, "algorithmic_flops": flops, "achieved_tflops": flops / (dur * 1e-3) / 1e12,
    "dram_bytes_read": rd, "dram_bytes_write": wr, "dram_bytes_per_launch": rd + wr,
    "algorithmic_bytes_min": alg_bytes,
    "dmma_pipe_active_pct_of_active_cycles": get("sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active"),
    "sm_throughput_pct": get("sm__throughput.avg.pct_of_peak_sustained_elapsed"),
    "registers_per_thread": int(get("launch__registers_per_thread")),
}, open(out, "w"), indent=1)
print(open(out).read())
