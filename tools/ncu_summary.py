"""Summarise an ncu --set full report: key throughput metrics + top stall reasons.

usage: python tools/ncu_summary.py report.ncu-rep [points_per_launch]
"""
import csv, io, json, subprocess, sys

rep = sys.argv[1]
n_points = float(sys.argv[2]) if len(sys.argv) > 2 else None
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
KEYS = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__bytes_read.sum.per_second", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__cycles_elapsed.avg.per_second", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size",
        "launch__block_size", "launch__shared_mem_per_block_dynamic", "lts__t_bytes.sum",
        "smsp__inst_executed.sum", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
out = []
for r in rows[2:]:
    d = {}
    for k in KEYS:
        if k in hdr:
            i = hdr.index(k)
            d[k] = (r[i], units[i])
    stalls = {h: r[i] for i, h in enumerate(hdr)
              if h.startswith("smsp__average_warp_latency_issue_stalled_") or
              (h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("_not_issued"))}
    top = sorted(((float(v.replace(",", "")), k) for k, v in stalls.items() if v not in ("", "n/a")), reverse=True)[:8]
    d["top_stalls"] = [(k.split("stalled_")[-1], v) for v, k in top]
    rd = float(d["dram__bytes_read.sum"][0].replace(",", "")) * SCALE.get(d["dram__bytes_read.sum"][1], 1)
    wr = float(d["dram__bytes_write.sum"][0].replace(",", "")) * SCALE.get(d["dram__bytes_write.sum"][1], 1)
    d["traffic_bytes"] = rd + wr
    if n_points:
        d["traffic_bytes_per_point"] = (rd + wr) / n_points
    out.append(d)
for d in out:
    for k, v in d.items():
        print(f"{k:62s} {v}")
    print()
if n_points and out:
    print(json.dumps({"dram_bytes_per_point": out[0]["traffic_bytes_per_point"], "points_per_launch": n_points}))
