"""Summarise an ncu report: key metrics + stall reasons + hottest SASS lines."""
import csv
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr = rows[0]
keys = ["gpu__time_duration.sum", "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "lts__t_bytes.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smsp__inst_executed.sum",
        "sm__inst_executed_pipe_fp64.sum", "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem"]
for row in rows[2:]:
    name = row[hdr.index("Kernel Name")][:50]
    print("==", name)
    for k in keys:
        if k in hdr:
            print(f"   {k:70s} {row[hdr.index(k)]}")
    st = []
    for i, h in enumerate(hdr):
        if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
            try:
                v = float(row[i])
            except ValueError:
                continue
            if v > 0.05:
                st.append((v, h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
    print("   stalls:", ", ".join(f"{n}={v:.2f}" for v, n in sorted(st, reverse=True)[:8]))
