"""Turn an ncu launch list (+ optional `--set full` report) into a markdown summary for profiles/.

python tools/profile_report.py --launches gpurun_out/launches_c2.csv [--rep gpurun_out/prof_c2.ncu-rep]
    [--bench gpurun_out/bench_c2.log] --title "..." > profiles/rNN_....md

The launch list is cold-cache and serialised (ncu), so only each kernel's SHARE
of the step is compared with the bench's live CUDA-event timings.
"""
import argparse
import csv
import json
import subprocess
from collections import defaultdict

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__occupancy_limit_registers", "CTA/SM limit (registers)"),
    ("launch__occupancy_limit_shared_mem", "CTA/SM limit (smem)"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("sm__issue_active.avg.pct_of_peak_sustained_elapsed", "issue active %"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 (DFMA) pipe %"),
    ("sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active", "DMMA sub-pipe %"),
    ("sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active", "shared FP64+tensor pipe %"),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe %"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput %"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("sm__inst_executed_pipe_fp64.sum", "FP64 warp instructions"),
]


def short(name):
    n = name.split("(")[0]
    return n.replace("void ", "").replace("(anonymous namespace)::", "").replace("unnamed>::", "")


def launches(path):
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[h]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    tot, cnt = defaultdict(float), defaultdict(int)
    unit = None
    for r in rows[h + 1:]:
        if len(r) <= vi:
            continue
        n = short(r[ki])
        tot[n] += float(r[vi].replace(",", ""))
        cnt[n] += 1
        unit = r[ui]
    return tot, cnt, unit


def full(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units = rows[0], rows[1]
    out = []
    for row in rows[2:]:
        d = {"kernel": short(row[hdr.index("Kernel Name")])}
        for k, lab in KEYS:
            if k in hdr:
                d[lab] = f"{row[hdr.index(k)]} {units[hdr.index(k)]}".strip()
        st = []
        for i, h in enumerate(hdr):
            if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
                try:
                    v = float(row[i])
                except ValueError:
                    continue
                if v > 0.05:
                    st.append((v, h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
        d["top stalls (warps per issue)"] = ", ".join(f"{n} {v:.2f}" for v, n in sorted(st, reverse=True)[:6])
        out.append(d)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--launches")
    ap.add_argument("--rep")
    ap.add_argument("--bench")
    ap.add_argument("--title", default="profile")
    ap.add_argument("--cmd", default="")
    a = ap.parse_args()
    print(f"# {a.title}\n")
    if a.cmd:
        print(f"Command: `{a.cmd}`\n")
    if a.bench:
        line = [ln for ln in open(a.bench) if ln.startswith("{")][-1]
        b = json.loads(line)
        print("## bench.py line (live CUDA events, not under ncu)\n")
        keys = ["value", "unit", "ms_per_step", "kernel_ms", "roofline", "e2e", "clocks", "mean_aca_rank",
                "fp64_dfma_measured_tflops", "near_evals_per_s", "cpu_baseline", "gpu_launches"]
        print("```json\n" + json.dumps({k: b.get(k) for k in keys}, indent=1) + "\n```\n")
    if a.launches:
        tot, cnt, unit = launches(a.launches)
        s = sum(tot.values())
        print(f"## ncu launch list (`gpu__time_duration.sum`, --clock-control none; cold-cache, serialised)\n")
        print(f"| kernel | launches | total ({unit}) | share |\n|---|---|---|---|")
        for n in sorted(tot, key=lambda k: -tot[k]):
            print(f"| `{n[:60]}` | {cnt[n]} | {tot[n]:.0f} | {100 * tot[n] / s:.1f}% |")
        print()
    if a.rep:
        print("## ncu --set full (per kernel)\n")
        for d in full(a.rep):
            print(f"### `{d.pop('kernel')[:80]}`\n")
            for k, v in d.items():
                print(f"- {k}: {v}")
            print()


if __name__ == "__main__":
    main()
