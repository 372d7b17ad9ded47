"""Collect bench.py JSON lines from a GPU run directory into a markdown table.

python tools/summarize_round.py gpurun_out/bench_default.log gpurun_out/b3.log ... > table.md
"""
import json
import sys


def load(path):
    for line in reversed(open(path).read().splitlines()):
        if line.startswith("{"):
            return json.loads(line)
    return None


print("| file | config | mode | operator | ms/step | value (unknowns·freq/s) | e2e | K1 near | K3 coupling | K2 up+down | "
      "roofline (kernel, bound, frac) | clocks |")
print("|---|---|---|---|---|---|---|---|---|---|---|---|")
for p in sys.argv[1:]:
    d = load(p)
    if d is None:
        continue
    k = d.get("kernel_ms", {})
    ro = d.get("roofline") or {}
    e2e = d.get("e2e") or {}
    cfg = d["config"]["workload"].split(":")[0]
    print(f"| {p.split('/')[-1]} | {cfg} | {d.get('mode')} | {d.get('operator', 'V')} | {d['ms_per_step']:.2f} | "
          f"{d['value']:.3g} | {e2e.get('value', float('nan')):.3g} | {k.get('near', 0):.2f} | {k.get('coupling', 0):.2f} | "
          f"{k.get('up', 0) + k.get('down', 0):.2f} | {ro.get('kernel', '')}, {ro.get('bound', '')}, "
          f"{ro.get('frac', float('nan')):.3f} | {d['clocks'].get('sm_mhz')} MHz {d['clocks'].get('reasons')} |")
