#!/usr/bin/env python
"""SASS opcode histograms of the hot kernels of libbem.so (SURVEY §5 evidence).

For each kernel: the whole-function opcode counts (DMMA = FP64 tensor core,
DFMA/DMUL/DADD = FP64 ALU), and, for the K1 near-field kernel, the FP64
instructions attributed (via -lineinfo) to the node loop of near.cu, divided by
the complex exponentials one pass of that loop evaluates (7 nodes x F classes):
the measured "FP64 instructions per evaluation" behind K1's roofline model.
Run: python tools/sass_report.py > profiles/r02_sass.md   (no GPU needed)
"""
from __future__ import annotations

import os
import re
import subprocess
import sys
import tempfile
from collections import Counter

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2006_05186_b200", "libbem.so")
CUDA = "/usr/local/cuda/bin"

KERNELS = [  # (cubin, mangled-name regex, label)
    ("far", r"far8_kernelILi2ELi4ELi0EE", "K3 far8<MT=2, NJ=4> (p = 64, config 3/4)"),
    ("far", r"far8_kernelILi2ELi4ELi4EE|far8_kernelILi2ELi4ELi0EE", None),
    ("far", r"far7_kernelILi2ELi3ELi3EE", "K3 far7<MT=2, NJ=3, REM=3> (p = 27, config 2)"),
    ("far", r"zgen_tile_kernel", "K3 factors-only Z-tile regeneration"),
    ("far", r"h2o_kernelILi2ELi2EE", "K3' h2o (plain H2, p = 64)"),
    ("near", r"near_kernelILi4EE", "K1 near_kernel<F=4>"),
    ("nearm", r"nearm_kernel", "K1m nearm_kernel (combined mode)"),
    ("apply", r"up_leaf_d_kernel", "K2 up leaf products (DMMA)"),
    ("apply", r"up_transfer_k_kernelILi4EE", "K2 up Kronecker transfers (m = 4)"),
    ("apply", r"down_leaf_d_kernel", "K2 down leaf products (DMMA)"),
    ("fft", r"stockham_kernel", "K4 Stockham mixed-radix FFT"),
    ("fft", r"bluestein_kernel", "K4 Bluestein (prime L)"),
    ("aca", r"aca_kernelILb0EE", "ACA assembly (far blocks, pinned arithmetic)"),
]
FP64 = ("DMMA", "DFMA", "DMUL", "DADD", "DSETP", "DMNMX")


def cubins(tmp):
    subprocess.run([f"{CUDA}/cuobjdump", "-xelf", "all", LIB], cwd=tmp, check=True, capture_output=True)
    return {f.split(".")[0]: os.path.join(tmp, f) for f in os.listdir(tmp) if f.endswith(".cubin")}


def functions(cubin):
    """name -> list of (opcode, source line or None)"""
    out = subprocess.run([f"{CUDA}/nvdisasm", "-c", "-g", cubin], capture_output=True, text=True).stdout
    funcs, cur, line = {}, None, None
    for ln in out.splitlines():
        m = re.match(r"\s*\.text\.(\S+):", ln)
        if m:
            cur = m.group(1)
            funcs[cur] = []
            continue
        m = re.search(r'//## File ".*?", line (\d+)', ln)
        if m:
            line = int(m.group(1))
            continue
        m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(@!?U?P[T0-9]+\s+)?([A-Z][A-Z0-9_]*)", ln)
        if m and cur:
            funcs[cur].append((m.group(2), line))
    return funcs


def main():
    print("# SASS opcode histograms (libbem.so, sm_100a, `python tools/sass_report.py`)\n")
    with tempfile.TemporaryDirectory() as tmp:
        cb = cubins(tmp)
        cache = {}
        done = set()
        for unit, pat, label in KERNELS:
            if label is None or unit not in cb:
                continue
            if unit not in cache:
                cache[unit] = functions(cb[unit])
            names = [n for n in cache[unit] if re.search(pat, n)]
            if not names:
                continue
            name = sorted(names, key=len)[0]
            if name in done:
                continue
            done.add(name)
            ops = Counter(o for o, _ in cache[unit][name])
            tot = sum(ops.values())
            fp = {k: ops.get(k, 0) for k in FP64}
            print(f"## {label}\n\n`{name}`: {tot} instructions; FP64: " +
                  ", ".join(f"{k} {v}" for k, v in fp.items() if v) + "\n")
            print("top opcodes: " + ", ".join(f"{k} {v}" for k, v in ops.most_common(16)) + "\n")
            if unit == "near":
                src = open(os.path.join(ROOT, "paper_2006_05186_b200", "csrc", "near.cu")).read().splitlines()
                lo = next(i for i, s in enumerate(src, 1) if "for (int q = 0; q < 7; ++q)" in s)
                hi = next(i for i, s in enumerate(src, 1) if i > lo and "cmac(acc1[f], v[f], x1[f]);" in s)
                # the unrolled loop is one contiguous address range: from the first to the last
                # instruction attributed to near.cu lines [lo, hi] (the inlined fast exp / sincos
                # carry fastmath.cuh line numbers inside that range)
                ins = cache[unit][name]
                idx = [i for i, (o, l) in enumerate(ins) if l is not None and lo <= l <= hi]
                body = Counter(o for o, _ in ins[min(idx):max(idx) + 1])
                fpb = sum(body.get(k, 0) for k in ("DFMA", "DMUL", "DADD"))
                print(f"node loop (near.cu:{lo}-{hi}, 7 nodes x F = 4 classes = 28 complex exponentials per pass, "
                      f"unrolled): DFMA {body.get('DFMA', 0)}, DMUL {body.get('DMUL', 0)}, DADD {body.get('DADD', 0)}"
                      f" -> {fpb / 28:.1f} FP64 instructions per evaluation ({body.get('DFMA', 0) / 28:.1f} DFMA); "
                      f"all instructions in the loop: {sum(body.values())} ({sum(body.values()) / 28:.1f} per "
                      f"evaluation)\n")


if __name__ == "__main__":
    sys.exit(main())
