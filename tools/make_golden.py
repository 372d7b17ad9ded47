#!/usr/bin/env python
"""Write the oracle's expected values for the full-size config-4 parity test
(tests/test_gpu_fullsize.py) to tests/golden/c4_oracle.npz.

Calls ONLY oracle/ (and the input generators in synth/): nothing here touches
the CUDA library.  Config 4 (81,920 panels, L = 513, p = 64) takes the oracle
several minutes (the ACA of all 98,386 far blocks and a 4-frequency H2ACA
apply), too long to repeat inside every GPU test run, so the result is stored
with the recipe that produced it:
  * y[lsel] = V(s_l) x_l for lsel = {0, 1, L/2, L-1} (identical-compression
    H2ACA apply, eq:lrfinal P:1404-1410) on x = synth.random_density(4, L, M);
  * the ACA ranks of every far block and the SHA-256 of the full pivot list
    (k_l, q_l) in block order (int32 little-endian), the bit-exact check of C13;
  * the SHA-256 of the tree / partition export (perm, clusters, boxes, near, far).
Run:  python tools/make_golden.py [--threads N]
"""
from __future__ import annotations

import argparse
import hashlib
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle as O  # noqa: E402
import synth  # noqa: E402


def sha(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--threads", type=int, default=0)
    ap.add_argument("--out", default=os.path.join(ROOT, "tests", "golden", "c4_oracle.npz"))
    args = ap.parse_args()
    if args.threads:
        O.set_threads(args.threads)
    cfg = 4
    c = synth.CONFIGS[cfg]
    V, T = synth.config_mesh(cfg)
    N = c["N"]
    M, L = len(T), N + 1
    lsel = np.array([0, 1, L // 2, L - 1], dtype=np.int32)
    s = O.frequencies(N, c["T"])
    t0 = time.time()
    h = O.H2(V, T, c["leaf"], c["eta"], c["m"])
    ex = h.export()
    t1 = time.time()
    a = h.aca(s, c["eps"], keep=lsel)
    t2 = time.time()
    x = synth.random_density(cfg, L, M)
    y = h.apply(O.MODE_H2ACA, s, x[lsel], lsel)
    t3 = time.time()
    np.savez_compressed(
        args.out, lsel=lsel, y=y, ranks=a["ranks"].astype(np.int16),
        pivots_sha256=np.array(sha(a["pivots"].astype("<i4"))),
        tree_sha256=np.array(sha(ex["perm"], ex["clusters"], ex["boxes"], ex["near"], ex["far"])),
        recipe=np.array(f"config 4 ({M} panels, N={N}, m={c['m']}, leaf={c['leaf']}, eta={c['eta']}, eps={c['eps']}); "
                        f"x = synth.random_density(4, {L}, {M}); y = oracle H2ACA apply at l in {lsel.tolist()}; "
                        f"oracle threads {O.num_threads()}: tree {t1 - t0:.1f} s, ACA {t2 - t1:.1f} s, "
                        f"apply {t3 - t2:.1f} s; numpy {np.__version__}"))
    print(f"wrote {args.out}: mean rank {a['ranks'].mean():.2f}, sum {a['ranks'].sum()}, "
          f"tree {t1 - t0:.1f}s ACA {t2 - t1:.1f}s apply {t3 - t2:.1f}s")


if __name__ == "__main__":
    main()
