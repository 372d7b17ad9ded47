"""Time-domain solve with compressed weights (NEXT-2) vs the frequency-decoupled solve.

python tools/bench_mot.py [--config 2] [--N 16] [--tol 1e-8]

Builds a BEM_MODE_COMBINED operator on the config's mesh with N time steps
(T = 2, so Courant = (2/N)/h_max), prepares the time weights (eq:fastdft),
runs cqm_mot_solve (marching on in time, eq:cqmrhs) and cqm_solve (Remark
P:1607-1614) on the pulse data, and prints one JSON line with both times and
their relative difference (O(R^L) where the recursion is stable).
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2006_05186_b200 as pb  # noqa: E402
import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--N", type=int, default=16)
ap.add_argument("--tol", type=float, default=1e-8)
a = ap.parse_args()
cfg = synth.CONFIGS[a.config]
V, T = synth.config_mesh(a.config)
N = a.N
R = 10.0 ** (-5.0 / N)
s = pb.cqm_frequencies(N, 2.0, R)
t0 = time.perf_counter()
op = pb.Operator(pb.Tree(V, T, cfg["leaf"], cfg["eta"], cfg["m"]), s, cfg["eps"], mode=pb.BEM_MODE_COMBINED)
torch.cuda.synchronize()
t_asm = time.perf_counter() - t0
t0 = time.perf_counter()
op.mot_prepare(R)
t_prep = time.perf_counter() - t0
g = torch.from_numpy(synth.pulse(V, T, N, 2.0, shift=2.2)).cuda()


def timed(f):
    f()  # warm-up
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    out = f()
    e1.record()
    e1.synchronize()
    return out, e0.elapsed_time(e1)


(q, st), ms_mot = timed(lambda: pb.cqm_mot_solve(op, g, tol=a.tol, raise_on_noconv=False))
(phi, st2), ms_freq = timed(lambda: pb.cqm_solve(op, g, R, tol=a.tol, raise_on_noconv=False))
diff = float(torch.linalg.vector_norm(q - phi) / torch.linalg.vector_norm(phi))
print(json.dumps({"config": a.config, "M": len(T), "N": N, "mode": "combined", "tol": a.tol,
                  "assembly_s": t_asm, "mot_prepare_s": t_prep, "mot_ms": ms_mot, "mot_stats": st,
                  "freq_solve_ms": ms_freq, "freq_stats": st2, "rel_diff_mot_vs_freq": diff,
                  "max_abs_q": float(q.abs().max())}))
