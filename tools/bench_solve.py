"""Full CQM solve benchmark (config 3's timed entry point is cqm_solve).

python tools/bench_solve.py [--config 3] [--tol 1e-8] [--restart 50] [--check-freqs 4]

Solves V(s_l) phi^_l = g^_l for every l by the library's batched GMRES
(cqm_solve: forward transform, GMRES per frequency, inverse), with the pulse
data of BASELINE.json, then re-evaluates the frequency-domain residual of the
returned phi through the library's own apply and (optionally) through the
CPU oracle's H2ACA apply on a few frequencies.  Prints one JSON line.
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2006_05186_b200 as pb  # noqa: E402
import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=3)
ap.add_argument("--tol", type=float, default=1e-8)
ap.add_argument("--restart", type=int, default=50)
ap.add_argument("--max-iter", type=int, default=2000)
ap.add_argument("--check-freqs", type=int, default=0, help="oracle residual check on this many frequencies")
ap.add_argument("--dirichlet", action="store_true",
                help="direct Dirichlet formulation V q = (-1/2 I + K) g (NEXT-1) instead of the indirect V phi = g")
ap.add_argument("--mode", default="h2aca", choices=["h2aca", "h2only"])
a = ap.parse_args()

cfg = synth.CONFIGS[a.config]
V, T = synth.config_mesh(a.config)
N = cfg["N"]
M, L = len(T), N + 1
R = 10.0 ** (-5.0 / N)
s = pb.cqm_frequencies(N, cfg["T"], R)
t0 = time.perf_counter()
leaf = cfg["leaf"] if not cfg.get("dense") else 10 ** 6
tree = pb.Tree(V, T, leaf, cfg["eta"], cfg["m"])
mode = pb.BEM_MODE_DENSE if cfg.get("dense") else (pb.BEM_MODE_H2ACA if a.mode == "h2aca" else pb.BEM_MODE_H2ONLY)
op = pb.Operator(tree, s, cfg["eps"], mode=mode)
torch.cuda.synchronize()
t_setup = time.perf_counter() - t0
g = torch.from_numpy(synth.pulse(V, T, N, cfg["T"])).cuda()

def solve():
    if a.dirichlet:
        return pb.dirichlet_solve(op, g, R, tol=a.tol, restart=a.restart, max_iter=a.max_iter)
    return pb.cqm_solve(op, g, R, tol=a.tol, restart=a.restart, max_iter=a.max_iter)


solve()  # warm-up (allocations, caches)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
phi, st = solve()
e1.record()
e1.synchronize()
ms = e0.elapsed_time(e1)
# residual re-evaluation through the library's apply: forward(phi) vs forward(g)
gf = pb.cqm_forward(g.to(torch.complex128), N, R)
pf = pb.cqm_forward(phi.to(torch.complex128), N, R)
res = op.apply(pf) - (op.apply_dl(gf, alpha=-0.5) if a.dirichlet else gf)
rhs_n = op.apply_dl(gf, alpha=-0.5) if a.dirichlet else gf
rel = (torch.linalg.vector_norm(res, dim=1) / torch.linalg.vector_norm(rhs_n, dim=1)).cpu().numpy()
out = {"config": a.config, "formulation": "direct Dirichlet (NEXT-1)" if a.dirichlet else "indirect V phi = g",
       "mode": a.mode, "M": M, "L": L, "tol": a.tol, "restart": a.restart, "solve_ms": ms,
       "setup_s": t_setup, "stats": st, "max_rel_residual_relib": float(rel.max()),
       "apply_equivalents_per_s": None}
if st["iters_sum"]:
    # every GMRES inner iteration applies V(s_l) to the still-active frequencies
    out["frequency_iterations"] = int(st["iters_sum"])
    out["unknowns_x_freq_iterations_per_s"] = M * st["iters_sum"] / (ms * 1e-3)
if a.check_freqs > 0 and not a.dirichlet:
    import oracle as O
    oh = O.H2(V, T, leaf, cfg["eta"], cfg["m"])
    if mode == pb.BEM_MODE_H2ACA:
        oh.aca(s, cfg["eps"])
    lsel = np.linspace(0, L - 1, a.check_freqs).round().astype(np.int32)
    pfn = pf.cpu().numpy()[lsel]
    gfn = gf.cpu().numpy()[lsel]
    omode = O.MODE_DENSE if cfg.get("dense") else O.MODE_H2ACA
    ro = oh.apply(omode, s, pfn, lsel) - gfn
    out["oracle_rel_residual"] = (np.linalg.norm(ro, axis=1) / np.linalg.norm(gfn, axis=1)).tolist()
    out["oracle_freqs"] = lsel.tolist()
print(json.dumps(out))
