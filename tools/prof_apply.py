"""Minimal driver for ncu captures: build a config, run a few applies."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2006_05186_b200 as pb  # noqa: E402
import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--mode", default="h2aca")
ap.add_argument("--time-step", action="store_true", help="forward + apply + inverse")
ap.add_argument("--skeleton", default="auto", choices=["auto", "z", "factors"])
a = ap.parse_args()
cfg = synth.CONFIGS[a.config]
V, T = synth.config_mesh(a.config)
N = cfg["N"]
R = 10.0 ** (-5.0 / N)
s = pb.cqm_frequencies(N, cfg["T"], R)
tree = pb.Tree(V, T, cfg["leaf"], cfg["eta"], cfg["m"])
mode = {"h2aca": pb.BEM_MODE_H2ACA, "h2only": pb.BEM_MODE_H2ONLY, "dense": pb.BEM_MODE_DENSE,
        "combined": pb.BEM_MODE_COMBINED}[a.mode]
if mode in (pb.BEM_MODE_H2ACA, pb.BEM_MODE_COMBINED):
    mode |= {"auto": 0, "z": pb.BEM_SKEL_Z, "factors": pb.BEM_SKEL_FACTORS}[a.skeleton]
op = pb.Operator(tree, s, cfg["eps"], mode=mode)
x = torch.from_numpy(synth.random_density(a.config, N + 1, len(T))).cuda()
for _ in range(a.reps):
    if a.time_step:
        pb.cqm_inverse(op.apply(pb.cqm_forward(x, N, R)), N, R)
    else:
        op.apply(x)
torch.cuda.synchronize()
print("ok", tree.stats)
