"""Small invocations of every hot kernel for compute-sanitizer (race and
memory checks).  1280-panel sphere, short frequency sets; each case runs one apply:
  far7 (p = 27, stored Z), far8 (p = 64 with leftover / padded columns; p = 125 with
  nu chunks), the factors-only Z-tile pass, h2o (plain H2), K1m (combined mode),
  the K2 leaf (DMMA) and Kronecker transfer kernels (every apply), K4 Stockham
  (L = 33, 129) and Bluestein (L = 257), the ACA assembly.
Usage: compute-sanitizer --tool racecheck python tools/sanitize_case.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2006_05186_b200 as pb  # noqa: E402
import synth  # noqa: E402

V, T = synth.icosphere(3)
M = len(T)
cases = [
    ("far7 p=27 stored Z", 3, 32, 32, pb.BEM_MODE_H2ACA | pb.BEM_SKEL_Z),
    ("far8 p=64 stored Z, L=34 (padded columns)", 4, 48, 33, pb.BEM_MODE_H2ACA | pb.BEM_SKEL_Z),
    ("far8 p=64 factors-only", 4, 48, 32, pb.BEM_MODE_H2ACA | pb.BEM_SKEL_FACTORS),
    ("far8 p=125 factors-only", 5, 64, 16, pb.BEM_MODE_H2ACA | pb.BEM_SKEL_FACTORS),
    ("far7 p=27 factors-only", 3, 32, 16, pb.BEM_MODE_H2ACA | pb.BEM_SKEL_FACTORS),
    ("h2o plain H2", 4, 48, 16, pb.BEM_MODE_H2ONLY),
    ("combined (K1m near-field MACA)", 3, 32, 16, pb.BEM_MODE_COMBINED),
]
for name, m, leaf, N, mode in cases:
    s = pb.cqm_frequencies(N, 2.0)
    op = pb.Operator(pb.Tree(V, T, leaf, 1.0, m), s, 1e-6, mode=mode)
    x = torch.from_numpy(synth.random_density(2, N + 1, M)).cuda()
    y = op.apply(x)
    torch.cuda.synchronize()
    print(name, "ok", float(torch.linalg.vector_norm(y)))
for N in (32, 128, 256):
    R = 10.0 ** (-5.0 / N)
    x = torch.from_numpy(np.random.default_rng(N).standard_normal((N + 1, 37)) + 0j).cuda()
    z = pb.cqm_inverse(pb.cqm_forward(x, N, R), N, R)
    torch.cuda.synchronize()
    print("K4 L =", N + 1, "ok", float(torch.linalg.vector_norm(z - x) / torch.linalg.vector_norm(x)))
