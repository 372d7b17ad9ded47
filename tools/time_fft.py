"""Warm timing of the K4 transforms (cqm_forward / cqm_inverse) at the configs' shapes."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2006_05186_b200 as pb  # noqa: E402

out = {}
for name, M, N in (("config2", 5120, 128), ("config3", 20480, 256), ("config4", 81920, 512),
                   ("config5_rank_of_2", 163840, 1024)):
    R = 10.0 ** (-5.0 / N)
    x = torch.randn(N + 1, M, dtype=torch.complex128, device="cuda")
    for _ in range(3):
        y = pb.cqm_forward(x, N, R)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 20
    e0.record()
    for _ in range(reps):
        y = pb.cqm_forward(x, N, R)
    e1.record()
    e1.synchronize()
    ms = e0.elapsed_time(e1) / reps
    e0.record()
    for _ in range(reps):
        z = pb.cqm_inverse(y, N, R)
    e1.record()
    e1.synchronize()
    msi = e0.elapsed_time(e1) / reps
    bytes_ = 32.0 * M * (N + 1)
    out[name] = {"forward_ms": ms, "inverse_ms": msi, "forward_GB/s": bytes_ / (ms * 1e-3) / 1e9,
                 "inverse_GB/s": bytes_ / (msi * 1e-3) / 1e9}
print(json.dumps(out))
