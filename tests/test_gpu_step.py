"""bem_time_step: the library's one-call time-domain step (K4 forward, apply,
K4 inverse from a captured CUDA graph), with device and host buffers, is
bitwise identical to the eager composition of the same C-ABI calls, and the
composition matches the oracle (forward, H2ACA apply, inverse)."""
import numpy as np
import pytest

import oracle as O
import synth

pytestmark = pytest.mark.gpu


def test_time_step_graph_matches_eager_and_oracle():
    import torch
    import paper_2006_05186_b200 as pb
    V, T = synth.icosphere(3)
    N = 32
    M, L, R = len(T), N + 1, O.default_R(N)
    s = pb.cqm_frequencies(N, 2.0)
    op = pb.Operator(pb.Tree(V, T, 32, 1.0, 3), s, 1e-6)
    xt = synth.random_time_data(2, N, M).astype(np.complex128)
    xd = torch.from_numpy(xt).cuda()
    ref = pb.cqm_inverse(op.apply(pb.cqm_forward(xd, N, R)), N, R)
    y1 = op.time_step(xd, R)            # first call: eager pass + capture
    y2 = op.time_step(xd, R)            # graph replay
    yh = op.time_step(torch.from_numpy(xt).pin_memory(), R)   # host buffers
    torch.cuda.synchronize()
    assert torch.equal(y1, ref) and torch.equal(y2, ref)
    assert np.array_equal(yh.numpy(), ref.cpu().numpy())
    y3 = op.time_step(xd, 0.5 * R + 0.5)  # another R: re-captured
    ref3 = pb.cqm_inverse(op.apply(pb.cqm_forward(xd, N, 0.5 * R + 0.5)), N, 0.5 * R + 0.5)
    assert torch.equal(y3, ref3)
    oh = O.H2(V, T, 32, 1.0, 3)
    oh.aca(s, 1e-6)
    yo = O.inverse(oh.apply(O.MODE_H2ACA, s, O.forward(xt, N, R)), N, R)
    yg = y2.cpu().numpy()
    assert np.linalg.norm(yg - yo) / np.linalg.norm(yo) <= 1e-10


@pytest.mark.parametrize("mode", ["h2only", "combined", "dense"])
def test_time_step_other_modes(mode):
    """The captured graph also covers the plain-H^2 couplings (K3'), the combined
    mode's near-field MACA (K1m, persistent work queue reset inside the graph) and
    the dense mode (no far field, no side stream)."""
    import torch
    import paper_2006_05186_b200 as pb
    V, T = synth.icosphere(2 if mode == "dense" else 3)
    N = 16
    M, R = len(T), O.default_R(N)
    s = pb.cqm_frequencies(N, 2.0)
    leaf = 10 ** 6 if mode == "dense" else 32
    m = {"h2only": pb.BEM_MODE_H2ONLY, "combined": pb.BEM_MODE_COMBINED, "dense": pb.BEM_MODE_DENSE}[mode]
    op = pb.Operator(pb.Tree(V, T, leaf, 1.0, 3 if mode != "dense" else 1), s, 1e-6, mode=m)
    xd = torch.from_numpy(synth.random_time_data(2, N, M).astype(np.complex128)).cuda()
    ref = pb.cqm_inverse(op.apply(pb.cqm_forward(xd, N, R)), N, R)
    for _ in range(3):
        y = op.time_step(xd, R)
    torch.cuda.synchronize()
    assert torch.equal(y, ref)
