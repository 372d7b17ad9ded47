"""GPU parity of the time-domain path with compressed weights (SURVEY §8(f)
NEXT-2: eq:fastdft P:1542-1553, eq:fastrhs P:1566-1573, MoT eq:cqmrhs
P:652-680) against the oracle (tests/test_oracle_mot.py pins the oracle).

Bars: the convolution with compressed weights within 1e-10 relative l2 of the
oracle's; the MoT solution within 1e-8 of the oracle's LU-based MoT (GMRES to
1e-12 per step); at config-2 size the recursion holds through the library's
own convolution and the solution agrees with the frequency-decoupled solve up
to the O(R^L) wrap-around.  Steps run at Courant numbers where the recursion of
this collocation discretisation is stable.
"""
import numpy as np
import pytest

import oracle as O
import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch():
    import torch as _t
    assert _t.cuda.is_available()
    return _t


@pytest.fixture(scope="module")
def pb():
    import paper_2006_05186_b200 as _pb
    _pb.lib()
    return _pb


def _rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


def _pair(pb, sub, leaf, m, N, eps):
    V, T = synth.icosphere(sub)
    R = O.default_R(N)
    s = pb.cqm_frequencies(N, 2.0)
    op = pb.Operator(pb.Tree(V, T, leaf, 1.0, m), s, eps, mode=pb.BEM_MODE_COMBINED)
    op.mot_prepare(R)
    oh = O.H2(V, T, leaf, 1.0, m)
    oh.aca(s, eps)
    oh.aca_near(s, eps)
    oh.time_weights(R)
    return V, T, R, s, op, oh


@pytest.mark.parametrize("sub,leaf,m,N", [(2, 16, 2, 16), (3, 32, 3, 32)])
def test_conv_time_vs_oracle(pb, torch, sub, leaf, m, N):
    V, T, R, s, op, oh = _pair(pb, sub, leaf, m, N, 1e-8)
    M, L = len(T), N + 1
    q = np.random.default_rng(3).standard_normal((L, M)) + 0j
    qd = torch.from_numpy(q).cuda()
    y = op.conv_time(qd).cpu().numpy()
    yo = oh.conv(q)
    assert _rel(y, yo) <= 1e-10
    y5 = op.conv_time(qd, kmax=5).cpu().numpy()
    assert _rel(y5, oh.conv(q, kmax=5)) <= 1e-10
    # the frequency path of the same op differs by the R^L wrap-around only
    yf = pb.cqm_inverse(op.apply(pb.cqm_forward(qd, N, R)), N, R).cpu().numpy()
    assert 1e-9 < _rel(yf, y) <= 1e-3


def test_mot_vs_oracle(pb, torch):
    V, T, R, s, op, oh = _pair(pb, 2, 16, 3, 16, 1e-8)
    N = 16
    g = synth.pulse(V, T, N, 2.0, shift=2.2)
    q, st = pb.cqm_mot_solve(op, torch.from_numpy(g).cuda(), tol=1e-12, restart=50)
    q = q.cpu().numpy()
    assert st["n_unconverged"] == 0 and st["resid_max"] <= 1e-12
    qo = oh.mot(g)
    assert _rel(q, qo) <= 1e-8


def test_mot_config2_mesh(pb, torch):
    """5,120-panel sphere at N = 16 (Courant ~1.5): the recursion through the
    library's convolution, and agreement with the frequency-decoupled solve."""
    V, T = synth.config_mesh(2)
    N = 16
    M, L, R = len(T), N + 1, O.default_R(N)
    s = pb.cqm_frequencies(N, 2.0)
    op = pb.Operator(pb.Tree(V, T, 32, 1.0, 3), s, 1e-8, mode=pb.BEM_MODE_COMBINED)
    op.mot_prepare(R)
    g = torch.from_numpy(synth.pulse(V, T, N, 2.0, shift=2.2)).cuda()
    q, st = pb.cqm_mot_solve(op, g, tol=1e-12)
    assert st["n_unconverged"] == 0
    res = op.conv_time(q.to(torch.complex128)).real - g
    assert float(torch.linalg.vector_norm(res) / torch.linalg.vector_norm(g)) <= 1e-10
    phi, st2 = pb.cqm_solve(op, g, R, tol=1e-12)
    assert float(torch.linalg.vector_norm(q - phi) / torch.linalg.vector_norm(phi)) <= 1e-4
