"""GPU parity of BEM_MODE_COMBINED (Alg. 3 in full: MACA on the near blocks too,
P:1414-1453 NEAR branch) against the oracle's MODE_COMBINED.

Bars (north_star / DESIGN.md §10): near- and far-block ranks and pivots
bit-exact; apply vs the identical-compression oracle <= 1e-10 relative l2;
l = 0 equals the exact near field (k_1 = 0 reading); bitwise reproducible.
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


def _apply(torch, op, x):
    y = op.apply(torch.from_numpy(np.ascontiguousarray(x)).cuda())
    torch.cuda.synchronize()
    return y.cpu().numpy()


def _case(pb, sub, leaf, m, N, eps, cfg=2):
    V, T = synth.icosphere(sub)
    s = pb.cqm_frequencies(N, 2.0)
    oh = O.H2(V, T, leaf, 1.0, m)
    oa = oh.aca(s, eps)
    on = oh.aca_near(s, eps)
    tree = pb.Tree(V, T, leaf, 1.0, m)
    op = pb.Operator(tree, s, eps, mode=pb.BEM_MODE_COMBINED)
    return V, T, s, oh, oa, on, tree, op


# (sub, leaf, m, N): leaves <= 32 rows (one row chunk) and <= 48 (two chunks);
# L = 33 (1 leftover column, one 32-column tile), 129 (1 leftover, two 64-column
# tiles), 70 (6 leftover columns)
@pytest.mark.parametrize("sub,leaf,m,N", [(3, 32, 3, 32), (3, 32, 3, 128), (3, 48, 4, 69), (2, 16, 2, 16)])
def test_combined_vs_oracle(pb, torch, sub, leaf, m, N):
    eps = 1e-6
    V, T, s, oh, oa, on, tree, op = _case(pb, sub, leaf, m, N, eps)
    M, L = len(T), N + 1
    ga = op.aca_export()
    assert np.array_equal(ga["ranks"], oa["ranks"]) and np.array_equal(ga["pivots"], oa["pivots"])
    gn = op.aca_export_near()
    assert np.array_equal(gn["ranks"], on["ranks"])
    assert np.array_equal(gn["pivots"], on["pivots"])
    x = synth.random_density(2, L, M)
    y = _apply(torch, op, x)
    lsel = np.unique(np.array([0, 1, L // 2, L // 2 + 1, L - 1]))
    yo = oh.apply(O.MODE_COMBINED, s, x[lsel], lsel)
    assert _rel(y[lsel], yo) <= 1e-10
    for i in range(len(lsel)):
        assert _rel(y[lsel[i]], yo[i]) <= 1e-8
    # l = 0 is every near block's first pivot: the near field there is exact
    ya = oh.apply(O.MODE_H2ACA, s, x[:1], np.array([0]))
    assert _rel(y[:1], ya) <= 1e-12
    assert np.array_equal(y, _apply(torch, op, x))  # bitwise reproducible


def test_combined_local_subset_and_dl(pb, torch):
    """Frequency shard (paired and unpaired local frequencies) and the double
    layer of a combined op (its near field stays exact: equals the H2ACA op's)."""
    V, T = synth.icosphere(3)
    N, eps = 32, 1e-6
    M = len(T)
    s = pb.cqm_frequencies(N, 2.0)
    loc = np.array([0, 5, 28, 7, 31, 16], dtype=np.int32)
    tree = pb.Tree(V, T, 32, 1.0, 3)
    op = pb.Operator(tree, s, eps, mode=pb.BEM_MODE_COMBINED, local_l=loc)
    oh = O.H2(V, T, 32, 1.0, 3)
    oh.aca(s, eps)
    oh.aca_near(s, eps)
    x = synth.random_density(4, len(loc), M)
    y = _apply(torch, op, x)
    assert _rel(y, oh.apply(O.MODE_COMBINED, s, x, loc)) <= 1e-10
    xt = torch.from_numpy(x).cuda()
    yk = op.apply_dl(xt, alpha=-0.5).cpu().numpy()
    op2 = pb.Operator(tree, s, eps, mode=pb.BEM_MODE_H2ACA, local_l=loc)
    yk2 = op2.apply_dl(xt, alpha=-0.5).cpu().numpy()
    assert np.array_equal(yk, yk2)


def test_combined_solve(pb, torch):
    """Frequency-decoupled GMRES on the combined operator; residual re-evaluated
    by the oracle's MODE_COMBINED apply."""
    V, T = synth.icosphere(3)
    N = 32
    R = 10.0 ** (-5.0 / N)
    s = pb.cqm_frequencies(N, 2.0)
    local = np.array([0, 3, 16, 17, 30], dtype=np.int32)
    op = pb.Operator(pb.Tree(V, T, 32, 1.0, 3), s, 1e-8, mode=pb.BEM_MODE_COMBINED, local_l=local)
    g = synth.pulse(V, T, N, 2.0)
    gf = O.forward(g.astype(np.complex128), N, R)[local]
    phi, st = pb.solve_multifreq(op, torch.from_numpy(np.ascontiguousarray(gf)).cuda(), tol=1e-9, restart=20)
    phi = phi.cpu().numpy()
    assert st["n_unconverged"] == 0 and st["resid_max"] <= 1e-9
    oh = O.H2(V, T, 32, 1.0, 3)
    oh.aca(s, 1e-8)
    oh.aca_near(s, 1e-8)
    res = oh.apply(O.MODE_COMBINED, s, phi, local) - gf
    assert np.max(np.linalg.norm(res, axis=1) / np.linalg.norm(gf, axis=1)) <= 1.5e-9


def test_combined_config2_full_size(pb, torch):
    """Config 2 at full size in the bench's launch configuration: near pivots
    bit-exact on a block sample, the combined apply within 10 eps of the H2ACA
    apply (exact near field), exact at l = 0, oracle-sampled frequencies."""
    V, T = synth.config_mesh(2)
    N, eps = 128, 1e-6
    M, L = len(T), N + 1
    s = pb.cqm_frequencies(N, 2.0)
    tree = pb.Tree(V, T, 32, 1.0, 3)
    op = pb.Operator(tree, s, eps, mode=pb.BEM_MODE_COMBINED)
    opa = pb.Operator(tree, s, eps, mode=pb.BEM_MODE_H2ACA)
    x = synth.random_density(2, L, M)
    y = _apply(torch, op, x)
    ya = _apply(torch, opa, x)
    assert _rel(y, ya) <= 10 * eps
    assert _rel(y[0], ya[0]) <= 1e-12
    gn = op.aca_export_near()
    oh = O.H2(V, T, 32, 1.0, 3)
    blk = np.arange(0, oh.n_near, 97, dtype=np.int32)
    on = oh.aca_near(s, eps, blocks=blk)
    off = np.r_[0, np.cumsum(gn["ranks"])]
    assert np.array_equal(gn["ranks"][blk], on["ranks"])
    assert np.array_equal(np.concatenate([gn["pivots"][off[b]:off[b + 1]] for b in blk]), on["pivots"])


def test_combined_edge_cases(pb, torch):
    """Leaves above 64 panels are refused (EINVAL); a tree whose partition has no
    far blocks (80 panels, one level) runs the near-only paths of the combined
    apply and of the time-domain convolution."""
    V, T = synth.icosphere(2)
    s = pb.cqm_frequencies(8, 2.0)
    with pytest.raises(pb.BemError):
        pb.Operator(pb.Tree(V, T, 10 ** 6, 1.0, 2), s, 1e-6, mode=pb.BEM_MODE_COMBINED)
    V, T = synth.icosphere(1)
    N = 8
    M, L, R = len(T), N + 1, O.default_R(N)
    tree = pb.Tree(V, T, 48, 1.0, 2)
    op = pb.Operator(tree, s, 1e-8, mode=pb.BEM_MODE_COMBINED)
    oh = O.H2(V, T, 48, 1.0, 2)
    oh.aca(s, 1e-8)
    oh.aca_near(s, 1e-8)
    x = synth.random_density(2, L, M)
    assert _rel(_apply(torch, op, x), oh.apply(O.MODE_COMBINED, s, x)) <= 1e-10
    op.mot_prepare(R)
    oh.time_weights(R)
    q = np.random.default_rng(5).standard_normal((L, M)) + 0j
    assert _rel(op.conv_time(torch.from_numpy(q).cuda()).cpu().numpy(), oh.conv(q)) <= 1e-10
