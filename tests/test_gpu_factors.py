"""Factors-only MACA skeleton (SURVEY D8 / C10 skeleton form, AM17): the
coupling kernel regenerates each far block's coefficient tile
Z_b = U_b^{-1} C^_b^{-1} A_b[Q, l] from the r_b x r_b LU factors of A_b[Q, K]
(eq:maca P:1314-1320) instead of reading a stored Z.  The regeneration runs
the ACA's own pinned substitutions, so the two storage modes must agree bit
for bit, and both must match the oracle's identical-compression apply
within 1e-10."""
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


@pytest.mark.parametrize("m,leaf,N,eps,kernel", [
    (3, 32, 128, 1e-6, "0"),   # p = 27: far7, 3 DMMA row tiles + DFMA rows, leftover column l = 0
    (3, 32, 130, 1e-6, "8"),   # p = 27 on far8, padded DMMA columns (L mod 8 = 3)
    (4, 48, 256, 1e-6, "0"),   # p = 64: far8, 3 frequency tiles
    (5, 64, 64, 1e-8, "0"),    # p = 125: far8 with nu chunks
])
def test_factors_vs_stored_bitwise_and_oracle(pb, torch, m, leaf, N, eps, kernel, monkeypatch):
    monkeypatch.setenv("BEM_FAR_KERNEL", kernel)
    V, T = synth.icosphere(3)
    M, L = len(T), N + 1
    s = pb.cqm_frequencies(N, 2.0)
    tree = pb.Tree(V, T, leaf, 1.0, m)
    opz = pb.Operator(tree, s, eps, mode=pb.BEM_MODE_H2ACA | pb.BEM_SKEL_Z)
    opf = pb.Operator(tree, s, eps, mode=pb.BEM_MODE_H2ACA | pb.BEM_SKEL_FACTORS)
    assert opz.skeleton() == "Z" and opf.skeleton() == "factors"
    for k in ("ranks", "pivots"):
        assert np.array_equal(opz.aca_export()[k], opf.aca_export()[k])
    x = torch.from_numpy(synth.random_density(9, L, M)).cuda()
    yz, yf = opz.apply(x), opf.apply(x)
    assert torch.equal(yz, yf)
    assert torch.equal(opf.apply(x), yf)  # reproducible
    lsel = np.unique(np.r_[0, 1, 7, 8, N // 2, N - 1, N])
    oh = O.H2(V, T, leaf, 1.0, m)
    oh.aca(s, eps, keep=lsel)
    yo = oh.apply(O.MODE_H2ACA, s, x.cpu().numpy()[lsel], lsel)
    assert _rel(yf.cpu().numpy()[lsel], yo) <= 1e-10


def test_factors_local_shard_and_double_layer(pb, torch):
    """A frequency shard (what one rank of a G-GPU run holds) and the double-layer
    apply (same skeleton, other column basis) in factors mode."""
    V, T = synth.icosphere(3)
    N, eps = 64, 1e-6
    M, L = len(T), N + 1
    s = pb.cqm_frequencies(N, 2.0)
    local = np.array([0, 3, 62, 5, 60, 31, 34, 17, 48, 9, 56], dtype=np.int32)
    tree = pb.Tree(V, T, 48, 1.0, 4)
    opz = pb.Operator(tree, s, eps, mode=pb.BEM_MODE_H2ACA | pb.BEM_SKEL_Z, local_l=local)
    opf = pb.Operator(tree, s, eps, mode=pb.BEM_MODE_H2ACA | pb.BEM_SKEL_FACTORS, local_l=local)
    x = torch.from_numpy(synth.random_density(10, len(local), M)).cuda()
    assert torch.equal(opz.apply(x), opf.apply(x))
    assert torch.equal(opz.apply_dl(x, alpha=-0.5), opf.apply_dl(x, alpha=-0.5))
    oh = O.H2(V, T, 48, 1.0, 4)
    oh.aca(s, eps, keep=local)
    assert _rel(opf.apply(x).cpu().numpy(), oh.apply(O.MODE_H2ACA, s, x.cpu().numpy(), local)) <= 1e-10


def test_factors_solve_matches_stored(pb, torch):
    """The batched GMRES (masked applies: converged frequencies are skipped) gives the
    same solution with either skeleton storage."""
    V, T = synth.icosphere(3)
    N = 32
    R = 10.0 ** (-5.0 / N)
    s = pb.cqm_frequencies(N, 2.0)
    tree = pb.Tree(V, T, 32, 1.0, 3)
    g = torch.from_numpy(synth.pulse(V, T, N, 2.0)).cuda()
    out = []
    for flag in (pb.BEM_SKEL_Z, pb.BEM_SKEL_FACTORS):
        op = pb.Operator(tree, s, 1e-6, mode=pb.BEM_MODE_H2ACA | flag)
        phi, st = pb.cqm_solve(op, g, R, tol=1e-8, restart=20)
        out.append((phi.cpu().numpy(), st))
        op.close()
    assert out[0][1]["iters_sum"] == out[1][1]["iters_sum"] and out[0][1]["n_unconverged"] == 0
    assert np.array_equal(out[0][0], out[1][0])


def test_assembly_rejects_asymmetric_frequencies(pb):
    """The operator evaluates l > L/2 as the conjugate of L - l: a frequency set
    that is not conjugation-symmetric is refused (EINVAL), not silently mis-applied."""
    V, T = synth.icosphere(2)
    s = pb.cqm_frequencies(16, 2.0)
    tree = pb.Tree(V, T, 16, 1.0, 2)
    bad = s.copy()
    bad[3] += 1e-3
    with pytest.raises(pb.BemError) as ei:
        pb.Operator(tree, bad, 1e-6)
    assert ei.value.code == -1
    with pytest.raises(pb.BemError):
        pb.Operator(tree, s, 1e-6, mode=pb.BEM_MODE_H2ACA | pb.BEM_SKEL_Z | pb.BEM_SKEL_FACTORS)
