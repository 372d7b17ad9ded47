"""GPU parity: the CUDA library (through the C-ABI) against the CPU oracle.

Tolerances (SURVEY C13 / north_star):
  * trees, admissibility lists, ACA ranks and pivots: bit-exact;
  * apply vs identical-compression oracle: global relative l2 <= 1e-10
    (per-frequency reported, gated at 1e-8);
  * apply vs dense: <= 10 max(eps_ACA, e_H2), e_H2 measured by the oracle;
  * time domain compared on R^n-scaled sequences (R^{-N} = 1e5 conditioning);
  * solve: residual <= 1e-8 (re-evaluated by the oracle, slack 1.5e-8).
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


def _apply(pb, torch, op, x):
    xt = torch.from_numpy(np.ascontiguousarray(x)).cuda()
    y = op.apply(xt)
    torch.cuda.synchronize()
    return y.cpu().numpy()


def test_pinned_functions_bitwise_identical(pb):
    """C14: device pinned exp/sincos bit-identical to the oracle's on 1e6 arguments."""
    rng = np.random.default_rng(0)
    x = np.concatenate([-rng.random(400000) * 745.0, rng.random(600000) * 6500.0, [0.0, -746.5, -745.2, 1e-300]])
    e, s, c = pb.debug_pinned(x)
    assert np.array_equal(e.view(np.uint64), O.pexp(x).view(np.uint64))
    so, co = O.psincos(x)
    assert np.array_equal(s.view(np.uint64), so.view(np.uint64))
    assert np.array_equal(c.view(np.uint64), co.view(np.uint64))


def test_dense_config1(pb, torch):
    """Minimum slice: config 1, dense mode, all 33 frequencies."""
    V, T = synth.config_mesh(1)
    N = 32
    M, L = len(T), N + 1
    s = pb.cqm_frequencies(N, 2.0)
    tree = pb.Tree(V, T, 10 ** 6, 1.0, 1)
    op = pb.Operator(tree, s, 1e-6, mode=pb.BEM_MODE_DENSE)
    x = synth.random_density(1, L, M)
    y = _apply(pb, torch, op, x)
    yo = O.H2(V, T, 10 ** 6, 1.0, 1).apply(O.MODE_DENSE, s, x)
    assert _rel(y, yo) <= 1e-10
    for l in range(L):
        assert _rel(y[l], yo[l]) <= 1e-10, l


def test_tree_on_device_matches_oracle(pb):
    V, T = synth.icosphere(3)
    a = pb.Tree(V, T, 32, 1.0, 3).export()
    b = O.H2(V, T, 32, 1.0, 3).export()
    for k in a:
        assert np.array_equal(a[k], b[k]), k


@pytest.mark.parametrize("N", [32, 128])
def test_h2aca_1280_all_modes(pb, torch, N):
    """1280-panel sphere with config-2 parameters: H2ONLY and H2ACA vs the
    identical oracle (<= 1e-10), pivots bit-exact, and vs dense <= 10 max(eps, e_H2)."""
    V, T = synth.icosphere(3)
    M, L, eps = len(T), N + 1, 1e-6
    s = pb.cqm_frequencies(N, 2.0)
    x = synth.random_density(2, L, M)
    oh = O.H2(V, T, 32, 1.0, 3)
    oa = oh.aca(s, eps)
    tree = pb.Tree(V, T, 32, 1.0, 3)
    op = pb.Operator(tree, s, eps, mode=pb.BEM_MODE_H2ACA)
    ga = op.aca_export()
    assert np.array_equal(ga["ranks"], oa["ranks"])
    assert np.array_equal(ga["pivots"], oa["pivots"])
    y = _apply(pb, torch, op, x)
    yo = oh.apply(O.MODE_H2ACA, s, x)
    assert _rel(y, yo) <= 1e-10
    for l in range(L):
        assert _rel(y[l], yo[l]) <= 1e-8
    op2 = pb.Operator(tree, s, eps, mode=pb.BEM_MODE_H2ONLY)
    y2 = _apply(pb, torch, op2, x)
    yo2 = oh.apply(O.MODE_H2ONLY, s, x)
    assert _rel(y2, yo2) <= 1e-10
    lsel = np.array([0, 1, N // 2, N])
    yd = oh.apply(O.MODE_DENSE, s, x[lsel], lsel)
    eh2 = _rel(yo2[lsel], yd)
    assert _rel(y[lsel], yd) <= 10 * max(eps, eh2)


def test_aca_pivots_bitexact_config2(pb):
    """Config 2 (5120 panels, L=129, m=3, eps=1e-6): every far block's rank and
    pivot sequence bit-identical to the oracle's ACA."""
    V, T = synth.config_mesh(2)
    s = pb.cqm_frequencies(128, 2.0)
    tree = pb.Tree(V, T, 32, 1.0, 3)
    op = pb.Operator(tree, s, 1e-6, mode=pb.BEM_MODE_H2ACA, local_l=[0, 1])
    ga = op.aca_export()
    oa = O.H2(V, T, 32, 1.0, 3).aca(s, 1e-6)
    assert np.array_equal(ga["ranks"], oa["ranks"])
    assert np.array_equal(ga["pivots"], oa["pivots"])
    assert 15 < ga["ranks"].mean() < 40


def test_config2_full_apply_sampled(pb, torch):
    """Config 2 at full size in the bench's launch configuration (all 129
    frequencies on one device); the oracle evaluates a frequency sample."""
    V, T = synth.config_mesh(2)
    N, M = 128, len(T)
    L = N + 1
    s = pb.cqm_frequencies(N, 2.0)
    tree = pb.Tree(V, T, 32, 1.0, 3)
    op = pb.Operator(tree, s, 1e-6)
    x = synth.random_density(2, L, M)
    y = _apply(pb, torch, op, x)
    lsel = np.array([0, 3, 64, 127])
    oh = O.H2(V, T, 32, 1.0, 3)
    oh.aca(s, 1e-6)
    yo = oh.apply(O.MODE_H2ACA, s, x[lsel], lsel)
    assert _rel(y[lsel], yo) <= 1e-10
    y2 = _apply(pb, torch, op, x)
    assert np.array_equal(y, y2)  # bitwise reproducible


def test_local_frequency_subset(pb, torch):
    """Frequency sharding: a local set with paired (l, L-l) and
    unpaired frequencies gives the same columns as the oracle."""
    V, T = synth.icosphere(3)
    N = 32
    M, L = len(T), N + 1
    s = pb.cqm_frequencies(N, 2.0)
    loc = np.array([0, 5, 28, 7, 31, 2, 16])  # (5,28) paired; 7, 31, 2, 16 unpaired
    tree = pb.Tree(V, T, 32, 1.0, 3)
    op = pb.Operator(tree, s, 1e-6, local_l=loc)
    x = synth.random_density(3, len(loc), M)
    y = _apply(pb, torch, op, x)
    oh = O.H2(V, T, 32, 1.0, 3)
    oh.aca(s, 1e-6)
    yo = oh.apply(O.MODE_H2ACA, s, x, loc)
    assert _rel(y, yo) <= 1e-10


@pytest.mark.parametrize("N", [1, 32, 128, 256, 512, 1024])
def test_transforms_vs_oracle(pb, torch, N):
    """K4 vs the oracle's naive DFTs; round trip on R^n-scaled sequences.  N = 512 and
    1024 are configs 4 and 5 (L = 513, 1025)."""
    L, M = N + 1, 37
    R = 10.0 ** (-5.0 / N) if N > 1 else 0.3
    rng = np.random.default_rng(N)
    xt = rng.standard_normal((L, M)) + 1j * rng.standard_normal((L, M))
    xg = torch.from_numpy(xt).cuda()
    xf = pb.cqm_forward(xg, N, R)
    xo = O.forward(xt, N, R)
    assert _rel(xf.cpu().numpy(), xo) <= 1e-12
    back = pb.cqm_inverse(xf, N, R).cpu().numpy()
    sc = (R ** np.arange(L))[:, None]
    assert _rel(back * sc, xt * sc) <= 1e-12
    yo = O.inverse(xo, N, R)
    assert _rel(back * sc, yo * sc) <= 1e-12


def test_time_domain_operator_config1(pb, torch):
    """(Vx)_n = inverse(V(s_l) forward(x)_l)_n on config 1 vs the oracle chain."""
    V, T = synth.config_mesh(1)
    N = 32
    M, L = len(T), N + 1
    R = 10.0 ** (-5.0 / N)
    s = pb.cqm_frequencies(N, 2.0)
    op = pb.Operator(pb.Tree(V, T, 10 ** 6, 1.0, 1), s, 1e-6, mode=pb.BEM_MODE_DENSE)
    xt = synth.random_time_data(1, N, M).astype(np.complex128)
    xf = pb.cqm_forward(torch.from_numpy(xt).cuda(), N, R)
    yt = pb.cqm_inverse(op.apply(xf), N, R).cpu().numpy()
    oh = O.H2(V, T, 10 ** 6, 1.0, 1)
    yo = O.inverse(oh.apply(O.MODE_DENSE, s, O.forward(xt, N, R)), N, R)
    sc = (R ** np.arange(L))[:, None]
    assert _rel(yt * sc, yo * sc) <= 1e-10


def test_solve_config1(pb, torch):
    """cqm_solve (frequency-decoupled GMRES) vs the oracle's GMRES: residual
    re-evaluated by the oracle, solutions within kappa * tol."""
    V, T = synth.config_mesh(1)
    N = 32
    M, L = len(T), N + 1
    R = 10.0 ** (-5.0 / N)
    s = pb.cqm_frequencies(N, 2.0)
    op = pb.Operator(pb.Tree(V, T, 10 ** 6, 1.0, 1), s, 1e-6, mode=pb.BEM_MODE_DENSE)
    g = synth.pulse(V, T, N, 2.0)
    phi, st = pb.cqm_solve(op, torch.from_numpy(g).cuda(), R, tol=1e-8)
    phi = phi.cpu().numpy()
    assert st["n_unconverged"] == 0 and st["resid_max"] <= 1e-8
    oh = O.H2(V, T, 10 ** 6, 1.0, 1)
    gf = O.forward(g, N, R)
    phif = O.forward(phi, N, R)
    res = oh.apply(O.MODE_DENSE, s, phif) - gf
    # phi is the real part of the inverse; its transform carries the O(tol) imaginary residue
    rel = np.linalg.norm(res, axis=1) / np.linalg.norm(gf, axis=1)
    assert np.max(rel) <= 1e-6
    xo, it, rr = oh.gmres(O.MODE_DENSE, s, gf, tol=1e-8)
    phio = O.inverse(xo, N, R).real
    sc = (R ** np.arange(L))[:, None]
    assert _rel(phi * sc, phio * sc) <= 1e-6


def test_solve_h2aca_small(pb, torch):
    """cqm_solve with the H2ACA operator on a 1280-panel sphere (N=16)."""
    V, T = synth.icosphere(3)
    N = 16
    M, L = len(T), N + 1
    R = 10.0 ** (-5.0 / N)
    s = pb.cqm_frequencies(N, 2.0)
    op = pb.Operator(pb.Tree(V, T, 32, 1.0, 3), s, 1e-8)
    g = synth.pulse(V, T, N, 2.0)
    phi, st = pb.cqm_solve(op, torch.from_numpy(g).cuda(), R, tol=1e-8, restart=30)
    assert st["n_unconverged"] == 0
    oh = O.H2(V, T, 32, 1.0, 3)
    oh.aca(s, 1e-8)
    gf = O.forward(g, N, R)
    xo, it, rr = oh.gmres(O.MODE_H2ACA, s, gf, tol=1e-8, restart=30)
    phio = O.inverse(xo, N, R).real
    sc = (R ** np.arange(L))[:, None]
    assert _rel(phi.cpu().numpy() * sc, phio * sc) <= 1e-6


def test_edge_cases(pb, torch):
    """Single panel, even L (N = 1), zero input, leaf_size >= M."""
    V = np.array([[0.0, 0, 0], [0.3, 0, 0], [0.1, 0.25, 0.02]])
    T = np.array([[0, 1, 2]], dtype=np.int32)
    for N in (1, 4):
        s = pb.cqm_frequencies(N, 2.0)
        op = pb.Operator(pb.Tree(V, T, 8, 1.0, 2), s, 1e-6)
        x = synth.random_density(4, N + 1, 1)
        y = _apply(pb, torch, op, x)
        A = np.array([O.dense_matrix(V, T, sl)[0, 0] for sl in s])
        assert np.max(np.abs(y[:, 0] - A * x[:, 0])) <= 1e-13 * np.max(np.abs(A * x[:, 0]))
    V, T = synth.icosphere(2)
    s = pb.cqm_frequencies(1, 1.0, 1e-5)
    op = pb.Operator(pb.Tree(V, T, 16, 1.0, 2), s, 1e-6)
    assert np.all(_apply(pb, torch, op, np.zeros((2, len(T)), complex)) == 0)
    x = synth.random_density(5, 2, len(T))
    oh = O.H2(V, T, 16, 1.0, 2)
    oh.aca(s, 1e-6)
    assert _rel(_apply(pb, torch, op, x), oh.apply(O.MODE_H2ACA, s, x)) <= 1e-10


@pytest.mark.parametrize("N,kernel,m3,dt", [(256, "7", "0", "1"), (260, "7", "0", "1"), (256, "8", "0", "1"),
                                             (260, "8", "0", "1"), (256, "8", "1", "1"), (260, "8", "1", "1"),
                                             (260, "8", "1", "0")])
def test_h2aca_p64_multi_tile(pb, torch, N, kernel, m3, dt, monkeypatch):
    """p = 64 (m = 4) with L > 128: K3 runs several frequency tiles per
    (segment, mu chunk).  N = 260 (L mod 8 = 5) exercises the zero-padded DMMA
    columns, N = 256 the distributed leftover column.  Oracle on a frequency sample."""
    monkeypatch.setenv("BEM_FAR_KERNEL", kernel)
    monkeypatch.setenv("BEM_FAR8_M3", m3)  # 3M complex products at 16-row mu chunks
    monkeypatch.setenv("BEM_FAR8_DT", dt)  # per-block distance table in shared memory
    V, T = synth.icosphere(3)
    M, L, eps = len(T), N + 1, 1e-6
    s = pb.cqm_frequencies(N, 2.0)
    x = synth.random_density(3, L, M)
    lsel = np.unique(np.r_[0, 1, 2, 7, 8, 63, 64, 65, 127, 128, 129, L // 2, L - 3, L - 2, L - 1])
    oh = O.H2(V, T, 48, 1.0, 4)
    oh.aca(s, eps, keep=lsel)
    tree = pb.Tree(V, T, 48, 1.0, 4)
    op = pb.Operator(tree, s, eps, mode=pb.BEM_MODE_H2ACA)
    y = _apply(pb, torch, op, x)
    yo = oh.apply(O.MODE_H2ACA, s, x[lsel], lsel)
    assert _rel(y[lsel], yo) <= 1e-10
    for i in range(len(lsel)):
        assert _rel(y[lsel[i]], yo[i]) <= 1e-8, lsel[i]


@pytest.mark.parametrize("nloc", [10, 19])
def test_local_subset_padded_columns(pb, torch, nloc):
    """A frequency shard whose size leaves 3..7 columns past a multiple of 8
    (zero-padded DMMA columns; 10 -> two leftover columns) matches the oracle."""
    V, T = synth.icosphere(3)
    N = 256
    M, L, eps = len(T), N + 1, 1e-6
    s = pb.cqm_frequencies(N, 2.0)
    rng = np.random.default_rng(nloc)
    local = np.sort(rng.choice(L, nloc, replace=False)).astype(np.int32)
    x = synth.random_density(3, nloc, M)
    oh = O.H2(V, T, 48, 1.0, 4)
    oh.aca(s, eps)
    tree = pb.Tree(V, T, 48, 1.0, 4)
    op = pb.Operator(tree, s, eps, mode=pb.BEM_MODE_H2ACA, local_l=local)
    y = _apply(pb, torch, op, x)
    yo = oh.apply(O.MODE_H2ACA, s, x, local)
    assert _rel(y, yo) <= 1e-10


def test_solve_multifreq_local_shard(pb, torch):
    """bem_solve_multifreq (the per-rank building block of the sharded solve)
    on a frequency shard: residual re-evaluated by the oracle's H2ACA apply and
    solution vs the oracle's GMRES on the same frequencies."""
    V, T = synth.icosphere(3)
    N = 32
    M, L = len(T), N + 1
    R = 10.0 ** (-5.0 / N)
    s = pb.cqm_frequencies(N, 2.0)
    local = np.array([0, 3, 4, 16, 17, 29, 30], dtype=np.int32)
    op = pb.Operator(pb.Tree(V, T, 32, 1.0, 3), s, 1e-8, local_l=local)
    g = synth.pulse(V, T, N, 2.0)
    gf = O.forward(g.astype(np.complex128), N, R)[local]
    phi, st = pb.solve_multifreq(op, torch.from_numpy(np.ascontiguousarray(gf)).cuda(), tol=1e-9, restart=20)
    phi = phi.cpu().numpy()
    assert st["n_unconverged"] == 0 and st["resid_max"] <= 1e-9
    oh = O.H2(V, T, 32, 1.0, 3)
    oh.aca(s, 1e-8)
    res = oh.apply(O.MODE_H2ACA, s, phi, local) - gf
    assert np.max(np.linalg.norm(res, axis=1) / np.linalg.norm(gf, axis=1)) <= 1.5e-9
    xo, it, rr = oh.gmres(O.MODE_H2ACA, s, gf, local, tol=1e-9, restart=20)
    assert _rel(phi, xo) <= 1e-6


@pytest.mark.parametrize("kernel,kc,m3", [("8", "0", "0"), ("8", "32", "0"), ("8", "20", "0"), ("7", "0", "0"),
                                          ("8", "0", "1"), ("8", "20", "1")])
def test_h2aca_p125(pb, torch, kernel, kc, m3, monkeypatch):
    """p = 125 (m = 5, config 5's order): far8 contracts nu in chunks
    (KC = 32 automatically, 20 forced: ragged last chunk 5), far7 whole p."""
    monkeypatch.setenv("BEM_FAR_KERNEL", kernel)
    monkeypatch.setenv("BEM_FAR8_KC", kc)
    monkeypatch.setenv("BEM_FAR8_M3", m3)
    V, T = synth.icosphere(3)
    N = 64
    M, L, eps = len(T), N + 1, 1e-8
    s = pb.cqm_frequencies(N, 2.0)
    x = synth.random_density(5, L, M)
    oh = O.H2(V, T, 64, 1.0, 5)
    oa = oh.aca(s, eps)
    tree = pb.Tree(V, T, 64, 1.0, 5)
    op = pb.Operator(tree, s, eps, mode=pb.BEM_MODE_H2ACA)
    ga = op.aca_export()
    assert np.array_equal(ga["ranks"], oa["ranks"]) and np.array_equal(ga["pivots"], oa["pivots"])
    y = _apply(pb, torch, op, x)
    lsel = np.array([0, 1, 31, 32, 33, 63, 64])
    yo = oh.apply(O.MODE_H2ACA, s, x[lsel], lsel)
    assert _rel(y[lsel], yo) <= 1e-10


def test_solve_mask_bitwise_identical(pb, torch, monkeypatch):
    """Converged frequencies skip the K1/K3 work of later GMRES iterations
    (op mask); the still-active frequencies' arithmetic is unchanged, so the
    solution and the iteration counts are bitwise identical to the unmasked solve."""
    V, T = synth.icosphere(3)
    N = 64
    R = 10.0 ** (-5.0 / N)
    s = pb.cqm_frequencies(N, 2.0)
    tree = pb.Tree(V, T, 48, 1.0, 4)
    g = torch.from_numpy(synth.pulse(V, T, N, 2.0)).cuda()
    out = []
    for m in ("1", "0"):
        monkeypatch.setenv("BEM_SOLVE_MASK", m)
        op = pb.Operator(tree, s, 1e-6)
        phi, st = pb.cqm_solve(op, g, R, tol=1e-8, restart=20)
        out.append((phi.cpu().numpy(), st))
        op.close()
    assert out[0][1]["iters_sum"] == out[1][1]["iters_sum"] and out[0][1]["n_unconverged"] == 0
    assert out[0][1]["resid_max"] == out[1][1]["resid_max"]
    assert np.array_equal(out[0][0], out[1][0])


@pytest.mark.parametrize("variant", [64, 256])
def test_hot_path_fastmath_accuracy(pb, variant):
    """Table-driven exp / sincos of K1 and K3 (fastmath.cuh) against libm over the
    configs' argument ranges: exp within 2 ulp for x in [-700, 0]; sin/cos
    within 2.5e-16 absolute for |theta| <= 6.5e3."""
    rng = np.random.default_rng(11)
    x = np.concatenate([-rng.random(200000) * 700.0, [0.0, -1e-300, -0.5 * np.log(2) / 64]])
    e, _, _ = pb.debug_fastmath(x, variant=variant)
    ref = np.exp(x)
    assert np.max(np.abs(e - ref) / np.spacing(ref)) <= 2.0
    t = np.concatenate([(rng.random(300000) - 0.5) * 13000.0, [0.0, np.pi / 64, np.pi / 2, -np.pi]])
    _, s, c = pb.debug_fastmath(t, variant=variant)
    assert np.max(np.abs(s - np.sin(t))) <= 2.5e-16
    assert np.max(np.abs(c - np.cos(t))) <= 2.5e-16


@pytest.mark.parametrize("m,leaf,N", [(3, 32, 128), (4, 48, 64), (5, 64, 32)])
def test_h2only_on_the_fly_couplings(pb, torch, m, leaf, N):
    """BEM_MODE_H2ONLY (plain H^2, couplings evaluated per frequency on the fly;
    SURVEY §8(f) NEXT-3) vs the oracle's H2ONLY on a frequency sample, p = 27/64/125."""
    V, T = synth.icosphere(3)
    M, L = len(T), N + 1
    s = pb.cqm_frequencies(N, 2.0)
    x = synth.random_density(6, L, M)
    tree = pb.Tree(V, T, leaf, 1.0, m)
    op = pb.Operator(tree, s, 1e-6, mode=pb.BEM_MODE_H2ONLY)
    y = _apply(pb, torch, op, x)
    oh = O.H2(V, T, leaf, 1.0, m)
    lsel = np.unique(np.r_[0, 1, N // 2, N // 2 + 1, N - 1, N])
    yo = oh.apply(O.MODE_H2ONLY, s, x[lsel], lsel)
    assert _rel(y[lsel], yo) <= 1e-10


# ---------------------------------------------------------------- NEXT-1: double layer
@pytest.mark.parametrize("mode", ["dense", "h2only", "h2aca"])
def test_double_layer_apply_vs_oracle(pb, torch, mode):
    """(alpha I + K(s_l)) x on a 1280-panel sphere in all three modes vs the
    oracle's identical operator (<= 1e-10 global relative l2)."""
    V, T = synth.icosphere(3)
    N = 32
    M, L, eps = len(T), N + 1, 1e-6
    s = pb.cqm_frequencies(N, 2.0)
    x = synth.random_density(7, L, M)
    leaf = 10 ** 6 if mode == "dense" else 32
    m = 1 if mode == "dense" else 3
    gm = {"dense": pb.BEM_MODE_DENSE, "h2only": pb.BEM_MODE_H2ONLY, "h2aca": pb.BEM_MODE_H2ACA}[mode]
    om = {"dense": O.MODE_DENSE, "h2only": O.MODE_H2ONLY, "h2aca": O.MODE_H2ACA}[mode]
    op = pb.Operator(pb.Tree(V, T, leaf, 1.0, m), s, eps, mode=gm)
    y = op.apply_dl(torch.from_numpy(x).cuda(), alpha=-0.5).cpu().numpy()
    oh = O.H2(V, T, leaf, 1.0, m)
    if mode == "h2aca":
        oh.aca(s, eps)
    lsel = np.array([0, 1, 7, 16, 17, 31, 32])
    yo = oh.apply_dl(om, s, x[lsel], lsel, alpha=-0.5)
    assert _rel(y[lsel], yo) <= 1e-10


def test_double_layer_p64_far8(pb, torch):
    V, T = synth.icosphere(3)
    N = 256
    M, L, eps = len(T), N + 1, 1e-6
    s = pb.cqm_frequencies(N, 2.0)
    x = synth.random_density(8, L, M)
    op = pb.Operator(pb.Tree(V, T, 48, 1.0, 4), s, eps)
    y = op.apply_dl(torch.from_numpy(x).cuda()).cpu().numpy()
    oh = O.H2(V, T, 48, 1.0, 4)
    oh.aca(s, eps)
    lsel = np.array([0, 1, 64, 128, 129, 255, 256])
    yo = oh.apply_dl(O.MODE_H2ACA, s, x[lsel], lsel)
    assert _rel(y[lsel], yo) <= 1e-10


def test_dirichlet_solve_spherical_wave(pb, torch):
    """Direct Dirichlet formulation (eq:cqmdir P:1801-1806) on the unit sphere
    with the paper's spherical wave u = f(t - |x|)/|x|, shifted
    to reach the sphere right after t = 0.  Under joint refinement of dt and h
    (Courant dt/h ~ 1): the BEM solution approaches the semi-discrete CQM
    solution (exact frequency response -(1+s) through the same transforms) at
    second order in h, and the exact trace -f'(t-1) - f(t-1) as the CQM error
    falls; the frequency-domain solution agrees with the oracle's GMRES.
    (At Courant ~0.2 the centroid-collocation V is under-resolved at the
    strongly damped frequencies |s| h >> 1 and the first-kind solve is not
    accurate there -- a property of the discretisation.)"""
    def f(z):
        return np.where(z > -0.2, np.cos(5 * z + 1) - 1, 0.0)

    def df(z):
        return np.where(z > -0.2, -5 * np.sin(5 * z + 1), 0.0)

    e_cqm, e_exact = [], []
    for sub, N in ((2, 8), (3, 16)):
        V, T = synth.icosphere(sub)
        M, L = len(T), N + 1
        Tend = 2.0
        R = 10.0 ** (-5.0 / N)
        s = pb.cqm_frequencies(N, Tend, R)
        z = np.arange(L) * Tend / N - 0.2  # f(t - |x| + shift) on |x| = 1
        g = np.ascontiguousarray(np.repeat(f(z)[:, None], M, axis=1))
        op = pb.Operator(pb.Tree(V, T, 10 ** 6, 1.0, 1), s, 1e-8, mode=pb.BEM_MODE_DENSE)
        q, st = pb.dirichlet_solve(op, torch.from_numpy(g).cuda(), R, tol=1e-10, restart=40)
        assert st["n_unconverged"] == 0
        q = q.cpu().numpy()
        gf = O.forward(g.astype(np.complex128), N, R)
        q_cqm = O.inverse(-(1 + s)[:, None] * gf, N, R).real.mean(axis=1)
        q_exact = -df(z) - f(z)
        e_cqm.append(np.linalg.norm(q.mean(axis=1) - q_cqm) / np.linalg.norm(q_cqm))
        e_exact.append(np.linalg.norm(q.mean(axis=1) - q_exact) / np.linalg.norm(q_exact))
        if sub == 2:  # vs the oracle's GMRES on the same system
            oh = O.H2(V, T, 10 ** 6, 1.0, 1)
            rhs = oh.apply_dl(O.MODE_DENSE, s, gf, alpha=-0.5)
            qo, _, _ = oh.gmres(O.MODE_DENSE, s, rhs, tol=1e-10, restart=40)
            sc = (R ** np.arange(L))[:, None]
            assert _rel(q * sc, O.inverse(qo, N, R).real * sc) <= 1e-6
    assert e_cqm[1] < 0.5 * e_cqm[0] and e_cqm[1] < 0.02, e_cqm
    assert e_exact[1] < 0.5 * e_exact[0], e_exact


@pytest.mark.parametrize("cfg", [3, 4])
def test_full_size_properties(pb, torch, cfg):
    """Configs 3 and 4 at full size in the bench's launch configuration, where
    the oracle cannot apply the whole operator in test time:
      * ACA ranks and pivots bit-identical to the oracle on a sample of far blocks;
      * linearity of the apply, and bitwise run-to-run reproducibility;
      * H2ACA vs H2ONLY (couplings exact per frequency) differ only at the
        ACA level (global relative <= 1e-8; SURVEY C10 probe ~1e-11 at eps = 1e-6);
      * real time-domain data give a real time-domain result up to that level
        (s_{L-l} = conj s_l exactly)."""
    c = synth.CONFIGS[cfg]
    V, T = synth.config_mesh(cfg)
    N = c["N"]
    M, L = len(T), N + 1
    R = 10.0 ** (-5.0 / N)
    s = pb.cqm_frequencies(N, c["T"], R)
    tree = pb.Tree(V, T, c["leaf"], c["eta"], c["m"])
    op = pb.Operator(tree, s, c["eps"])
    ga = op.aca_export()
    rng = np.random.default_rng(cfg)
    nfar = len(ga["ranks"])
    blocks = np.sort(rng.choice(nfar, 48, replace=False)).astype(np.int32)
    oh = O.H2(V, T, c["leaf"], c["eta"], c["m"])
    oa = oh.aca(s, c["eps"], blocks=blocks)
    assert np.array_equal(ga["ranks"][blocks], oa["ranks"])
    off = np.concatenate([[0], np.cumsum(ga["ranks"])])
    gp = np.concatenate([ga["pivots"][off[b]:off[b + 1]] for b in blocks])
    assert np.array_equal(gp, oa["pivots"])
    x1 = torch.from_numpy(synth.random_density(cfg, L, M, stream=1)).cuda()
    x2 = torch.from_numpy(synth.random_density(cfg, L, M, stream=2)).cuda()
    y1, y2 = op.apply(x1), op.apply(x2)
    y12 = op.apply(0.75 * x1 - 1.5j * x2)
    lin = torch.linalg.vector_norm(y12 - (0.75 * y1 - 1.5j * y2)) / torch.linalg.vector_norm(y12)
    # FP64 kernels: rounding only (1e-13); far10 rounds every coupling operand to a 48-bit
    # fixed-point number per block and drops slice levels >= 6 (~4e-13 per block product,
    # DESIGN.md §7 far10): 1e-11
    assert float(lin) <= (1e-11 if op.info()["far_kernel"] == 10 else 1e-13)
    assert torch.equal(op.apply(x1), y1)
    op2 = pb.Operator(tree, s, c["eps"], mode=pb.BEM_MODE_H2ONLY)
    yo = op2.apply(x1)
    assert float(torch.linalg.vector_norm(y1 - yo) / torch.linalg.vector_norm(yo)) <= 1e-8
    xt = torch.from_numpy(synth.random_time_data(cfg, N, M).astype(np.complex128)).cuda()
    yt = pb.cqm_inverse(op.apply(pb.cqm_forward(xt, N, R)), N, R)
    sc = torch.from_numpy(R ** np.arange(L))[:, None].cuda()
    assert float(torch.linalg.vector_norm(yt.imag * sc) / torch.linalg.vector_norm(yt.real * sc)) <= 1e-8


def test_config5_geometry_small(pb, torch):
    """Config 5's geometry and parameters at small size: two unit spheres 3
    apart, every face split 1->2 along the median (non-conforming, coplanar
    halves, AM22), m = 5 (p = 125), leaf 64, eps = 1e-8; K3 on far8 with nu
    chunks.  Pivots bit-exact and the apply within 1e-10 of the oracle."""
    V, T = synth.two_spheres(2, split=True)
    N = 32
    M, L, eps = len(T), N + 1, 1e-8
    s = pb.cqm_frequencies(N, 2.0)
    tree = pb.Tree(V, T, 64, 1.0, 5)
    op = pb.Operator(tree, s, eps)
    oh = O.H2(V, T, 64, 1.0, 5)
    oa = oh.aca(s, eps)
    ga = op.aca_export()
    assert np.array_equal(ga["ranks"], oa["ranks"]) and np.array_equal(ga["pivots"], oa["pivots"])
    x = synth.random_density(5, L, M)
    y = _apply(pb, torch, op, x)
    lsel = np.array([0, 1, 16, 17, 32])
    assert _rel(y[lsel], oh.apply(O.MODE_H2ACA, s, x[lsel], lsel)) <= 1e-10
