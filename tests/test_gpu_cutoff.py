"""Underflow cutoffs of K1 and K3 (include/bem.h bem_op_get_work).

|e^{-s r}| = e^{-Re s r} (eq:fundsol P:479-482): at the strongly damped CQM frequencies the
kernel underflows beyond a few mesh widths, so K1 leaves out a frequency class over a warp step
of sources when Re s r_min > 42 and far10 leaves out a (far block, 128-frequency tile) whose
compressed fibres (eq:maca P:1314-1320) are bounded by 2^-70 / max(|s_t|, 1).  Both must be
invisible at the parity bar: the apply with the cutoffs agrees with the apply without them to
rounding (every frequency on its own, the most damped ones included), still meets the oracle
bar, and the work counters show that something was in fact left out."""
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


@pytest.mark.parametrize("sub,m,leaf,N,eps,skel", [
    (4, 3, 32, 128, 1e-6, "z"),        # p = 27, one frequency tile + leftover column: K1 cutoff only
    (4, 3, 32, 512, 1e-6, "z"),        # four tiles (config 4's L): tiles 1 and 2 hold the damped half circle
    (3, 4, 48, 512, 1e-7, "factors"),  # p = 64, the mask recomputed per regenerated tile
])
def test_cutoffs_invisible(pb, torch, sub, m, leaf, N, eps, skel, monkeypatch):
    V, T = synth.icosphere(sub)  # 5120 / 1280 panels; Re s up to 4 N / T
    M, L = len(T), N + 1
    s = pb.cqm_frequencies(N, 2.0)
    x = synth.random_density(12, L, M)
    tree = pb.Tree(V, T, leaf, 1.0, m)
    mode = pb.BEM_MODE_H2ACA | (pb.BEM_SKEL_FACTORS if skel == "factors" else pb.BEM_SKEL_Z)
    monkeypatch.setenv("BEM_FAR_KERNEL", "10")
    op = pb.Operator(tree, s, eps, mode=mode)
    op.set_profiling(True)
    y = _apply(torch, op, x)
    w = op.work()
    op.set_profiling(False)
    assert np.array_equal(_apply(torch, op, x), y)  # deterministic, profiling does not change the result
    assert w["near_tau"] == 42.0 and w["far_delta"] == 2.0 ** -70
    assert 0 < w["near_evals_run"] < w["near_evals_total"]
    assert 0 < w["far_rank_cols_run"] <= w["far_rank_cols_total"]
    if N >= 512:
        assert w["far_rank_cols_run"] < w["far_rank_cols_total"]
    monkeypatch.setenv("BEM_NEAR_TAU", "0")
    monkeypatch.setenv("BEM_FAR_SKIP_LOG2", "0")
    op0 = pb.Operator(tree, s, eps, mode=mode)
    op0.set_profiling(True)
    y0 = _apply(torch, op0, x)
    w0 = op0.work()
    assert w0["near_evals_run"] == w0["near_evals_total"] == w["near_evals_total"]
    assert w0["far_rank_cols_run"] == w0["far_rank_cols_total"] == w["far_rank_cols_total"]
    assert w0["far_delta"] == 0.0 and w0["near_tau"] == 0.0
    assert _rel(y, y0) <= 1e-14
    for l in range(L):  # every frequency on its own: the damped ones are the ones that lose work
        assert _rel(y[l], y0[l]) <= 1e-13, l
    lsel = np.unique(np.r_[0, 1, L // 4, L // 2 - 1, L // 2, L // 2 + 1, 3 * L // 4, L - 1])
    oh = O.H2(V, T, leaf, 1.0, m)
    oh.aca(s, eps, keep=lsel)
    yo = oh.apply(O.MODE_H2ACA, s, x[lsel], lsel)
    assert _rel(y[lsel], yo) <= 1e-10
    for i in range(len(lsel)):
        assert _rel(y[lsel[i]], yo[i]) <= 1e-10, lsel[i]


def test_cutoff_dense_mode(pb, torch, monkeypatch):
    """Dense mode (config 1's path: K1 over every panel pair) against the oracle's dense operator."""
    V, T = synth.icosphere(2)
    N = 64
    M, L = len(T), N + 1
    s = pb.cqm_frequencies(N, 2.0)
    x = synth.random_density(13, L, M)
    tree = pb.Tree(V, T, 32, 1.0, 3)
    op = pb.Operator(tree, s, 1e-6, mode=pb.BEM_MODE_DENSE)
    op.set_profiling(True)
    y = _apply(torch, op, x)
    w = op.work()
    assert 0 < w["near_evals_run"] < w["near_evals_total"]
    for l in (0, 1, L // 2, L - 1):
        yo = O.dense_matrix(V, T, s[l]) @ x[l]
        assert _rel(y[l], yo) <= 1e-10, l


def test_cutoff_h2only(pb, torch, monkeypatch):
    """Plain-H^2 couplings (NEXT-3, K3'): a far block is left out for a class tile with
    min Re s * r_lb > tau + 8 (r_lb = distance of the node boxes); on vs off and the oracle's
    plain-H^2 apply."""
    V, T = synth.icosphere(4)
    N, m, leaf = 512, 3, 32
    M, L = len(T), N + 1
    s = pb.cqm_frequencies(N, 2.0)
    x = synth.random_density(14, L, M)
    tree = pb.Tree(V, T, leaf, 1.0, m)
    op = pb.Operator(tree, s, 1e-6, mode=pb.BEM_MODE_H2ONLY)
    y = _apply(torch, op, x)
    monkeypatch.setenv("BEM_NEAR_TAU", "0")
    op0 = pb.Operator(tree, s, 1e-6, mode=pb.BEM_MODE_H2ONLY)
    y0 = _apply(torch, op0, x)
    assert _rel(y, y0) <= 1e-14
    for l in range(L):
        assert _rel(y[l], y0[l]) <= 1e-13, l
    lsel = np.unique(np.r_[0, 1, L // 4, L // 2, L // 2 + 1, L - 1])
    oh = O.H2(V, T, leaf, 1.0, m)
    yo = oh.apply(O.MODE_H2ONLY, s, x[lsel], lsel)
    assert _rel(y[lsel], yo) <= 1e-10
    for i in range(len(lsel)):
        assert _rel(y[lsel[i]], yo[i]) <= 1e-10, lsel[i]
