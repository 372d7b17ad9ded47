"""K3 on the INT8 tensor cores (far10, csrc/farq.cu): the MACA coupling step with
its complex FP64 products emulated exactly by six-byte fixed-point slices on
tcgen05.mma kind::i8.  It must meet the same bar as the FP64 kernels against the
oracle's identical-compression apply (<= 1e-10 global relative l2,
<= 1e-8 per frequency), agree with far8 to the emulation's precision, be
deterministic, and give bitwise the same result from the stored and the
factors-only skeleton (their Z coefficients are bitwise equal)."""
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


@pytest.mark.parametrize("m,leaf,N,eps", [
    (3, 32, 128, 1e-6),   # p = 27 (config 2's order): one mu chunk of 27 rows, leftover l = 0
    (4, 48, 256, 1e-6),   # p = 64: two frequency tiles + leftover column, two mu chunks
    (4, 48, 260, 1e-6),   # L mod 128 = 5: no leftover, ragged third tile (5 columns)
    (5, 64, 64, 1e-8),    # p = 125: ragged fourth mu chunk (29 rows), ragged last nu chunk
])
def test_far10_vs_oracle_and_far8(pb, torch, m, leaf, N, eps, monkeypatch):
    V, T = synth.icosphere(3)
    M, L = len(T), N + 1
    s = pb.cqm_frequencies(N, 2.0)
    x = synth.random_density(11, L, M)
    tree = pb.Tree(V, T, leaf, 1.0, m)
    monkeypatch.setenv("BEM_FAR_KERNEL", "10")
    op10 = pb.Operator(tree, s, eps, mode=pb.BEM_MODE_H2ACA)
    y10 = _apply(torch, op10, x)
    assert np.array_equal(_apply(torch, op10, x), y10)  # deterministic
    monkeypatch.setenv("BEM_FAR_KERNEL", "8" if m > 3 else "7")
    op8 = pb.Operator(tree, s, eps, mode=pb.BEM_MODE_H2ACA)
    y8 = _apply(torch, op8, x)
    assert _rel(y10, y8) <= 1e-11
    lsel = np.unique(np.r_[0, 1, 2, 63, 64, 127, 128, 129, L // 2, L - 2, L - 1])
    lsel = lsel[lsel < L]
    oh = O.H2(V, T, leaf, 1.0, m)
    oh.aca(s, eps, keep=lsel)
    yo = oh.apply(O.MODE_H2ACA, s, x[lsel], lsel)
    assert _rel(y10[lsel], yo) <= 1e-10
    for i in range(len(lsel)):
        assert _rel(y10[lsel[i]], yo[i]) <= 1e-8, lsel[i]


def test_far10_factors_vs_stored_bitwise(pb, torch, monkeypatch):
    monkeypatch.setenv("BEM_FAR_KERNEL", "10")
    V, T = synth.icosphere(3)
    N = 256
    M, L = len(T), N + 1
    s = pb.cqm_frequencies(N, 2.0)
    tree = pb.Tree(V, T, 48, 1.0, 4)
    opz = pb.Operator(tree, s, 1e-6, mode=pb.BEM_MODE_H2ACA | pb.BEM_SKEL_Z)
    opf = pb.Operator(tree, s, 1e-6, mode=pb.BEM_MODE_H2ACA | pb.BEM_SKEL_FACTORS)
    x = torch.from_numpy(synth.random_density(12, L, M)).cuda()
    assert torch.equal(opz.apply(x), opf.apply(x))


@pytest.mark.parametrize("nloc", [10, 19, 130])
def test_far10_frequency_shard(pb, torch, nloc, monkeypatch):
    """A frequency shard (bench --shard-of / multi-GPU rank): one partial tile, or a
    tile plus two leftover columns (130 = 128 + 2)."""
    monkeypatch.setenv("BEM_FAR_KERNEL", "10")
    V, T = synth.icosphere(3)
    N = 256
    M, L, eps = len(T), N + 1, 1e-6
    s = pb.cqm_frequencies(N, 2.0)
    rng = np.random.default_rng(nloc)
    local = np.sort(rng.choice(L, nloc, replace=False)).astype(np.int32)
    x = synth.random_density(3, nloc, M)
    oh = O.H2(V, T, 48, 1.0, 4)
    oh.aca(s, eps, keep=local)
    op = pb.Operator(pb.Tree(V, T, 48, 1.0, 4), s, eps, mode=pb.BEM_MODE_H2ACA, local_l=local)
    y = _apply(torch, op, x)
    yo = oh.apply(O.MODE_H2ACA, s, x, local)
    assert _rel(y, yo) <= 1e-10


def test_far10_term_groups(pb, torch, monkeypatch):
    """Blocks longer than gmax ACA terms are read out in groups (the int32 level sums stay
    exact); forcing groups of 3 terms changes only the FP64 summation order."""
    V, T = synth.icosphere(3)
    N = 256
    M, L = len(T), N + 1
    s = pb.cqm_frequencies(N, 2.0)
    tree = pb.Tree(V, T, 48, 1.0, 4)
    x = synth.random_density(13, L, M)
    monkeypatch.setenv("BEM_FAR_KERNEL", "10")
    y = _apply(torch, pb.Operator(tree, s, 1e-6, mode=pb.BEM_MODE_H2ACA), x)
    monkeypatch.setenv("BEM_FAR10_GMAX", "3")
    yg = _apply(torch, pb.Operator(tree, s, 1e-6, mode=pb.BEM_MODE_H2ACA), x)
    assert _rel(yg, y) <= 1e-13
    lsel = np.array([0, 1, 128, 256])
    oh = O.H2(V, T, 48, 1.0, 4)
    oh.aca(s, 1e-6, keep=lsel)
    assert _rel(yg[lsel], oh.apply(O.MODE_H2ACA, s, x[lsel], lsel)) <= 1e-10


def test_far10_fused_near_field(pb, torch, monkeypatch):
    """K1 fused into the far10 launch (near-field warps beside the coupling work + a tail
    kernel for the items they leave; the default where far10 runs with 4-class tiles) gives
    the same near field as the standalone K1 kernel -- the same per-item code, so bitwise --
    and the same operator as the oracle. Also through the graph-replayed time step."""
    V, T = synth.icosphere(3)
    N = 256  # 129 classes -> 4-class tiles
    M, L = len(T), N + 1
    s = pb.cqm_frequencies(N, 2.0)
    tree = pb.Tree(V, T, 48, 1.0, 4)
    x = synth.random_density(17, L, M)
    monkeypatch.setenv("BEM_FAR_KERNEL", "10")
    opf = pb.Operator(tree, s, 1e-6, mode=pb.BEM_MODE_H2ACA)
    yf = _apply(torch, opf, x)
    monkeypatch.setenv("BEM_K1_FUSE", "0")
    ops = pb.Operator(tree, s, 1e-6, mode=pb.BEM_MODE_H2ACA)
    ys = _apply(torch, ops, x)
    assert np.array_equal(yf, ys)
    lsel = np.array([0, 1, 128, 256])
    oh = O.H2(V, T, 48, 1.0, 4)
    oh.aca(s, 1e-6, keep=lsel)
    assert _rel(yf[lsel], oh.apply(O.MODE_H2ACA, s, x[lsel], lsel)) <= 1e-10
    R = 10.0 ** (-5.0 / N)
    xt = torch.from_numpy(synth.random_time_data(5, N, M).astype(np.complex128)).cuda()
    yt_f = opf.time_step(xt, R)
    yt_s = ops.time_step(xt, R)
    torch.cuda.synchronize()
    assert torch.equal(yt_f, yt_s)
