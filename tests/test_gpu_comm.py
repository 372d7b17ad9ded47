"""The NCCL frequency-sharded path of the C-ABI on the one GPU a
test box has: a 1-rank communicator exercises the whole code path --
bem_comm_init, the shard map, K4 fused with the all-to-all packing (row table in
the kernel parameters), grouped ncclSend/ncclRecv, the strided 2-D copies, the
apply of the rank's frequency list, and the reverse direction -- and the
sharded cqm_solve with its NCCL reductions of the statistics.  Results must
equal the single-device calls (bem_time_step / cqm_solve without a communicator).
The multi-rank host logic is covered by tests/test_dist_cpu.py (gloo, world 2/3)."""
import numpy as np
import pytest

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


@pytest.fixture(scope="module")
def comm(pb, torch):
    from paper_2006_05186_b200 import bem as B
    c = B.Comm(0, 1, 0)
    yield c
    c.close()


def _rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


@pytest.mark.parametrize("m,leaf,N", [(3, 32, 32), (4, 48, 64)])
def test_sharded_step_one_rank_equals_time_step(pb, torch, comm, m, leaf, N):
    from paper_2006_05186_b200 import bem as B
    V, T = synth.icosphere(3)
    M, L = len(T), N + 1
    R = 10.0 ** (-5.0 / N)
    s = pb.cqm_frequencies(N, 2.0)
    tree = pb.Tree(V, T, leaf, 1.0, m)
    local = B.shard_frequencies(L, 1)[0]
    assert sorted(local.tolist()) == list(range(L)) and local[1] == 1 and local[2] == L - 1  # class order
    ops = pb.Operator(tree, s, 1e-6, local_l=local)
    opf = pb.Operator(tree, s, 1e-6)
    x = torch.from_numpy(synth.random_time_data(2, N, M).astype(np.complex128)).cuda()
    ys = B.time_step_sharded(ops, x, R, comm)
    yf = opf.time_step(x, R)
    torch.cuda.synchronize()
    sc = (R ** np.arange(L))[:, None]
    assert _rel(ys.cpu().numpy() * sc, yf.cpu().numpy() * sc) <= 1e-13
    assert torch.equal(B.time_step_sharded(ops, x, R, comm), ys)  # reproducible
    with pytest.raises(pb.BemError) as e:  # op not holding the rank's shard
        B.time_step_sharded(opf, x, R, comm)
    assert e.value.code == -1
    with pytest.raises(pb.BemError):  # wrong DOF count for this rank
        B.time_step_sharded(ops, x[:, :M - 1].contiguous(), R, comm)


def test_sharded_solve_one_rank_equals_solve(pb, torch, comm):
    from paper_2006_05186_b200 import bem as B
    V, T = synth.icosphere(3)
    N = 16
    M, L = len(T), N + 1
    R = 10.0 ** (-5.0 / N)
    s = pb.cqm_frequencies(N, 2.0)
    tree = pb.Tree(V, T, 32, 1.0, 3)
    g = torch.from_numpy(synth.pulse(V, T, N, 2.0)).cuda()
    ops = pb.Operator(tree, s, 1e-8, local_l=B.shard_frequencies(L, 1)[0])
    opf = pb.Operator(tree, s, 1e-8)
    phs, sts = pb.cqm_solve(ops, g, R, tol=1e-8, restart=30, comm=comm)
    phf, stf = pb.cqm_solve(opf, g, R, tol=1e-8, restart=30)
    assert sts["n_unconverged"] == 0 and sts["iters_sum"] == stf["iters_sum"]
    assert sts["iters_max"] == stf["iters_max"] and sts["resid_max"] <= 1e-8
    sc = (R ** np.arange(L))[:, None]
    assert _rel(phs.cpu().numpy() * sc, phf.cpu().numpy() * sc) <= 1e-12


@pytest.mark.parametrize("G,m,leaf,N", [(2, 3, 32, 32), (3, 4, 48, 64), (5, 3, 32, 16)])
def test_virtual_ranks_sharded_step_equals_time_step(pb, torch, G, m, leaf, N):
    """G ranks in one process (bem_debug_sharded_step): the NCCL path's packing and unpacking
    code with the all-to-all replaced by device copies, so the G > 1 transposes -- ragged DOF
    ranges (M = 1280 over 3 and 5 ranks), uneven frequency shards, the conjugate-pair
    classes -- are checked against the single-device step on the one GPU a box has."""
    from paper_2006_05186_b200 import bem as B
    V, T = synth.icosphere(3)
    M, L = len(T), N + 1
    R = 10.0 ** (-5.0 / N)
    s = pb.cqm_frequencies(N, 2.0)
    tree = pb.Tree(V, T, leaf, 1.0, m)
    lists = B.shard_frequencies(L, G)
    assert sorted(np.concatenate(lists).tolist()) == list(range(L))
    ops = [pb.Operator(tree, s, 1e-6, local_l=lists[g]) for g in range(G)]
    opf = pb.Operator(tree, s, 1e-6)
    x = torch.from_numpy(synth.random_time_data(3, N, M).astype(np.complex128)).cuda()
    rng = [B.dof_range(M, G, g) for g in range(G)]
    xs = [x[:, b:e].contiguous() for b, e in rng]
    ys = B.debug_sharded_step(ops, xs, R)
    yf = opf.time_step(x, R)
    torch.cuda.synchronize()
    y = torch.cat(ys, dim=1).cpu().numpy()
    sc = (R ** np.arange(L))[:, None]
    assert _rel(y * sc, yf.cpu().numpy() * sc) <= 1e-13
    assert all(torch.equal(a, b) for a, b in zip(B.debug_sharded_step(ops, xs, R), ys))
