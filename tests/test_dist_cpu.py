"""Multi-rank host logic of the frequency-sharded path on CPU:
world_size 2 (and 3) over gloo.  The sharded time-domain operator
(DOF-sharded time data -> forward -> all-to-all -> per-rank apply of its own
frequency classes -> all-to-all -> inverse) must reproduce the single-process
result.  The transforms and the per-frequency apply are the oracle's here
(CPU test infrastructure); on GPUs the same ShardedTimeOperator drives
libbem's kernels over NCCL (bench.py --gpus N)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
import synth
from paper_2006_05186_b200.dist import ShardedSolver, ShardedTimeOperator, dof_ranges, freq_classes, shard_frequencies

N = 16
L = N + 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _problem():
    V, T = synth.icosphere(2)
    h = O.H2(V, T, 24, 1.0, 2)
    s = O.frequencies(N, 2.0)
    h.aca(s, 1e-6)
    x = synth.random_time_data(1, N, len(T)).astype(np.complex128)
    return h, s, x


def _reference(h, s, x, R):
    return O.inverse(h.apply(O.MODE_H2ACA, s, O.forward(x, N, R)), N, R)


def _worker(rank, world, port, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        h, s, x = _problem()
        R = O.default_R(N)
        M = x.shape[1]
        local = shard_frequencies(L, world)[rank]

        def apply_fn(xl):  # [L_g][M] frequency shard, panel order
            return torch.from_numpy(h.apply(O.MODE_H2ACA, s, xl.numpy(), local))

        def fwd(z):
            return torch.from_numpy(O.forward(z.numpy(), N, R))

        def inv(z):
            return torch.from_numpy(O.inverse(z.numpy(), N, R))

        top = ShardedTimeOperator(rank, world, M, L, apply_fn, fwd, inv)
        b, e = dof_ranges(M, world)[rank]
        y = top.step(torch.from_numpy(np.ascontiguousarray(x[:, b:e])))
        out_q.put((rank, b, e, y.numpy()))
    except BaseException as ex:  # report instead of leaving the parent waiting
        out_q.put((rank, -1, -1, repr(ex)))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_time_operator_matches_single_process(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    parts = [q.get(timeout=300) for _ in range(world)]
    errs = [p[3] for p in parts if p[1] < 0]
    assert not errs, errs
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    h, s, x = _problem()
    R = O.default_R(N)
    ref = _reference(h, s, x, R)
    y = np.empty_like(ref)
    for _, b, e, yp in parts:
        y[:, b:e] = yp
    sc = (R ** np.arange(L))[:, None]
    # identical arithmetic per frequency and per DOF; only the packing differs
    assert np.linalg.norm((y - ref) * sc) / np.linalg.norm(ref * sc) <= 1e-14


def test_frequency_classes_and_shards():
    """Conjugate pairs stay on one rank; shards partition 0..L-1; balanced."""
    for Lx in (33, 129, 257, 513, 1025):
        cls = freq_classes(Lx)
        assert sorted(l for c in cls for l in c) == list(range(Lx))
        for c in cls:
            assert len(c) == 1 or c[0] + c[1] == Lx
        for G in (1, 2, 4, 8):
            sh = shard_frequencies(Lx, G)
            assert sorted(np.concatenate(sh).tolist()) == list(range(Lx))
            for part in sh:
                ps = set(part.tolist())
                assert all((Lx - l) % Lx in ps for l in ps)
            sizes = [len(p) for p in sh]
            assert max(sizes) - min(sizes) <= 3
    for M in (5120, 81920, 327680):
        for G in (2, 8):
            rg = dof_ranges(M, G)
            assert rg[0][0] == 0 and rg[-1][1] == M and all(rg[i][1] == rg[i + 1][0] for i in range(G - 1))


def _solve_worker(rank, world, port, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        h, s, _ = _problem()
        V, T = synth.icosphere(2)
        R = O.default_R(N)
        M = len(T)
        g = synth.pulse(V, T, N, 2.0)
        local = shard_frequencies(L, world)[rank]

        def solve_fn(gl):  # [L_g][M] frequency shard -> (phi^, stats)
            x, it, rr = h.gmres(O.MODE_H2ACA, s, gl.numpy(), local, tol=1e-10)
            return torch.from_numpy(x), {"iters_max": int(it.max()), "iters_sum": int(it.sum()),
                                         "resid_max": float(rr.max()), "n_unconverged": int((rr > 1e-10).sum())}

        def fwd(z):
            return torch.from_numpy(O.forward(z.numpy(), N, R))

        def inv(z):
            return torch.from_numpy(O.inverse(z.numpy(), N, R))

        sol = ShardedSolver(rank, world, M, L, solve_fn, fwd, inv)
        b, e = dof_ranges(M, world)[rank]
        phi, st = sol.solve(torch.from_numpy(np.ascontiguousarray(g[:, b:e])))
        out_q.put((rank, b, e, (phi.numpy(), st)))
    except BaseException as ex:
        out_q.put((rank, -1, -1, repr(ex)))
        raise
    finally:
        dist.destroy_process_group()


def test_sharded_solve_matches_single_process():
    """Frequency-sharded decoupled solve (forward -> all-to-all -> GMRES on each
    rank's frequency classes -> all-to-all -> inverse) reproduces the
    single-process solve; global stats are reduced over ranks."""
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_solve_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    parts = [q.get(timeout=300) for _ in range(world)]
    errs = [p[3] for p in parts if p[1] < 0]
    assert not errs, errs
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    h, s, _ = _problem()
    V, T = synth.icosphere(2)
    R = O.default_R(N)
    g = synth.pulse(V, T, N, 2.0)
    xo, it, rr = h.gmres(O.MODE_H2ACA, s, O.forward(g.astype(np.complex128), N, R), tol=1e-10)
    ref = O.inverse(xo, N, R).real
    phi = np.empty_like(ref)
    for _, b, e, (pp, st) in parts:
        phi[:, b:e] = pp
        assert st["n_unconverged"] == 0 and st["iters_max"] == int(it.max()) and st["iters_sum"] == int(it.sum())
    sc = (R ** np.arange(L))[:, None]
    assert np.linalg.norm((phi - ref) * sc) / np.linalg.norm(ref * sc) <= 1e-13


def test_library_shard_map_equals_dist_py():
    """The C-ABI's frequency shard (bem_shard_frequencies, used by the NCCL transposes
    inside libbem) is the same class partition as dist.shard_frequencies."""
    from paper_2006_05186_b200 import bem as B
    for L in list(range(1, 70)) + [129, 257, 513, 1025]:
        for G in range(1, min(L // 2 + 1, 16) + 1):
            a, b = B.shard_frequencies(L, G), shard_frequencies(L, G)
            assert len(a) == len(b) and all(np.array_equal(x, y) for x, y in zip(a, b)), (L, G)
    with pytest.raises(B.BemError):
        B.shard_frequencies(5, 4)  # 3 classes only


def test_bench_gpus_n_spawns_n_ranks():
    """`python bench.py --gpus 2` (no torchrun around it) starts 2 ranks itself."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--ranks-dry-run"],
                       capture_output=True, text=True, timeout=300, cwd=root)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert sorted(d["rank"] for d in lines) == [0, 1] and all(d["world"] == 2 for d in lines)
