"""Fused transform + transpose over peer memory, exercised with
2 ranks that share this box's GPU: CUDA IPC handles map each rank's buffers
into the other, cqm_forward_rows / cqm_inverse_rows store / load frequency
rows of the other rank directly, and the ranks meet at host barriers between
the phases (no kernel waits on another rank).  The result must be bitwise
identical to the all-to-all path (host-staged gloo here, NCCL on a multi-GPU
box) and to the single-process operator."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

N = 32


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    try:
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import paper_2006_05186_b200 as pb
        import synth
        from paper_2006_05186_b200.dist import PeerTimeOperator, ShardedTimeOperator, dof_ranges, shard_frequencies
        V, T = synth.icosphere(3)
        M, L = len(T), N + 1
        R = 10.0 ** (-5.0 / N)
        s = pb.cqm_frequencies(N, 2.0, R)
        local = shard_frequencies(L, world)[rank]
        op = pb.Operator(pb.Tree(V, T, 32, 1.0, 3, device=0), s, 1e-6, local_l=local)
        b, e = dof_ranges(M, world)[rank]
        x = torch.from_numpy(np.ascontiguousarray(synth.random_time_data(3, N, M)[:, b:e].astype(np.complex128))).cuda()
        peer = PeerTimeOperator(rank, world, M, L, op, R, 0)
        y_peer = peer.step(x)
        y_peer2 = peer.step(x)  # buffers reused across steps
        a2a = ShardedTimeOperator(rank, world, M, L, op.apply, lambda z: pb.cqm_forward(z, N, R),
                                  lambda z: pb.cqm_inverse(z, N, R))
        y_a2a = a2a.step(x)
        torch.cuda.synchronize()
        peer.close()
        q.put((rank, b, e, y_peer.cpu().numpy(), y_peer2.cpu().numpy(), y_a2a.cpu().numpy(), None))
        dist.destroy_process_group()
    except BaseException as ex:  # report to the parent instead of hanging it
        q.put((rank, 0, 0, None, None, None, repr(ex)))
        raise


def test_peer_transpose_two_ranks_one_gpu():
    import torch.multiprocessing as mp
    import oracle as O
    import synth
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = [q.get(timeout=600) for _ in range(world)]
    for p in ps:
        p.join(timeout=120)
    errs = [r[6] for r in res if r[6]]
    assert not errs, errs
    V, T = synth.icosphere(3)
    M, L = len(T), N + 1
    R = 10.0 ** (-5.0 / N)
    xt = synth.random_time_data(3, N, M).astype(np.complex128)
    oh = O.H2(V, T, 32, 1.0, 3)
    s = O.frequencies(N, 2.0)
    oh.aca(s, 1e-6)
    ref = O.inverse(oh.apply(O.MODE_H2ACA, s, O.forward(xt, N, R)), N, R)
    y = np.empty_like(ref)
    for rank, b, e, yp, yp2, ya, _ in res:
        assert np.array_equal(yp, ya), rank      # fused peer transpose == all-to-all, bitwise
        assert np.array_equal(yp, yp2), rank
        y[:, b:e] = yp
    sc = (R ** np.arange(L))[:, None]
    assert np.linalg.norm((y - ref) * sc) / np.linalg.norm(ref * sc) <= 1e-10
