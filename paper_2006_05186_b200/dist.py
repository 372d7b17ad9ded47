"""Frequency sharding and the time<->frequency transpose.

* Frequency classes {0} and {j, L-j} (j = 1..) are kept whole on one rank so
  the near field (K1) shares one exp/sincos per conjugate pair; contiguous
  balanced class ranges per rank (Remark P:1607-1614: frequencies decouple).
* Time-domain data are DOF-sharded: rank g owns panels [M g/G, M (g+1)/G).
* The transpose between DOF shards [L][M_g] and frequency shards [L_g][M] is
  ONE all-to-all per direction (torch.distributed all_to_all_single: NCCL over
  NVLink on GPUs, gloo in the CPU tests).  Packing is plumbing (torch copies);
  every transform and apply runs in libbem's kernels (apply/forward/inverse
  callables passed in).
"""
from __future__ import annotations

import numpy as np


def freq_classes(L: int):
    cls = [[0]]
    for j in range(1, L // 2 + 1):
        if L - j != j:
            cls.append([j, L - j])
        else:
            cls.append([j])
    return cls


def shard_frequencies(L: int, G: int):
    """local frequency lists per rank: class i -> rank i mod G (every rank holds an even sample of
    the frequency circle, so the underflow cutoffs of K1 / K3 take the same share from every rank)."""
    cls = freq_classes(L)
    if G > len(cls):
        raise ValueError(f"{G} ranks but only {len(cls)} frequency classes")
    return [np.array([l for c in cls[g::G] for l in c], dtype=np.int32) for g in range(G)]


def dof_ranges(M: int, G: int):
    return [(M * g // G, M * (g + 1) // G) for g in range(G)]


class ShardedTimeOperator:
    """y = inverse(V forward(x)) with DOF-sharded time data on G ranks."""

    def __init__(self, rank: int, world: int, M: int, L: int, apply_fn, forward_fn, inverse_fn, group=None):
        import torch
        self.rank, self.G, self.M, self.L = rank, world, M, L
        self.local = shard_frequencies(L, world)
        self.ranges = dof_ranges(M, world)
        self.apply_fn, self.forward_fn, self.inverse_fn = apply_fn, forward_fn, inverse_fn
        self.group = group
        self._torch = torch

    def local_frequencies(self):
        return self.local[self.rank]

    def _a2a(self, send_chunks, recv_shapes, device):
        import torch.distributed as dist
        torch = self._torch
        send = torch.cat([torch.view_as_real(c.contiguous()).reshape(-1) for c in send_chunks])
        rsz = [int(np.prod(s)) * 2 for s in recv_shapes]
        ssz = [c.numel() * 2 for c in send_chunks]
        if send.is_cuda and dist.get_backend(self.group) == "gloo":  # host-staged (tests on one GPU)
            recv = torch.empty(sum(rsz), dtype=torch.float64)
            dist.all_to_all_single(recv, send.cpu(), output_split_sizes=rsz, input_split_sizes=ssz, group=self.group)
            recv = recv.to(device)
        else:
            recv = torch.empty(sum(rsz), dtype=torch.float64, device=device)
            dist.all_to_all_single(recv, send, output_split_sizes=rsz, input_split_sizes=ssz, group=self.group)
        out, o = [], 0
        for s, n in zip(recv_shapes, rsz):
            out.append(torch.view_as_complex(recv[o:o + n].view(*s, 2)))
            o += n
        return out

    def to_frequency_shard(self, xf):
        """[L][M_g] (all frequencies, this rank's DOFs) -> [L_g][M] (this rank's frequencies, all DOFs)."""
        torch = self._torch
        g = self.rank
        send = [xf.index_select(0, torch.as_tensor(self.local[h], dtype=torch.long, device=xf.device))
                for h in range(self.G)]
        Mg = [e - b for b, e in self.ranges]
        Lg = len(self.local[g])
        recv = self._a2a(send, [(Lg, Mg[h]) for h in range(self.G)], xf.device)
        return torch.cat(recv, dim=1).contiguous()

    def to_dof_shard(self, yl):
        """[L_g][M] -> [L][M_g] (inverse of to_frequency_shard)."""
        torch = self._torch
        g = self.rank
        Mg = [e - b for b, e in self.ranges]
        send = [yl[:, b:e] for (b, e) in self.ranges]
        recv = self._a2a(send, [(len(self.local[h]), Mg[g]) for h in range(self.G)], yl.device)
        yf = torch.empty((self.L, Mg[g]), dtype=yl.dtype, device=yl.device)
        for h in range(self.G):
            yf.index_copy_(0, torch.as_tensor(self.local[h], dtype=torch.long, device=yl.device), recv[h])
        return yf

    def step(self, x_loc):
        """x_loc: [L][M_g] complex (this rank's DOF shard) -> y_loc [L][M_g]."""
        xf = self.forward_fn(x_loc)  # [L][M_g]
        yl = self.apply_fn(self.to_frequency_shard(xf))
        return self.inverse_fn(self.to_dof_shard(yl))


class ShardedSolver(ShardedTimeOperator):
    """Frequency-decoupled CQM solve (Remark P:1607-1614) on G ranks:
    phi = Re inverse(V(s_l)^{-1} forward(g)) with DOF-sharded time data.
    solve_fn maps this rank's frequency shard [L_g][M] of g^ to phi^ and
    returns (phi^, stats dict); the library's bem_solve_multifreq on GPUs."""

    def __init__(self, rank, world, M, L, solve_fn, forward_fn, inverse_fn, group=None):
        super().__init__(rank, world, M, L, None, forward_fn, inverse_fn, group)
        self.solve_fn = solve_fn

    def solve(self, g_loc):
        """g_loc: [N+1][M_g] real (this rank's DOFs) -> (phi_loc [N+1][M_g] real, global stats)."""
        import torch.distributed as dist
        torch = self._torch
        gf = self.forward_fn(g_loc.to(torch.complex128))
        phil, st = self.solve_fn(self.to_frequency_shard(gf))
        phi = self.inverse_fn(self.to_dof_shard(phil))
        agg = torch.tensor([st["iters_max"], st["resid_max"], st["n_unconverged"], st["iters_sum"]],
                           dtype=torch.float64, device=g_loc.device)
        mx = agg[:2].clone()
        sm = agg[2:].clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX, group=self.group)
        dist.all_reduce(sm, op=dist.ReduceOp.SUM, group=self.group)
        stats = {"iters_max": int(mx[0]), "resid_max": float(mx[1]), "n_unconverged": int(sm[0]),
                 "iters_sum": int(sm[1])}
        return phi.real.contiguous(), stats


class PeerTimeOperator:
    """Time-domain operator y = inverse(V forward(x)) on G ranks with the
    time<->frequency transposes fused into the transforms over peer memory
    (no NCCL all-to-all): every rank exposes two device buffers through CUDA
    IPC -- its frequency shard's input [L_g][M] and the apply's output
    [L_g][M] -- and cqm_forward_rows stores frequency row l of this rank's DOF
    columns directly into the owner of l; cqm_inverse_rows reads the owners'
    output rows back.  Between the phases the ranks synchronise their devices
    and meet at a process-group barrier (no kernel waits on another rank).
    On an NVSwitch box the row stores/loads go over NVLink peer memory."""

    def __init__(self, rank: int, world: int, M: int, L: int, op, R: float, device: int, group=None):
        import torch
        import torch.distributed as dist
        from . import bem as B
        self.rank, self.G, self.M, self.L, self.R = rank, world, M, L, R
        self.N = L - 1
        self.op, self.device, self.group = op, device, group
        self._torch, self._dist, self._B = torch, dist, B
        self.local = shard_frequencies(L, world)
        self.ranges = dof_ranges(M, world)
        owner = np.empty(L, dtype=np.int64)
        slot = np.empty(L, dtype=np.int64)
        for h, fl in enumerate(self.local):
            owner[fl] = h
            slot[fl] = np.arange(len(fl))
        self.owner, self.slot = owner, slot
        nbytes = max(1, len(self.local[rank])) * M * 16
        self.xin = B.device_alloc(nbytes, device)
        self.yout = B.device_alloc(nbytes, device)
        hs = [None] * world
        dist.all_gather_object(hs, (B.ipc_handle_ptr(self.xin), B.ipc_handle_ptr(self.yout)), group=group)
        self.peer_x, self.peer_y = [], []
        for h in range(world):
            if h == rank:
                self.peer_x.append(self.xin)
                self.peer_y.append(self.yout)
            else:
                self.peer_x.append(B.ipc_open(hs[h][0], device))
                self.peer_y.append(B.ipc_open(hs[h][1], device))
        b = self.ranges[rank][0]
        self.out_rows = [self.peer_x[owner[l]] + int((slot[l] * M + b) * 16) for l in range(L)]
        self.in_rows = [self.peer_y[owner[l]] + int((slot[l] * M + b) * 16) for l in range(L)]

    def _fence(self):
        self._torch.cuda.synchronize(self.device)
        self._dist.barrier(group=self.group)

    def step(self, x_loc):
        """x_loc: [N+1][M_g] complex (this rank's DOFs) -> y_loc [N+1][M_g]."""
        B = self._B
        B.cqm_forward_rows(x_loc, self.N, self.R, self.out_rows)
        self._fence()  # every rank's rows have landed in the owners' input buffers
        self.op.apply_raw(self.xin, self.yout)
        self._fence()  # every owner's output is complete
        y = B.cqm_inverse_rows(self.in_rows, self.N, self.R, x_loc.shape[1], device=x_loc.device)
        self._fence()  # peers finished reading our output before it is overwritten
        return y

    def close(self):
        B = self._B
        for h in range(self.G):
            if h != self.rank:
                B.ipc_close(self.peer_x[h])
                B.ipc_close(self.peer_y[h])
        B.device_free(self.xin)
        B.device_free(self.yout)
