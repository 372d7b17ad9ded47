"""Thin ctypes binding of libbem.so (include/bem.h): argument marshalling only.

Every step of the hot path runs in the library's CUDA kernels; torch is used
for device memory and streams.  There is no CPU fallback: if libbem.so is
missing or fails to load, every call raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("BEM_LIB_PATH") or os.path.join(HERE, "libbem.so")  # override: A/B builds (tools)

BEM_MODE_H2ACA, BEM_MODE_H2ONLY, BEM_MODE_DENSE, BEM_MODE_COMBINED = 0, 1, 2, 3
BEM_SKEL_Z, BEM_SKEL_FACTORS = 0x100, 0x200  # skeleton storage flags OR-ed into mode (include/bem.h)
BEM_ENOCONV = -5
_lib = None


class BemError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"bem error {code}: {msg}")
        self.code = code


class TreeStats(C.Structure):
    _fields_ = [("M", C.c_int64), ("clusters", C.c_int64), ("leaves", C.c_int64), ("near_blocks", C.c_int64),
                ("far_blocks", C.c_int64), ("nnz_near", C.c_int64), ("depth", C.c_int32), ("p", C.c_int32)]


class OpInfo(C.Structure):
    _fields_ = [("mode", C.c_int32), ("skeleton", C.c_int32), ("n_local", C.c_int32), ("rmax", C.c_int32),
                ("total_rank", C.c_int64), ("z_bytes", C.c_int64), ("f_bytes", C.c_int64),
                ("device_bytes", C.c_int64), ("far_kernel", C.c_int32), ("reserved_", C.c_int32)]


class OpWork(C.Structure):
    _fields_ = [("far_rank_cols_total", C.c_int64), ("far_rank_cols_run", C.c_int64),
                ("near_evals_total", C.c_int64), ("near_evals_run", C.c_int64),
                ("near_tau", C.c_double), ("far_delta", C.c_double)]


class SolveStats(C.Structure):
    _fields_ = [("iters_max", C.c_int32), ("iters_sum", C.c_int32), ("n_unconverged", C.c_int32),
                ("pad_", C.c_int32), ("resid_max", C.c_double), ("imag_rel_max", C.c_double)]


EXPORTS = [
    "bem_last_error", "cqm_frequencies", "bem_build_tree", "bem_tree_get_stats", "bem_tree_export",
    "bem_tree_destroy", "bem_assemble_h2_aca", "bem_aca_export", "bem_aca_export_near", "bem_mot_prepare", "bem_conv_time", "cqm_mot_solve", "bem_time_step", "bem_op_destroy", "bem_apply_multifreq", "bem_apply_double_layer",
    "cqm_forward", "cqm_inverse", "cqm_forward_rows", "cqm_inverse_rows", "bem_ipc_get_handle",
    "bem_ipc_open_handle", "bem_ipc_close", "bem_device_alloc", "bem_device_free", "cqm_solve", "bem_solve_multifreq", "bem_debug_pinned", "bem_debug_fastmath", "bem_debug_fp64_peak",
    "bem_op_set_profiling", "bem_op_get_timings", "bem_op_launch_count", "bem_debug_fp64_peak_ex",
    "bem_op_get_info", "bem_comm_unique_id", "bem_comm_init", "bem_comm_destroy", "bem_shard_frequencies",
    "bem_time_step_sharded", "bem_debug_aca_blocks", "bem_debug_sharded_step", "bem_debug_i8_gemm",
    "bem_debug_i8_rate", "bem_debug_i8_gemm_pair", "bem_op_get_work",
]


def lib():
    """Load libbem.so (fails loudly when it is missing: no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
    L = C.CDLL(LIB_PATH)
    vp, i32, i64, d = C.c_void_p, C.c_int32, C.c_int64, C.c_double
    L.bem_last_error.restype = C.c_char_p
    sig = {
        "cqm_frequencies": [i32, d, d, i32, vp],
        "bem_build_tree": [vp, i64, vp, i64, i32, d, i32, i32, vp],
        "bem_tree_get_stats": [vp, vp],
        "bem_tree_export": [vp, vp, vp, vp, vp, vp],
        "bem_tree_destroy": [vp],
        "bem_assemble_h2_aca": [vp, vp, i32, vp, i32, d, i32, vp, vp],
        "bem_aca_export": [vp, vp, vp, vp],
        "bem_aca_export_near": [vp, vp, vp, vp],
        "bem_mot_prepare": [vp, d, vp],
        "bem_time_step": [vp, vp, vp, d, vp],
        "bem_conv_time": [vp, vp, vp, i32, vp],
        "cqm_mot_solve": [vp, vp, vp, d, i32, i32, vp, vp],
        "bem_op_destroy": [vp],
        "bem_apply_multifreq": [vp, vp, vp, vp],
        "bem_apply_double_layer": [vp, vp, vp, d, vp],
        "cqm_forward": [vp, vp, i64, i32, d, vp],
        "cqm_inverse": [vp, vp, i64, i32, d, vp],
        "cqm_solve": [vp, vp, vp, i64, d, d, i32, i32, vp, vp, vp],
        "cqm_forward_rows": [vp, i64, vp, i32, d, vp],
        "cqm_inverse_rows": [vp, vp, i64, i32, d, vp],
        "bem_ipc_get_handle": [vp, vp],
        "bem_ipc_open_handle": [vp, i32, vp],
        "bem_ipc_close": [vp],
        "bem_device_alloc": [i64, i32, vp],
        "bem_device_free": [vp],
        "bem_solve_multifreq": [vp, vp, vp, d, i32, i32, vp, vp],
        "bem_debug_pinned": [vp, i64, vp, vp, vp, i32],
        "bem_debug_fastmath": [vp, i64, vp, vp, vp, i32, i32],
        "bem_debug_fp64_peak": [i32, vp, vp],
        "bem_op_set_profiling": [vp, i32],
        "bem_op_get_timings": [vp, vp],
        "bem_op_launch_count": [vp, vp],
        "bem_debug_fp64_peak_ex": [i32, vp, i32, vp],
        "bem_op_get_info": [vp, vp],
        "bem_op_get_work": [vp, vp],
        "bem_comm_unique_id": [vp],
        "bem_comm_init": [vp, i32, i32, i32, vp],
        "bem_comm_destroy": [vp],
        "bem_shard_frequencies": [i32, i32, vp, vp],
        "bem_time_step_sharded": [vp, vp, vp, i64, d, vp, vp],
        "bem_debug_aca_blocks": [vp, vp, i32, d, vp, i32, vp, vp, vp],
        "bem_debug_sharded_step": [i32, vp, vp, vp, d, vp],
        "bem_debug_i8_gemm": [vp, vp, vp, i32, i32, i32, i32],
        "bem_debug_i8_rate": [i32, i32, i32, i32, vp, vp],
        "bem_debug_i8_gemm_pair": [vp, vp, vp, i32, i32, i32],
    }
    for name, args in sig.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = C.c_int32
    _lib = L
    return L


def _check(code):
    if code != 0:
        raise BemError(code, lib().bem_last_error().decode())


def _p(a):
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        return a.ctypes.data_as(C.c_void_p)
    return C.c_void_p(a.data_ptr())  # torch tensor


def _stream(stream):
    if stream is None:
        import torch
        if not torch.cuda.is_available():
            return C.c_void_p(0)  # the library reports the missing device itself
        return C.c_void_p(torch.cuda.current_stream().cuda_stream)
    if isinstance(stream, int):
        return C.c_void_p(stream)
    return C.c_void_p(stream.cuda_stream)


def cqm_frequencies(N: int, T: float, R: float | None = None, method: int = 2) -> np.ndarray:
    """s_l, l < L = N+1 (eq:cqm_freq P:443-447); R defaults to 10^{-5/N}."""
    R = 10.0 ** (-5.0 / N) if (R is None and N >= 1) else (R if R is not None else 0.5)
    out = np.empty(max(N, 0) + 1, dtype=np.complex128)
    _check(lib().cqm_frequencies(int(N), float(T), float(R), int(method), _p(out)))
    return out


class Tree:
    """bem_build_tree handle (cluster tree, partition, bases on one device)."""

    def __init__(self, V, T, leaf_size: int, eta: float, m: int, device: int = 0):
        V = np.ascontiguousarray(V, dtype=np.float64)
        T = np.ascontiguousarray(T, dtype=np.int32)
        h = C.c_void_p()
        _check(lib().bem_build_tree(_p(V), len(V), _p(T), len(T), int(leaf_size), float(eta), int(m), int(device),
                                    C.byref(h)))
        self.h = h
        self.device = device
        st = TreeStats()
        _check(lib().bem_tree_get_stats(self.h, C.byref(st)))
        self.stats = {k: int(getattr(st, k)) for k, _ in TreeStats._fields_}
        self.M = self.stats["M"]
        self.p = self.stats["p"]

    def export(self):
        s = self.stats
        perm = np.empty(s["M"], dtype=np.int32)
        clusters = np.empty((s["clusters"], 5), dtype=np.int32)
        boxes = np.empty((s["clusters"], 6))
        near = np.empty((s["near_blocks"], 2), dtype=np.int32)
        far = np.empty((s["far_blocks"], 2), dtype=np.int32)
        _check(lib().bem_tree_export(self.h, _p(perm), _p(clusters), _p(boxes), _p(near), _p(far)))
        return dict(perm=perm, clusters=clusters, boxes=boxes, near=near, far=far)

    def close(self):
        if getattr(self, "h", None):
            _check(lib().bem_tree_destroy(self.h))
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Operator:
    """bem_assemble_h2_aca handle: y_t = V(s_{local_l[t]}) x_t."""

    def __init__(self, tree: Tree, s, eps: float, mode: int = BEM_MODE_H2ACA, local_l=None, stream=None):
        s = np.ascontiguousarray(s, dtype=np.complex128)
        self.L = len(s)
        self.s = s
        self.tree = tree
        if local_l is None:
            loc, nloc = None, self.L
            self.local_l = np.arange(self.L, dtype=np.int32)
        else:
            loc = np.ascontiguousarray(local_l, dtype=np.int32)
            nloc = len(loc)
            self.local_l = loc
        self.n_local = nloc
        self.mode = mode
        h = C.c_void_p()
        _check(lib().bem_assemble_h2_aca(tree.h, _p(s), self.L, _p(loc), nloc, float(eps), int(mode),
                                         _stream(stream), C.byref(h)))
        self.h = h

    def aca_export(self):
        nfar = self.tree.stats["far_blocks"]
        ranks = np.empty(nfar, dtype=np.int32)
        tot = C.c_int64()
        _check(lib().bem_aca_export(self.h, _p(ranks), None, C.byref(tot)))
        piv = np.empty((tot.value, 2), dtype=np.int32)
        _check(lib().bem_aca_export(self.h, None, _p(piv), None))
        return dict(ranks=ranks, pivots=piv)

    def info(self):
        """Skeleton storage and the op's device footprint (bem_op_get_info)."""
        st = OpInfo()
        _check(lib().bem_op_get_info(self.h, C.byref(st)))
        return {k: int(getattr(st, k)) for k, _ in OpInfo._fields_}

    def skeleton(self) -> str:
        return {0: "none", 1: "Z", 2: "factors"}[self.info()["skeleton"]]

    def aca_export_near(self):
        """Near-block skeletons of a BEM_MODE_COMBINED operator (Alg. 3 NEAR branch)."""
        nn = self.tree.stats["near_blocks"]
        ranks = np.empty(nn, dtype=np.int32)
        tot = C.c_int64()
        _check(lib().bem_aca_export_near(self.h, _p(ranks), None, C.byref(tot)))
        piv = np.empty((tot.value, 2), dtype=np.int32)
        _check(lib().bem_aca_export_near(self.h, None, _p(piv), None))
        return dict(ranks=ranks, pivots=piv)

    def time_step(self, x_time, R: float, y=None, stream=None):
        """y = cqm_inverse(V(s_l) cqm_forward(x_time)) in one library call (graph-replayed device
        part); x_time: [L][M] complex128 torch tensor on the host (pinned for async) or device."""
        import torch
        assert x_time.dtype == torch.complex128 and x_time.is_contiguous()
        assert tuple(x_time.shape) == (self.L, self.tree.M), "x_time must be [L][M]"
        y = torch.empty_like(x_time, pin_memory=not x_time.is_cuda) if y is None else y
        assert y.dtype == torch.complex128 and y.is_contiguous() and tuple(y.shape) == tuple(x_time.shape)
        assert (y.is_cuda == x_time.is_cuda) and (not y.is_cuda or y.device == x_time.device)
        _check(lib().bem_time_step(self.h, _p(x_time), _p(y), float(R), _stream(stream)))
        return y

    def mot_prepare(self, R: float, stream=None):
        """Time-domain weights of the compressed tensor (eq:fastdft; BEM_MODE_COMBINED, all L)."""
        _check(lib().bem_mot_prepare(self.h, float(R), _stream(stream)))

    def conv_time(self, q, kmax: int | None = None, stream=None):
        """y_n = sum_{k <= min(n, kmax)} V^_{n-k} q_k (eq:fastrhs); q device [L][M] complex."""
        import torch
        assert q.dtype == torch.complex128 and q.is_cuda and q.is_contiguous()
        y = torch.empty_like(q)
        _check(lib().bem_conv_time(self.h, _p(q), _p(y), int(q.shape[0] - 1 if kmax is None else kmax),
                                   _stream(stream)))
        return y

    def apply(self, x, y=None, stream=None):
        """x, y: torch complex128 [n_local][M] on the tree's device (input panel order)."""
        import torch
        assert x.dtype == torch.complex128 and x.is_cuda and x.is_contiguous()
        assert tuple(x.shape) == (self.n_local, self.tree.M)
        if y is None:
            y = torch.empty_like(x)
        assert y.dtype == torch.complex128 and y.is_contiguous() and y.shape == x.shape and y.device == x.device
        _check(lib().bem_apply_multifreq(self.h, _p(x), _p(y), _stream(stream)))
        return y

    def apply_raw(self, x_ptr: int, y_ptr: int, stream=None):
        """y = V x on raw device addresses ([n_local][M] complex each), e.g. IPC-shared buffers."""
        _check(lib().bem_apply_multifreq(self.h, C.c_void_p(x_ptr), C.c_void_p(y_ptr), _stream(stream)))

    def apply_dl(self, x, alpha: float = 0.0, y=None, stream=None):
        """y_t = (alpha I + K(s_{local_l[t]})) x_t (double layer, NEXT-1)."""
        import torch
        assert x.dtype == torch.complex128 and x.is_cuda and x.is_contiguous()
        assert tuple(x.shape) == (self.n_local, self.tree.M)
        if y is None:
            y = torch.empty_like(x)
        assert y.dtype == torch.complex128 and y.is_contiguous() and y.shape == x.shape and y.device == x.device
        _check(lib().bem_apply_double_layer(self.h, _p(x), _p(y), float(alpha), _stream(stream)))
        return y

    def work(self) -> dict:
        """Work an apply runs under the underflow cutoffs (bem_op_get_work)."""
        w = OpWork()
        _check(lib().bem_op_get_work(self.h, C.byref(w)))
        return {k: getattr(w, k) for k, _ in OpWork._fields_}

    def launch_count(self) -> int:
        n = C.c_int32()
        _check(lib().bem_op_launch_count(self.h, C.byref(n)))
        return n.value

    def set_profiling(self, on: bool):
        _check(lib().bem_op_set_profiling(self.h, 1 if on else 0))

    def timings(self):
        out = np.empty(5)
        _check(lib().bem_op_get_timings(self.h, _p(out)))
        return dict(near=out[0], up=out[1], coupling=out[2], down=out[3])

    def close(self):
        if getattr(self, "h", None):
            _check(lib().bem_op_destroy(self.h))
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def cqm_forward(x_time, N: int, R: float, out=None, stream=None):
    import torch
    assert x_time.dtype == torch.complex128 and x_time.is_cuda and x_time.is_contiguous()
    assert x_time.dim() == 2 and x_time.shape[0] == N + 1, "x_time must be [N+1][M_loc]"
    out = torch.empty_like(x_time) if out is None else out
    assert out.dtype == torch.complex128 and out.is_contiguous() and out.shape == x_time.shape
    assert out.device == x_time.device and out.data_ptr() != x_time.data_ptr()
    _check(lib().cqm_forward(_p(x_time), _p(out), x_time.shape[1], int(N), float(R), _stream(stream)))
    return out


def cqm_inverse(y_freq, N: int, R: float, out=None, stream=None):
    import torch
    assert y_freq.dtype == torch.complex128 and y_freq.is_cuda and y_freq.is_contiguous()
    assert y_freq.dim() == 2 and y_freq.shape[0] == N + 1, "y_freq must be [N+1][M_loc]"
    out = torch.empty_like(y_freq) if out is None else out
    assert out.dtype == torch.complex128 and out.is_contiguous() and out.shape == y_freq.shape
    assert out.device == y_freq.device and out.data_ptr() != y_freq.data_ptr()
    _check(lib().cqm_inverse(_p(y_freq), _p(out), y_freq.shape[1], int(N), float(R), _stream(stream)))
    return out


def _row_array(ptrs):
    arr = (C.c_void_p * len(ptrs))(*[int(p) for p in ptrs])
    return arr


def cqm_forward_rows(x_time, N: int, R: float, out_rows, stream=None):
    """Forward transform of x_time [N+1][M_loc] whose frequency row l is stored at the
    device address out_rows[l] (possibly a peer rank's buffer): transform + transpose in one kernel."""
    import torch
    assert x_time.dtype == torch.complex128 and x_time.is_cuda and x_time.is_contiguous()
    assert len(out_rows) == N + 1
    _check(lib().cqm_forward_rows(_p(x_time), x_time.shape[1], _row_array(out_rows), int(N), float(R),
                                  _stream(stream)))


def cqm_inverse_rows(in_rows, N: int, R: float, M_loc: int, out=None, device=None, stream=None):
    """Inverse transform reading frequency row l at device address in_rows[l] -> [N+1][M_loc]."""
    import torch
    assert len(in_rows) == N + 1
    if out is None:
        out = torch.empty((N + 1, M_loc), dtype=torch.complex128, device=device or torch.cuda.current_device())
    _check(lib().cqm_inverse_rows(_row_array(in_rows), _p(out), int(M_loc), int(N), float(R), _stream(stream)))
    return out


def ipc_handle(t) -> bytes:
    """64-byte CUDA IPC handle of the allocation holding tensor t (t must start the allocation)."""
    buf = C.create_string_buffer(64)
    _check(lib().bem_ipc_get_handle(C.c_void_p(t.data_ptr()), buf))
    return buf.raw


def ipc_handle_ptr(ptr: int) -> bytes:
    """64-byte CUDA IPC handle of a raw allocation from device_alloc."""
    buf = C.create_string_buffer(64)
    _check(lib().bem_ipc_get_handle(C.c_void_p(ptr), buf))
    return buf.raw


def ipc_open(handle: bytes, device: int) -> int:
    out = C.c_void_p()
    _check(lib().bem_ipc_open_handle(C.c_char_p(handle), int(device), C.byref(out)))
    return out.value


def ipc_close(ptr: int):
    _check(lib().bem_ipc_close(C.c_void_p(ptr)))


def device_alloc(nbytes: int, device: int) -> int:
    out = C.c_void_p()
    _check(lib().bem_device_alloc(int(nbytes), int(device), C.byref(out)))
    return out.value


def device_free(ptr: int):
    _check(lib().bem_device_free(C.c_void_p(ptr)))


def shard_frequencies(L: int, G: int):
    """The library's frequency shard of every rank (bem_shard_frequencies): local lists
    (the op's local_l of each rank, in order)."""
    owner = np.empty(L, dtype=np.int32)
    slot = np.empty(L, dtype=np.int32)
    _check(lib().bem_shard_frequencies(int(L), int(G), _p(owner), _p(slot)))
    out = [np.empty(int((owner == g).sum()), dtype=np.int32) for g in range(G)]
    for l in range(L):
        out[owner[l]][slot[l]] = l
    return out


def dof_range(M: int, G: int, g: int):
    return M * g // G, M * (g + 1) // G


class Comm:
    """NCCL communicator of a frequency-sharded run (bem_comm_init), one per rank.
    The 128-byte unique id is created on rank 0 and broadcast over `group`
    (torch.distributed): plumbing only, the collectives run inside libbem."""

    def __init__(self, rank: int, world: int, device: int, group=None):
        import torch.distributed as dist
        uid = C.create_string_buffer(128)
        if rank == 0:
            _check(lib().bem_comm_unique_id(uid))
        obj = [uid.raw if rank == 0 else None]
        if world > 1:
            dist.broadcast_object_list(obj, src=0, group=group)
        h = C.c_void_p()
        _check(lib().bem_comm_init(C.c_char_p(obj[0]), int(world), int(rank), int(device), C.byref(h)))
        self.h, self.rank, self.world, self.device = h, rank, world, device

    def close(self):
        if getattr(self, "h", None):
            _check(lib().bem_comm_destroy(self.h))
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def time_step_sharded(op: Operator, x_loc, R: float, comm: Comm, y=None, stream=None):
    """The time-domain step on G ranks (bem_time_step_sharded): x_loc [L][M_g] complex, this
    rank's DOF columns, on the op's device; NCCL all-to-alls inside the library."""
    import torch
    assert x_loc.dtype == torch.complex128 and x_loc.is_cuda and x_loc.is_contiguous() and x_loc.shape[0] == op.L
    y = torch.empty_like(x_loc) if y is None else y
    assert y.shape == x_loc.shape and y.dtype == x_loc.dtype and y.is_contiguous()
    _check(lib().bem_time_step_sharded(op.h, _p(x_loc), _p(y), int(x_loc.shape[1]), float(R), comm.h,
                                       _stream(stream)))
    return y


def cqm_solve(op: Operator, g_time, R: float, tol: float = 1e-8, restart: int = 50, max_iter: int = 2000,
              stream=None, raise_on_noconv: bool = True, comm: Comm | None = None):
    """phi = Re inverse(V(s_l)^{-1} forward(g)) (frequency-decoupled GMRES).  With comm
    (G ranks): g_time is this rank's DOF shard [N+1][M_g] and op holds this rank's
    frequency shard; the transposes are NCCL all-to-alls inside the library."""
    import torch
    assert g_time.dtype == torch.float64 and g_time.is_cuda and g_time.is_contiguous()
    phi = torch.empty_like(g_time)
    st = SolveStats()
    code = lib().cqm_solve(op.h, _p(g_time), _p(phi), g_time.shape[1], float(R), float(tol), int(restart),
                           int(max_iter), comm.h if comm is not None else None, _stream(stream), C.byref(st))
    if code != 0 and not (code == BEM_ENOCONV and not raise_on_noconv):
        _check(code)
    return phi, {k: getattr(st, k) for k, _ in SolveStats._fields_ if k != "pad_"}


def cqm_mot_solve(op: Operator, g_time, tol: float = 1e-10, restart: int = 50, max_iter: int = 2000, stream=None,
                  raise_on_noconv: bool = True):
    """Marching on in time with the compressed weights (eq:cqmrhs; op.mot_prepare first)."""
    import torch
    assert g_time.dtype == torch.float64 and g_time.is_cuda and g_time.is_contiguous()
    phi = torch.empty_like(g_time)
    st = SolveStats()
    code = lib().cqm_mot_solve(op.h, _p(g_time), _p(phi), float(tol), int(restart), int(max_iter), _stream(stream),
                               C.byref(st))
    if code != 0 and not (code == BEM_ENOCONV and not raise_on_noconv):
        _check(code)
    return phi, {k: getattr(st, k) for k, _ in SolveStats._fields_ if k != "pad_"}


def solve_multifreq(op: Operator, g_freq, tol: float = 1e-8, restart: int = 50, max_iter: int = 2000, stream=None,
                    raise_on_noconv: bool = True):
    """phi^_t = V(s_{local_l[t]})^{-1} g^_t for the op's local frequencies (batched GMRES, frequency domain)."""
    import torch
    assert g_freq.dtype == torch.complex128 and g_freq.is_cuda and g_freq.is_contiguous()
    phi = torch.empty_like(g_freq)
    st = SolveStats()
    code = lib().bem_solve_multifreq(op.h, _p(g_freq), _p(phi), float(tol), int(restart), int(max_iter),
                                     _stream(stream), C.byref(st))
    if code != 0 and not (code == BEM_ENOCONV and not raise_on_noconv):
        _check(code)
    return phi, {k: getattr(st, k) for k, _ in SolveStats._fields_ if k != "pad_"}


def debug_sharded_step(ops, xs, R: float, stream=None):
    """bem_debug_sharded_step: G virtual ranks in one process (device-copy exchange)."""
    import torch
    G = len(ops)
    oa = (C.c_void_p * G)(*[o.h.value for o in ops])
    ys = [torch.empty_like(x) for x in xs]
    xa = (C.c_void_p * G)(*[x.data_ptr() for x in xs])
    ya = (C.c_void_p * G)(*[y.data_ptr() for y in ys])
    _check(lib().bem_debug_sharded_step(G, oa, xa, ya, float(R), _stream(stream)))
    return ys


def debug_aca_blocks(tree: Tree, s, eps: float, blocks):
    """The assembly's MACA on the listed far blocks only: ranks and pivots (k_l, q_l)."""
    s = np.ascontiguousarray(s, dtype=np.complex128)
    blocks = np.ascontiguousarray(blocks, dtype=np.int32)
    ranks = np.empty(len(blocks), dtype=np.int32)
    piv = np.empty((len(blocks) * min(len(s), tree.p * tree.p), 2), dtype=np.int32)
    tot = C.c_int64()
    _check(lib().bem_debug_aca_blocks(tree.h, _p(s), len(s), float(eps), _p(blocks), len(blocks), _p(ranks),
                                      _p(piv), C.byref(tot)))
    return dict(ranks=ranks, pivots=piv[:tot.value])


def debug_pinned(x, device: int = 0):
    x = np.ascontiguousarray(x, dtype=np.float64).ravel()
    e, s, c = np.empty_like(x), np.empty_like(x), np.empty_like(x)
    _check(lib().bem_debug_pinned(_p(x), len(x), _p(e), _p(s), _p(c), int(device)))
    return e, s, c


def dirichlet_solve(op: Operator, g_time, R: float, tol: float = 1e-8, restart: int = 50, max_iter: int = 2000,
                    stream=None):
    """Direct Dirichlet formulation (eq:cqmdir P:1801-1806), frequency-decoupled
    (Remark P:1607-1614): V(s_l) q^_l = (-1/2 I + K(s_l)) g^_l for every l,
    q = Re inverse(q^).  Every step runs in libbem's kernels: K4 forward, the
    double-layer apply, batched GMRES on V, K4 inverse.  g_time: [N+1][M] real."""
    import torch
    N = op.L - 1
    gf = cqm_forward(g_time.to(torch.complex128).contiguous(), N, R, stream=stream)
    rhs = op.apply_dl(gf, alpha=-0.5, stream=stream)
    qf, st = solve_multifreq(op, rhs, tol=tol, restart=restart, max_iter=max_iter, stream=stream)
    return cqm_inverse(qf, N, R, stream=stream).real.contiguous(), st


def debug_fastmath(x, device: int = 0, variant: int = 64):
    """Device table-driven exp (x <= 0) / sin / cos of the hot kernels, for accuracy tests."""
    x = np.ascontiguousarray(x, dtype=np.float64).ravel()
    e, s, c = np.empty_like(x), np.empty_like(x), np.empty_like(x)
    _check(lib().bem_debug_fastmath(_p(x), len(x), _p(e), _p(s), _p(c), int(device), int(variant)))
    return e, s, c


def fp64_peak(device: int = 0, stream=None, mode: int = 0) -> float:
    """mode 0: DFMA loop, 1: DMMA (mma.sync f64) loop, 2: both concurrently."""
    out = C.c_double()
    _check(lib().bem_debug_fp64_peak_ex(int(device), _stream(stream), int(mode), C.byref(out)))
    return out.value
