"""ctypes wrapper of the CPU oracle -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this package.  The product (paper_2006_05186_b200)
never imports it and shares no code with it.

Function-to-paper map (P = /root/reference/PAPER.md):
  geometry / self_integral   C1/C3: flat triangles P:558-559, 7-pt rule (north_star)
  kernel                     eq:fundsol P:479-482
  frequencies                eq:cqm_freq P:443-447 (L = N+1, north_star sign)
  dense_matrix               collocation analogue of the Galerkin entries P:584-609
  H2.build                   cluster tree P:807-835, partition P:843-912, bases P:957-978
  H2.aca                     MACA Alg. 2, stop P:1298-1310
  H2.apply                   eq:lrfinal P:1404-1410 (DENSE / H2ONLY / H2ACA / COMBINED)
  H2.aca_near                Alg. 3 NEAR branch P:1426-1431, P:1444-1450 (NEXT-4)
  dense_matrix_pinned        C3 entries in the pinned arithmetic the near MACA reads
  H2.time_weights            eq:fastdft P:1542-1553 (dhat = R-scaled inverse DFT of Z rows)
  H2.conv / weight_dense     eq:fastrhs P:1566-1573 / the weights V^_n assembled densely
  H2.mot                     eq:cqmrhs P:652-680 with one LU of V^_0
Every function is pinned by tests/test_oracle_*.py and tests/test_golden.py (no
"parity unpinned" entries).
  forward / inverse          eq:omega_n P:436-441, eq:slphelm P:529-540
  H2.gmres                   frequency-decoupled solve, Remark P:1607-1614
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from .build import build as _build

MODE_DENSE, MODE_H2ONLY, MODE_H2ACA, MODE_COMBINED = 0, 1, 2, 3

_lib = None


def lib():
    global _lib
    if _lib is None:
        path = _build()
        L = C.CDLL(path)
        d, i32, i64, vp = C.c_double, C.c_int32, C.c_int64, C.c_void_p
        P = C.POINTER
        L.orc_num_threads.restype = C.c_int
        L.orc_set_threads.argtypes = [C.c_int]
        L.orc_geometry.argtypes = [vp, vp, i64, vp, vp, vp, vp, vp]
        L.orc_self_integral.argtypes = [vp, vp, vp]
        L.orc_self_integral.restype = d
        L.orc_kernel.argtypes = [d, d, d, vp]
        L.orc_kernel_pinned.argtypes = [d, d, d, vp]
        L.orc_phi_self.argtypes = [d, d, d, vp]
        L.orc_pexp_n.argtypes = [vp, vp, i64]
        L.orc_psincos_n.argtypes = [vp, vp, vp, i64]
        L.orc_psum.argtypes = [vp, i64]
        L.orc_psum.restype = d
        L.orc_frequencies.argtypes = [i32, d, d, i32, vp]
        L.orc_dense_matrix.argtypes = [vp, vp, i64, d, d, vp]
        L.orc_h2_build.argtypes = [vp, vp, i64, i32, d, i32]
        L.orc_h2_build.restype = vp
        L.orc_h2_destroy.argtypes = [vp]
        L.orc_h2_stats.argtypes = [vp, vp]
        L.orc_h2_export.argtypes = [vp, vp, vp, vp, vp, vp]
        L.orc_h2_export_bases.argtypes = [vp, vp, vp, vp, vp]
        L.orc_h2_aca.argtypes = [vp, vp, i32, d, vp, i64, vp, vp]
        L.orc_h2_aca.restype = i64
        L.orc_h2_aca_keep.argtypes = [vp, vp, i32, d, vp, i64, vp, i32, vp, vp]
        L.orc_h2_aca_keep.restype = i64
        L.orc_h2_apply_sample.argtypes = [vp, i32, vp, i32, vp, i32, vp, vp, vp, i64, vp, i64]
        L.orc_h2_apply_sample.restype = C.c_int
        L.orc_h2_aca_export.argtypes = [vp, vp, i64, vp, vp]
        L.orc_h2_apply.argtypes = [vp, i32, vp, i32, vp, i32, vp, vp]
        L.orc_h2_apply.restype = C.c_int
        L.orc_forward.argtypes = [vp, vp, i64, i32, d]
        L.orc_inverse.argtypes = [vp, vp, i64, i32, d]
        L.orc_h2_gmres.argtypes = [vp, i32, vp, i32, vp, i32, vp, vp, d, i32, i32, vp, vp]
        L.orc_h2_gmres.restype = C.c_int
        L.orc_admissible.argtypes = [vp, vp, d]
        L.orc_admissible.restype = i32
        L.orc_aca_matrix.argtypes = [vp, i32, i32, d, vp, vp, vp, vp, vp]
        L.orc_aca_matrix.restype = i32
        L.orc_h2_apply_dl.argtypes = [vp, i32, vp, i32, vp, i32, vp, vp, d]
        L.orc_h2_apply_dl.restype = C.c_int
        L.orc_dense_matrix_dl.argtypes = [vp, vp, i64, d, d, vp]
        L.orc_normals.argtypes = [vp, vp, i64, vp]
        L.orc_h2_aca_near.argtypes = [vp, vp, i32, d, vp, i64, vp, vp]
        L.orc_h2_aca_near.restype = i64
        L.orc_h2_aca_near_export.argtypes = [vp, vp, i64, vp, vp]
        L.orc_dense_matrix_pinned.argtypes = [vp, vp, i64, d, d, vp]
        L.orc_pexpm1.argtypes = [d]
        L.orc_h2_time_weights.argtypes = [vp, d]
        L.orc_h2_time_weights.restype = C.c_int
        L.orc_h2_conv.argtypes = [vp, vp, vp, i32]
        L.orc_h2_conv.restype = C.c_int
        L.orc_h2_weight_dense.argtypes = [vp, i32, vp]
        L.orc_h2_weight_dense.restype = C.c_int
        L.orc_pexpm1.restype = d
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _c128(a):
    return np.ascontiguousarray(a, dtype=np.complex128)


def _i32(a):
    return np.ascontiguousarray(a, dtype=np.int32)


def set_threads(n: int):
    lib().orc_set_threads(int(n))


def num_threads() -> int:
    return int(lib().orc_num_threads())


def geometry(V, T):
    V, T = _f64(V), _i32(T)
    M = len(T)
    cen = np.empty((M, 3)); area = np.empty(M); node = np.empty((M, 7, 3)); wq = np.empty(7); J = np.empty(M)
    lib().orc_geometry(_p(V), _p(T), M, _p(cen), _p(area), _p(node), _p(wq), _p(J))
    return dict(cen=cen, area=area, node=node, wq=wq, J=J)


def self_integral(a, b, c):
    return lib().orc_self_integral(_p(_f64(a)), _p(_f64(b)), _p(_f64(c)))


def kernel(r, s, pinned=False):
    out = np.empty(2)
    f = lib().orc_kernel_pinned if pinned else lib().orc_kernel
    f(float(r), float(np.real(s)), float(np.imag(s)), _p(out))
    return complex(out[0], out[1])


def phi_self(r, s):
    out = np.empty(2)
    lib().orc_phi_self(float(r), float(np.real(s)), float(np.imag(s)), _p(out))
    return complex(out[0], out[1])


def pexp(x):
    x = _f64(x).ravel()
    y = np.empty_like(x)
    lib().orc_pexp_n(_p(x), _p(y), len(x))
    return y


def psincos(t):
    t = _f64(t).ravel()
    s = np.empty_like(t); c = np.empty_like(t)
    lib().orc_psincos_n(_p(t), _p(s), _p(c), len(t))
    return s, c


def psum(v):
    v = _f64(v).ravel()
    return lib().orc_psum(_p(v), len(v))


def default_R(N: int) -> float:
    """R = 10^{-5/N}."""
    return 10.0 ** (-5.0 / N)


def frequencies(N, T, R=None, method=2):
    R = default_R(N) if R is None else R
    out = np.empty(2 * (N + 1))
    lib().orc_frequencies(int(N), float(T), float(R), int(method), _p(out))
    return out[0::2] + 1j * out[1::2]


def admissible(box_r, box_c, eta):
    """eq:qadm; boxes as (lo_x,lo_y,lo_z,hi_x,hi_y,hi_z)."""
    return bool(lib().orc_admissible(_p(_f64(box_r)), _p(_f64(box_c)), float(eta)))


def aca_matrix(A, eps):
    """MACA (Alg. 2) on the unfolding A[q,l] (pp x L complex)."""
    A = _c128(A)
    pp, L = A.shape
    rmax = min(pp, L)
    piv = np.empty((rmax, 2), dtype=np.int32)
    Z = np.empty((rmax, L), dtype=np.complex128)
    Cm = np.empty((rmax, pp), dtype=np.complex128)
    Dm = np.empty((rmax, L), dtype=np.complex128)
    nrm = np.empty(rmax)
    r = lib().orc_aca_matrix(_p(A), pp, L, float(eps), _p(piv), _p(Z), _p(Cm), _p(Dm), _p(nrm))
    return dict(rank=r, pivots=piv[:r], Z=Z[:r], C=Cm[:r], D=Dm[:r], nrm2=nrm[:r])


def dense_matrix(V, T, s):
    V, T = _f64(V), _i32(T)
    M = len(T)
    A = np.empty((M, M), dtype=np.complex128)
    lib().orc_dense_matrix(_p(V), _p(T), M, float(np.real(s)), float(np.imag(s)), _p(A))
    return A


def dense_matrix_pinned(V, T, s):
    """C3 collocation matrix with every entry in pinned arithmetic (the values
    the near-field MACA reads, NEXT-4)."""
    V, T = _f64(V), _i32(T)
    M = len(T)
    A = np.empty((M, M), dtype=np.complex128)
    lib().orc_dense_matrix_pinned(_p(V), _p(T), M, float(np.real(s)), float(np.imag(s)), _p(A))
    return A


def pexpm1(x):
    return lib().orc_pexpm1(float(x))


def dense_matrix_dl(V, T, s):
    """Double-layer collocation matrix K(s) (NEXT-1), K[i,i] = 0."""
    V, T = _f64(V), _i32(T)
    M = len(T)
    A = np.empty((M, M), dtype=np.complex128)
    lib().orc_dense_matrix_dl(_p(V), _p(T), M, float(np.real(s)), float(np.imag(s)), _p(A))
    return A


def normals(V, T):
    V, T = _f64(V), _i32(T)
    n = np.empty((len(T), 3))
    lib().orc_normals(_p(V), _p(T), len(T), _p(n))
    return n


def forward(xt, N, R):
    xt = _c128(xt)
    M = xt.shape[1]
    xf = np.empty((N + 1, M), dtype=np.complex128)
    lib().orc_forward(_p(xt), _p(xf), M, int(N), float(R))
    return xf


def inverse(yf, N, R):
    yf = _c128(yf)
    M = yf.shape[1]
    yt = np.empty((N + 1, M), dtype=np.complex128)
    lib().orc_inverse(_p(yf), _p(yt), M, int(N), float(R))
    return yt


class H2:
    """Oracle H^2 structure (+ optional ACA) on a mesh."""

    def __init__(self, V, T, nmin, eta, m):
        self._V, self._T = _f64(V), _i32(T)
        self.M = len(self._T)
        self.m, self.p = int(m), int(m) ** 3
        self.h = lib().orc_h2_build(_p(self._V), _p(self._T), self.M, int(nmin), float(eta), int(m))
        st = np.empty(7, dtype=np.int64)
        lib().orc_h2_stats(self.h, _p(st))
        self.n_clusters, self.n_leaves, self.n_near, self.n_far, self.nnz_near, self.depth, _ = map(int, st)
        self.s = None

    def __del__(self):
        h = getattr(self, "h", None)
        if h:
            try:
                lib().orc_h2_destroy(h)
            except Exception:  # interpreter shutdown: module globals already gone
                pass
            self.h = None

    def export(self):
        perm = np.empty(self.M, dtype=np.int32)
        clusters = np.empty((self.n_clusters, 5), dtype=np.int32)
        boxes = np.empty((self.n_clusters, 6))
        near = np.empty((self.n_near, 2), dtype=np.int32)
        far = np.empty((self.n_far, 2), dtype=np.int32)
        lib().orc_h2_export(self.h, _p(perm), _p(clusters), _p(boxes), _p(near), _p(far))
        return dict(perm=perm, clusters=clusters, boxes=boxes, near=near, far=far)

    def bases(self):
        U = np.empty((self.M, self.p)); W = np.empty((self.M, self.p))
        E = np.empty((self.n_clusters, self.p, self.p)); xi = np.empty((self.n_clusters, 3, self.m))
        lib().orc_h2_export_bases(self.h, _p(U), _p(W), _p(E), _p(xi))
        return dict(U=U, W=W, E=E, xi=xi)

    def aca(self, s, eps, blocks=None, keep=None):
        """MACA of every far block (or of `blocks`); keep: the frequencies whose Z
        columns are stored (default all L; applies are then limited to them)."""
        s = _c128(s)
        self.s = s
        L = len(s)
        if blocks is None:
            blk, nb = None, self.n_far
        else:
            blk = np.ascontiguousarray(blocks, dtype=np.int32)
            nb = len(blk)
        kp = None if keep is None else np.ascontiguousarray(np.unique(keep), dtype=np.int32)
        nk = L if kp is None else len(kp)
        ranks = np.empty(nb, dtype=np.int32)
        fragile = np.empty(nb, dtype=np.int32)
        tot = lib().orc_h2_aca_keep(self.h, _p(s), L, float(eps), _p(blk), nb, _p(kp), 0 if kp is None else nk,
                                    _p(ranks), _p(fragile))
        piv = np.empty((tot, 2), dtype=np.int32)
        Z = np.empty(tot * nk, dtype=np.complex128)
        lib().orc_h2_aca_export(self.h, _p(blk), nb, _p(piv), _p(Z))
        return dict(ranks=ranks, pivots=piv, Z=Z, fragile=fragile)

    def aca_near(self, s, eps, blocks=None):
        """Near-field MACA on the near blocks (Alg. 3 NEAR branch; MODE_COMBINED)."""
        s = _c128(s)
        L = len(s)
        if blocks is None:
            blk, nb = None, self.n_near
        else:
            blk = np.ascontiguousarray(blocks, dtype=np.int32)
            nb = len(blk)
        ranks = np.empty(nb, dtype=np.int32)
        fragile = np.empty(nb, dtype=np.int32)
        tot = lib().orc_h2_aca_near(self.h, _p(s), L, float(eps), _p(blk), nb, _p(ranks), _p(fragile))
        if tot < 0:
            raise RuntimeError("oracle aca_near: far ACA was assembled for another L")
        piv = np.empty((tot, 2), dtype=np.int32)
        Z = np.empty(tot * L, dtype=np.complex128)
        lib().orc_h2_aca_near_export(self.h, _p(blk), nb, _p(piv), _p(Z))
        return dict(ranks=ranks, pivots=piv, Z=Z, fragile=fragile)

    def time_weights(self, R):
        """dhat = R-scaled inverse DFT of every far / near skeleton coefficient row
        (eq:fastdft P:1542-1553); needs aca() and aca_near() on all L frequencies."""
        if lib().orc_h2_time_weights(self.h, float(R)) != 0:
            raise RuntimeError("oracle time_weights: run aca() and aca_near() first")
        self.R = float(R)

    def conv(self, q, kmax=None):
        """y[n] = sum_{k <= min(n, kmax)} V^_{n-k} q[k] with the compressed time weights
        (eq:fastrhs P:1566-1573); q [L][M] (input order), complex result."""
        q = _c128(q)
        L = q.shape[0]
        y = np.empty_like(q)
        if lib().orc_h2_conv(self.h, _p(q), _p(y), int(L - 1 if kmax is None else kmax)) != 0:
            raise RuntimeError("oracle conv: call time_weights() first")
        return y

    def weight_dense(self, n):
        """Dense V^_n (input order) assembled from the compressed weights."""
        A = np.empty((self.M, self.M), dtype=np.complex128)
        if lib().orc_h2_weight_dense(self.h, int(n), _p(A)) != 0:
            raise RuntimeError("oracle weight_dense: call time_weights() first / n out of range")
        return A

    def mot(self, g):
        """Marching on in time with the compressed weights (eq:cqmrhs P:652-680, one LU
        of V^_0 P:686-703; Dirichlet single-layer problem V q = g): for n = 0..N,
        Re V^_0 q_n = g_n - Re sum_{k<n} V^_{n-k} q_k.  g real [L][M]; returns q real."""
        import scipy.linalg as sla
        g = np.asarray(g, dtype=np.float64)
        L, M = g.shape
        W = [self.weight_dense(n).real for n in range(L)]
        lu = sla.lu_factor(W[0])
        q = np.zeros((L, M))
        for n in range(L):
            rhs = g[n] - sum(W[n - k] @ q[k] for k in range(n))
            q[n] = sla.lu_solve(lu, rhs)
        return q

    def apply(self, mode, s, x, lsel=None):
        """y[t] = V(s[lsel[t]]) x[t]; x shape [nsel][M] complex (input order)."""
        s = _c128(s)
        L = len(s)
        lsel = np.arange(L, dtype=np.int32) if lsel is None else _i32(lsel)
        x = _c128(x)
        assert x.shape == (len(lsel), self.M)
        y = np.empty_like(x)
        rc = lib().orc_h2_apply(self.h, int(mode), _p(s), L, _p(lsel), len(lsel), _p(x), _p(y))
        if rc != 0:
            raise RuntimeError("oracle apply: ACA not assembled for these frequencies")
        return y

    def apply_sample(self, s, x, lsel, far_blocks, near_blocks):
        """H2ACA apply with only the listed far / near blocks contributing: a bounded
        sample of the apply's work (bench.py times the oracle with it; not a parity path)."""
        s = _c128(s)
        lsel = _i32(lsel)
        x = _c128(x)
        fb, nb = _i32(far_blocks), _i32(near_blocks)
        y = np.empty_like(x)
        rc = lib().orc_h2_apply_sample(self.h, MODE_H2ACA, _p(s), len(s), _p(lsel), len(lsel), _p(x), _p(y),
                                       _p(fb), len(fb), _p(nb), len(nb))
        if rc != 0:
            raise RuntimeError("oracle apply_sample: ACA missing for a sampled block / frequency")
        return y

    def apply_dl(self, mode, s, x, lsel=None, alpha=0.0):
        """y[t] = (alpha I + K(s[lsel[t]])) x[t] (double layer, NEXT-1)."""
        s = _c128(s)
        L = len(s)
        lsel = np.arange(L, dtype=np.int32) if lsel is None else _i32(lsel)
        x = _c128(x)
        assert x.shape == (len(lsel), self.M)
        y = np.empty_like(x)
        rc = lib().orc_h2_apply_dl(self.h, int(mode), _p(s), L, _p(lsel), len(lsel), _p(x), _p(y), float(alpha))
        if rc != 0:
            raise RuntimeError("oracle apply_dl: ACA not assembled for these frequencies")
        return y

    def gmres(self, mode, s, b, lsel=None, tol=1e-8, restart=50, maxit=2000):
        s = _c128(s)
        L = len(s)
        lsel = np.arange(L, dtype=np.int32) if lsel is None else _i32(lsel)
        b = _c128(b)
        x = np.empty_like(b)
        it = np.empty(len(lsel), dtype=np.int32)
        rr = np.empty(len(lsel))
        rc = lib().orc_h2_gmres(self.h, int(mode), _p(s), L, _p(lsel), len(lsel), _p(b), _p(x), float(tol),
                                int(restart), int(maxit), _p(it), _p(rr))
        if rc != 0:
            raise RuntimeError("oracle gmres: ACA not assembled")
        return x, it, rr
