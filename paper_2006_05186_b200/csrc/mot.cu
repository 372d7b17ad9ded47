// Time-domain path with compressed weights.
//
// On a BEM_MODE_COMBINED operator (every block b in P+ and P- in MACA skeleton
// form, eq:lrfinal P:1404-1410) the CQM integration weights inherit the format
// (eq:fastdft P:1542-1553):
//   V^_n[b] = sum_t C_{b,t} dhat_{b,t}[n],
//   dhat_{b,t}[n] = (R^{-n}/L) sum_l Z_b[t,l] e^{+2 pi i (n l mod L)/L}   (reading D2, L = N+1),
//   C_{b,t} = S_b(s_{k_t}) between the cluster bases (far) or V_{k_t}[b] (near, stored),
// so the discrete convolution of the right-hand side (eq:fastrhs P:1566-1573) is
//   f_n = sum_b sum_t C_{b,t} ( sum_{k<=n} dhat_{b,t}[n-k] X_{c,k} ),
// X_{c,k} = W_c^T q_k (far) or q_k|_c (near).  cqm_mot_solve marches on in time
// (eq:cqmrhs P:652-680): Re V^_0 q_n = g_n - Re f_n(q_0..q_{n-1}), with V^_0 solved
// by GMRES through the same skeleton (the paper factorises V^_0 once, P:686-703;
// an iterative solver is its stated alternative).
//
// Kernels (memory/latency-bound matrix-vector work; deterministic): dhat_kernel
// (the transform of the coefficient rows, setup), far_slice_kernel (stores the
// pivot slices S_b(s_{k_t}), setup), conv_block_kernel<far|near> (one CTA per
// block and time column: history sums, then the slice products) with fixed-order
// row reductions, g0_block_kernel<far|near> (Re V^_0 as a real H^2 matrix, every
// GMRES step).
#include <algorithm>
#include <cmath>
#include <vector>

#include "common.cuh"

namespace bem {
namespace {

__global__ void dhat_kernel(const double2* __restrict__ Z, double2* __restrict__ D, int64_t rows, int L, double R) {
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= rows * L) return;
  const int64_t row = idx / L;
  const int n = (int)(idx - row * L);
  const double2* z = Z + row * L;
  double ar = 0.0, ai = 0.0;
  for (int l = 0; l < L; ++l) {
    const int m = (int)(((int64_t)n * l) % L);
    double sn, cs;
    sincospi(2.0 * (double)m / (double)L, &sn, &cs);
    ar += z[l].x * cs - z[l].y * sn;
    ai += z[l].x * sn + z[l].y * cs;
  }
  const double sc = pow(R, -(double)n) / (double)L;
  D[idx] = make_double2(ar * sc, ai * sc);
}

// S_b(s_{k_t})[mu][nu] = e^{-s r}/(4 pi r), r = |xi_{c,nu} - xi_{r,mu}|
__global__ void far_slice_kernel(const int32_t* __restrict__ far_r, const int32_t* __restrict__ far_c,
                                 const double* __restrict__ xi, const double2* __restrict__ s,
                                 const int32_t* __restrict__ rank, const int32_t* __restrict__ pivk, int rcap,
                                 const int64_t* __restrict__ fsoff, double2* __restrict__ S, int m, int p) {
  const int b = blockIdx.x;
  const double* xr = xi + (int64_t)far_r[b] * 3 * m;
  const double* xc = xi + (int64_t)far_c[b] * 3 * m;
  const int rk = rank[b];
  for (int idx = threadIdx.x; idx < rk * p * p; idx += blockDim.x) {
    const int t = idx / (p * p), e = idx - t * p * p;
    const int mu = e / p, nu = e - mu * p;
    const double dx = xc[nu % m] - xr[mu % m];
    const double dy = xc[m + (nu / m) % m] - xr[m + (mu / m) % m];
    const double dz = xc[2 * m + nu / (m * m)] - xr[2 * m + mu / (m * m)];
    const double r = sqrt((dx * dx + dy * dy) + dz * dz);
    const double2 sv = s[pivk[(int64_t)b * rcap + t]];
    const double E = exp(-(sv.x * r));
    double sn, cs;
    sincos(sv.y * r, &sn, &cs);
    const double inv = 1.0 / (12.566370614359172954 * r);
    S[fsoff[b] + idx] = make_double2(E * cs * inv, -(E * sn) * inv);
  }
}

struct ConvArgs {
  int64_t M;
  int L, p, HS, n0, kmax;  // HS: history stride (time columns held in XH / Q)
  const int32_t* far_ptr;
  const int32_t* far_sorted;
  const int32_t* far_c;
  const int32_t* rank;
  const int64_t* zoff;
  const int64_t* fsoff;
  const double2* Df;
  const double2* fS;
  const double2* XH;  // [C][HS][p]
  double2* yhat;      // [C][ncols][p]
  int ncols;
  // near
  const int32_t* leaves;
  const int32_t* nb_ptr;
  const int32_t* nb_sorted;
  const int32_t* near_r;
  const int32_t* near_c;
  const int32_t* cbegin;
  const int32_t* cend;
  const int32_t* nrank;
  const int64_t* nzoff;
  const int64_t* nsoff;
  const double2* Dn;
  const double2* nS;
  const double2* Q;  // [HS][M] cluster order
  double2* ycn;      // [ncols][M] cluster order
};

__device__ __forceinline__ void cmac(double2& a, double2 x, double2 y) {
  a.x = fma(x.x, y.x, a.x);
  a.x = fma(-x.y, y.y, a.x);
  a.y = fma(x.x, y.y, a.y);
  a.y = fma(x.y, y.x, a.y);
}

// One CTA per (block, time column): u_t = sum_{k<=min(n,kmax)} dhat_{b,t}[n-k] X_c[k] for a chunk
// of kTC terms at a time (shared memory), then thread (tc, row) accumulates
// sum_{t in its share} C_{b,t}[row,:] u_t; the kConvTC partial sums are added in a fixed
// order into the block's partial output (deterministic; rows are reduced per row cluster /
// row leaf by block_reduce_kernel).  far: X = XH[c][k][0..p), C_{b,t} = S_b(s_{k_t}) (p x p);
// near: X = Q[k][c0..c0+nc), C_{b,t} = V_{k_t}[b] (nr x nc).
constexpr int kTC = 8;       // terms staged per chunk
constexpr int kConvThreads = 256;

template <bool NEAR>
__global__ void __launch_bounds__(kConvThreads) conv_block_kernel(ConvArgs a, double2* __restrict__ part, int pmax) {
  extern __shared__ double2 sm[];
  const int b = blockIdx.x, j = blockIdx.y, n = a.n0 + j;
  int nr, nc, rk;
  const double2* D;
  const double2* S;
  if constexpr (NEAR) {
    const int r = a.near_r[b], c = a.near_c[b];
    nr = a.cend[r] - a.cbegin[r];
    nc = a.cend[c] - a.cbegin[c];
    rk = a.nrank[b];
    D = a.Dn + a.nzoff[b];
    S = a.nS + a.nsoff[b];
  } else {
    nr = nc = a.p;
    rk = a.rank[b];
    D = a.Df + a.zoff[b];
    S = a.fS + a.fsoff[b];
  }
  const int kend = min(n, a.kmax);
  double2* u = sm;                 // kTC x nc
  double2* red = sm + kTC * pmax;  // kTC x nr partials
  const int tc = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double2 acc[4] = {make_double2(0.0, 0.0), make_double2(0.0, 0.0), make_double2(0.0, 0.0), make_double2(0.0, 0.0)};
  for (int t0 = 0; t0 < rk; t0 += kTC) {
    const int nt = min(kTC, rk - t0);
    __syncthreads();
    for (int idx = threadIdx.x; idx < nt * nc; idx += kConvThreads) {
      const int tt = idx / nc, nu = idx - tt * nc;
      const double2* d = D + (int64_t)(t0 + tt) * a.L;
      double2 sacc = make_double2(0.0, 0.0);
      if constexpr (NEAR) {
        const int64_t col = a.cbegin[a.near_c[b]] + nu;
        for (int k = 0; k <= kend; ++k) cmac(sacc, d[n - k], a.Q[(int64_t)k * a.M + col]);
      } else {
        const int64_t base = (int64_t)a.far_c[b] * a.HS * a.p + nu;
        for (int k = 0; k <= kend; ++k) cmac(sacc, d[n - k], a.XH[base + (int64_t)k * a.p]);
      }
      u[tt * nc + nu] = sacc;
    }
    __syncthreads();
    if (tc < nt) {
      const double2* St = S + (int64_t)(t0 + tc) * nr * nc;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int row = lane + 32 * i;
        if (row < nr) {
          const double2* Sr = St + (int64_t)row * nc;
          for (int nu = 0; nu < nc; ++nu) cmac(acc[i], Sr[nu], u[tc * nc + nu]);
        }
      }
    }
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int row = lane + 32 * i;
    if (row < nr) red[tc * pmax + row] = acc[i];
  }
  __syncthreads();
  for (int row = threadIdx.x; row < nr; row += kConvThreads) {
    double2 v = make_double2(0.0, 0.0);
    for (int w = 0; w < kTC; ++w) { v.x += red[w * pmax + row].x; v.y += red[w * pmax + row].y; }
    part[((int64_t)b * a.ncols + j) * pmax + row] = v;
  }
}

// far: yhat[r][j][:] = sum over the row's blocks (far CSR order) of the block partials
__global__ void far_reduce_kernel(const int32_t* __restrict__ far_ptr, const int32_t* __restrict__ far_sorted,
                                  const double2* __restrict__ part, double2* __restrict__ yhat, int ncols, int p) {
  const int r = blockIdx.x, j = blockIdx.y;
  const int b0 = far_ptr[r], b1 = far_ptr[r + 1];
  if (b0 == b1) return;
  for (int mu = threadIdx.x; mu < p; mu += blockDim.x) {
    double2 v = make_double2(0.0, 0.0);
    for (int bi = b0; bi < b1; ++bi) {
      const double2 w = part[((int64_t)far_sorted[bi] * ncols + j) * p + mu];
      v.x += w.x; v.y += w.y;
    }
    yhat[((int64_t)r * ncols + j) * p + mu] = v;
  }
}

// near: ycn[j][rows of leaf] = sum over the leaf's near blocks of the block partials
__global__ void near_reduce_kernel(const int32_t* __restrict__ leaves, const int32_t* __restrict__ nb_ptr,
                                   const int32_t* __restrict__ nb_sorted, const int32_t* __restrict__ cb,
                                   const int32_t* __restrict__ ce, const double2* __restrict__ part,
                                   double2* __restrict__ ycn, int64_t M, int ncols, int pmax) {
  const int li = blockIdx.x, j = blockIdx.y;
  const int r = leaves[li];
  const int rb0 = cb[r], nr = ce[r] - rb0;
  for (int i = threadIdx.x; i < nr; i += blockDim.x) {
    double2 v = make_double2(0.0, 0.0);
    for (int bi = nb_ptr[li]; bi < nb_ptr[li + 1]; ++bi) {
      const double2 w = part[((int64_t)nb_sorted[bi] * ncols + j) * pmax + i];
      v.x += w.x; v.y += w.y;
    }
    ycn[(int64_t)j * M + rb0 + i] = v;
  }
}

// Re V^_0 as a real H^2 matrix: G_b = Re sum_t C_{b,t} dhat_{b,t}[0] (far: p x p between the
// cluster bases; near: n_r x n_c), assembled once so that each GMRES step of the MoT applies
// one real matrix per block instead of r_b terms.
__global__ void g0_far_build_kernel(const double2* __restrict__ fS, const int64_t* __restrict__ fsoff,
                                    const double2* __restrict__ Df, const int64_t* __restrict__ zoff,
                                    const int32_t* __restrict__ rank, int L, int p, double* __restrict__ G) {
  const int b = blockIdx.x;
  for (int e = threadIdx.x; e < p * p; e += blockDim.x) {
    double acc = 0.0;
    for (int t = 0; t < rank[b]; ++t) {
      const double2 sv = fS[fsoff[b] + (int64_t)t * p * p + e], d = Df[zoff[b] + (int64_t)t * L];
      acc += sv.x * d.x - sv.y * d.y;
    }
    G[(int64_t)b * p * p + e] = acc;
  }
}

__global__ void g0_near_build_kernel(const double2* __restrict__ nS, const int64_t* __restrict__ nsoff,
                                     const double2* __restrict__ Dn, const int64_t* __restrict__ nzoff,
                                     const int32_t* __restrict__ nrank, const int32_t* __restrict__ near_r,
                                     const int32_t* __restrict__ near_c, const int32_t* __restrict__ cb,
                                     const int32_t* __restrict__ ce, const int64_t* __restrict__ goff, int L,
                                     double* __restrict__ G) {
  const int b = blockIdx.x;
  const int nrnc = (ce[near_r[b]] - cb[near_r[b]]) * (ce[near_c[b]] - cb[near_c[b]]);
  for (int e = threadIdx.x; e < nrnc; e += blockDim.x) {
    double acc = 0.0;
    for (int t = 0; t < nrank[b]; ++t) {
      const double2 sv = nS[nsoff[b] + (int64_t)t * nrnc + e], d = Dn[nzoff[b] + (int64_t)t * L];
      acc += sv.x * d.x - sv.y * d.y;
    }
    G[goff[b] + e] = acc;
  }
}

// Re V^_0 x per block (one CTA per block; x_c staged in shared memory, thread = output
// row), partials reduced per row cluster / row leaf by far_reduce_kernel / near_reduce_kernel.
template <bool NEAR>
__global__ void __launch_bounds__(128) g0_block_kernel(const int32_t* __restrict__ blk_r,
                                                       const int32_t* __restrict__ blk_c,
                                                       const int32_t* __restrict__ cb, const int32_t* __restrict__ ce,
                                                       const int64_t* __restrict__ goff, const double* __restrict__ G,
                                                       const double2* __restrict__ x, double2* __restrict__ part,
                                                       int p, int pmax) {
  extern __shared__ double2 xs[];
  const int b = blockIdx.x;
  int nr, nc;
  const double2* xb;
  const double* Gb;
  if constexpr (NEAR) {
    nr = ce[blk_r[b]] - cb[blk_r[b]];
    nc = ce[blk_c[b]] - cb[blk_c[b]];
    xb = x + cb[blk_c[b]];
    Gb = G + goff[b];
  } else {
    nr = nc = p;
    xb = x + (int64_t)blk_c[b] * p;
    Gb = G + (int64_t)b * p * p;
  }
  for (int j = threadIdx.x; j < nc; j += blockDim.x) xs[j] = xb[j];
  __syncthreads();
  for (int i = threadIdx.x; i < nr; i += blockDim.x) {
    double2 acc = make_double2(0.0, 0.0);
    const double* Gi = Gb + (int64_t)i * nc;
    for (int j = 0; j < nc; ++j) {
      acc.x = fma(Gi[j], xs[j].x, acc.x);
      acc.y = fma(Gi[j], xs[j].y, acc.y);
    }
    part[(int64_t)b * pmax + i] = acc;
  }
}

__global__ void rhs_kernel(const double* __restrict__ g, const double2* __restrict__ f, double2* __restrict__ b,
                           int64_t M, int has_f) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= M) return;
  b[i] = make_double2(g[i] - (has_f ? f[i].x : 0.0), 0.0);
}

__global__ void store_step_kernel(const double2* __restrict__ x, double* __restrict__ phi, double2* __restrict__ xr,
                                  int64_t M) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= M) return;
  phi[i] = x[i].x;
  xr[i] = make_double2(x[i].x, 0.0);
}

__global__ void copy_column_kernel(const double2* __restrict__ xh1, double2* __restrict__ XH, int C, int HS, int col,
                                   int p) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= (int64_t)C * p) return;
  const int64_t c = i / p, mu = i - c * p;
  XH[(c * HS + col) * p + mu] = xh1[i];
}

inline unsigned nb(int64_t n) { return (unsigned)((n + 255) / 256); }

ConvArgs conv_args(Op& op) {
  Tree& t = *op.tree;
  ConvArgs a{};
  a.M = t.M; a.L = op.L; a.p = t.p;
  a.far_ptr = t.d_far_ptr.p; a.far_sorted = t.d_far_sorted.p; a.far_c = t.d_far_c.p; a.rank = op.d_rank.p;
  a.zoff = op.d_zoff.p; a.fsoff = op.d_fsoff.p; a.Df = (const double2*)op.d_Df.p; a.fS = (const double2*)op.d_fS.p;
  a.leaves = t.d_leaves.p; a.nb_ptr = t.d_nb_ptr.p; a.nb_sorted = t.d_nb_sorted.p; a.near_c = t.d_near_c.p;
  a.near_r = t.d_near_r.p;
  a.cbegin = t.d_begin.p; a.cend = t.d_end.p; a.nrank = op.d_nrank.p; a.nzoff = op.d_nzoff.p; a.nsoff = op.d_nsoff.p;
  a.Dn = (const double2*)op.d_Dn.p; a.nS = (const double2*)op.d_nS.p;
  return a;
}

// y (input order, [ncols][M]) = sum_{k<=min(n,kmax)} V^_{n-k} (history), n = n0 .. n0+ncols-1
bem_status conv_launch(Op& op, const double2* XH, const double2* Q, int HS, int n0, int ncols, int kmax, double2* yhat,
                       double2* ycn, double2* y, cudaStream_t st) {
  Tree& t = *op.tree;
  ConvArgs a = conv_args(op);
  a.HS = HS; a.n0 = n0; a.ncols = ncols; a.kmax = kmax; a.XH = XH; a.Q = Q; a.yhat = yhat; a.ycn = ycn;
  const int nfar = (int)t.far_r.size(), nnear = (int)t.near_r.size();
  const size_t need = std::max((size_t)nfar * ncols * t.p, (size_t)nnear * ncols * t.max_leaf) * 2;
  if (op.d_conv_part.n < need) BEM_CK(op.d_conv_part.alloc(need));
  double2* part = (double2*)op.d_conv_part.p;
  if (nfar > 0) {
    BEM_CK(cudaMemsetAsync(yhat, 0, sizeof(double2) * (size_t)t.C * ncols * t.p, st));
    const size_t smf = sizeof(double2) * 2 * kTC * t.p;
    BEM_CK(cudaFuncSetAttribute(conv_block_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smf));
    conv_block_kernel<false><<<dim3((unsigned)nfar, (unsigned)ncols), kConvThreads, smf, st>>>(a, part, t.p);
    BEM_CK(cudaGetLastError());
    far_reduce_kernel<<<dim3((unsigned)t.C, (unsigned)ncols), 128, 0, st>>>(t.d_far_ptr.p, t.d_far_sorted.p, part,
                                                                             yhat, ncols, t.p);
    BEM_CK(cudaGetLastError());
  }
  const size_t smn = sizeof(double2) * 2 * kTC * t.max_leaf;
  BEM_CK(cudaFuncSetAttribute(conv_block_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smn));
  conv_block_kernel<true><<<dim3((unsigned)nnear, (unsigned)ncols), kConvThreads, smn, st>>>(a, part, t.max_leaf);
  BEM_CK(cudaGetLastError());
  near_reduce_kernel<<<dim3((unsigned)t.n_leaves, (unsigned)ncols), 64, 0, st>>>(
      t.d_leaves.p, t.d_nb_ptr.p, t.d_nb_sorted.p, t.d_begin.p, t.d_end.p, part, ycn, t.M, ncols, t.max_leaf);
  BEM_CK(cudaGetLastError());
  return h2_down_scatter(op, yhat, ycn, y, ncols, st);
}

bem_status check_op(Op& op, const char* who) {
  if (op.mode != BEM_MODE_COMBINED) {
    set_error("%s: the operator must be assembled with BEM_MODE_COMBINED", who);
    return BEM_ESTATE;
  }
  BEM_REQ(op.n_local == op.L, "%s: the operator must hold all L frequencies", who);
  for (int t = 0; t < op.n_local; ++t) BEM_REQ(op.local_l[t] == t, "%s: local_l must be 0..L-1 in order", who);
  return BEM_OK;
}

}  // namespace
}  // namespace bem

using namespace bem;

extern "C" bem_status bem_mot_prepare(bem_op oh, double R, void* cuda_stream) {
  BEM_REQ(oh, "bem_mot_prepare: NULL op");
  BEM_REQ(R > 0.0 && R < 1.0, "bem_mot_prepare: R must lie in (0,1)");
  Op& op = oh->o;
  bem_status rs = check_op(op, "bem_mot_prepare");
  if (rs != BEM_OK) return rs;
  Tree& t = *op.tree;
  DeviceGuard dg(t.device);
  cudaStream_t st = (cudaStream_t)cuda_stream;
  const int L = op.L, p = t.p;
  int64_t rows_f = 0, rows_n = 0;
  for (int r : op.ranks) rows_f += r;
  for (int r : op.nranks) rows_n += r;
  BEM_CK(op.d_Df.alloc((size_t)std::max<int64_t>(rows_f, 1) * L * 2));
  BEM_CK(op.d_Dn.alloc((size_t)std::max<int64_t>(rows_n, 1) * L * 2));
  if (rows_f > 0)
    dhat_kernel<<<nb(rows_f * L), 256, 0, st>>>((const double2*)op.d_Z.p, (double2*)op.d_Df.p, rows_f, L, R);
  if (rows_n > 0)
    dhat_kernel<<<nb(rows_n * L), 256, 0, st>>>((const double2*)op.d_nZ.p, (double2*)op.d_Dn.p, rows_n, L, R);
  BEM_CK(cudaGetLastError());
  const int nfar = (int)t.far_r.size();
  std::vector<int64_t> fsoff(std::max(nfar, 1), 0);
  int64_t tot = 0;
  for (int b = 0; b < nfar; ++b) { fsoff[b] = tot; tot += (int64_t)op.ranks[b] * p * p; }
  BEM_CK(op.d_fsoff.upload(fsoff));
  BEM_CK(op.d_fS.alloc((size_t)std::max<int64_t>(tot, 1) * 2));
  if (nfar > 0) {
    far_slice_kernel<<<nfar, 256, 0, st>>>(t.d_far_r.p, t.d_far_c.p, t.d_xi.p, (const double2*)op.d_s.p, op.d_rank.p,
                                           op.d_pivk.p, op.rcap, op.d_fsoff.p, (double2*)op.d_fS.p, t.m, p);
    BEM_CK(cudaGetLastError());
  }
  // Re V^_0 blocks
  BEM_CK(op.d_g0f.alloc((size_t)std::max(nfar, 1) * p * p));
  if (nfar > 0) {
    g0_far_build_kernel<<<nfar, 256, 0, st>>>((const double2*)op.d_fS.p, op.d_fsoff.p, (const double2*)op.d_Df.p,
                                              op.d_zoff.p, op.d_rank.p, L, p, op.d_g0f.p);
    BEM_CK(cudaGetLastError());
  }
  const int nnear = (int)t.near_r.size();
  std::vector<int64_t> goff(std::max(nnear, 1), 0);
  int64_t gt = 0;
  for (int b = 0; b < nnear; ++b) {
    goff[b] = gt;
    gt += (int64_t)(t.end[t.near_r[b]] - t.begin[t.near_r[b]]) * (t.end[t.near_c[b]] - t.begin[t.near_c[b]]);
  }
  BEM_CK(op.d_g0noff.upload(goff));
  BEM_CK(op.d_g0n.alloc((size_t)std::max<int64_t>(gt, 1)));
  if (nnear > 0) {
    g0_near_build_kernel<<<nnear, 256, 0, st>>>((const double2*)op.d_nS.p, op.d_nsoff.p, (const double2*)op.d_Dn.p,
                                                op.d_nzoff.p, op.d_nrank.p, t.d_near_r.p, t.d_near_c.p, t.d_begin.p,
                                                t.d_end.p, op.d_g0noff.p, L, op.d_g0n.p);
    BEM_CK(cudaGetLastError());
  }
  BEM_CK(cudaStreamSynchronize(st));
  op.mot_ready = true;
  op.mot_R = R;
  return BEM_OK;
}

extern "C" bem_status bem_conv_time(bem_op oh, const bem_c128* q, bem_c128* y, int32_t kmax, void* cuda_stream) {
  BEM_REQ(oh && q && y && q != y, "bem_conv_time: NULL or aliased argument");
  Op& op = oh->o;
  if (!op.mot_ready) {
    set_error("bem_conv_time: call bem_mot_prepare first");
    return BEM_ESTATE;
  }
  Tree& t = *op.tree;
  DeviceGuard dg(t.device);
  cudaStream_t st = (cudaStream_t)cuda_stream;
  const int L = op.L;
  DBuf<double> Qc, XH, yh, ycn;
  BEM_CK(Qc.alloc((size_t)L * t.M * 2)); BEM_CK(XH.alloc((size_t)t.C * L * t.p * 2));
  BEM_CK(yh.alloc((size_t)t.C * L * t.p * 2)); BEM_CK(ycn.alloc((size_t)L * t.M * 2));
  bem_status rs = h2_gather(op, (const double2*)q, (double2*)Qc.p, L, st);
  if (rs == BEM_OK && !t.far_r.empty()) rs = h2_up(op, (const double2*)Qc.p, (double2*)XH.p, L, st);
  if (rs == BEM_OK)
    rs = conv_launch(op, (const double2*)XH.p, (const double2*)Qc.p, L, 0, L, std::min<int>(kmax, L - 1),
                     (double2*)yh.p, (double2*)ycn.p, (double2*)y, st);
  if (rs != BEM_OK) return rs;
  BEM_CK(cudaStreamSynchronize(st));
  return BEM_OK;
}

extern "C" bem_status cqm_mot_solve(bem_op oh, const double* g_time, double* phi_time, double tol, int32_t restart,
                                    int32_t max_iter, void* cuda_stream, bem_solve_stats* stats) {
  BEM_REQ(oh && g_time && phi_time, "cqm_mot_solve: NULL argument");
  BEM_REQ(tol > 0.0 && restart >= 1 && max_iter >= 1, "cqm_mot_solve: bad tol/restart/max_iter");
  Op& op = oh->o;
  if (!op.mot_ready) {
    set_error("cqm_mot_solve: call bem_mot_prepare first");
    return BEM_ESTATE;
  }
  Tree& t = *op.tree;
  DeviceGuard dg(t.device);
  cudaStream_t st = (cudaStream_t)cuda_stream;
  const int L = op.L, p = t.p, C = t.C;
  const int64_t M = t.M;
  const bool far = !t.far_r.empty();
  DBuf<double> Q, XH, xc1, xh1, yh1, ycn1, r1, b1, x1, xr1;
  BEM_CK(Q.alloc((size_t)L * M * 2)); BEM_CK(XH.alloc((size_t)C * L * p * 2));
  BEM_CK(xc1.alloc((size_t)M * 2)); BEM_CK(xh1.alloc((size_t)C * p * 2)); BEM_CK(yh1.alloc((size_t)C * p * 2));
  BEM_CK(ycn1.alloc((size_t)M * 2)); BEM_CK(r1.alloc((size_t)M * 2)); BEM_CK(b1.alloc((size_t)M * 2));
  BEM_CK(x1.alloc((size_t)M * 2)); BEM_CK(xr1.alloc((size_t)M * 2));
  BEM_CK(cudaMemsetAsync(Q.p, 0, sizeof(double) * Q.n, st));
  BEM_CK(cudaMemsetAsync(XH.p, 0, sizeof(double) * XH.n, st));
  // w = Re V^_0 x (one column, input order)
  auto v0 = [&](const double* x, double* w) -> bem_status {
    bem_status s = h2_gather(op, (const double2*)x, (double2*)xc1.p, 1, st);
    if (s != BEM_OK) return s;
    const int nfar = (int)t.far_r.size(), nnear = (int)t.near_r.size();
    const size_t need = (size_t)std::max(nfar * p, nnear * t.max_leaf) * 2;
    if (op.d_conv_part.n < need) BEM_CK(op.d_conv_part.alloc(need));
    double2* part = (double2*)op.d_conv_part.p;
    if (far) {
      s = h2_up(op, (const double2*)xc1.p, (double2*)xh1.p, 1, st);
      if (s != BEM_OK) return s;
      BEM_CK(cudaMemsetAsync(yh1.p, 0, sizeof(double2) * (size_t)C * p, st));
      g0_block_kernel<false><<<nfar, 128, sizeof(double2) * p, st>>>(t.d_far_r.p, t.d_far_c.p, t.d_begin.p,
                                                                     t.d_end.p, nullptr, op.d_g0f.p,
                                                                     (const double2*)xh1.p, part, p, p);
      far_reduce_kernel<<<dim3((unsigned)C, 1), 128, 0, st>>>(t.d_far_ptr.p, t.d_far_sorted.p, part,
                                                               (double2*)yh1.p, 1, p);
      BEM_CK(cudaGetLastError());
    }
    g0_block_kernel<true><<<nnear, 128, sizeof(double2) * t.max_leaf, st>>>(
        t.d_near_r.p, t.d_near_c.p, t.d_begin.p, t.d_end.p, op.d_g0noff.p, op.d_g0n.p, (const double2*)xc1.p, part,
        p, t.max_leaf);
    near_reduce_kernel<<<dim3((unsigned)t.n_leaves, 1), 64, 0, st>>>(t.d_leaves.p, t.d_nb_ptr.p, t.d_nb_sorted.p,
                                                                     t.d_begin.p, t.d_end.p, part, (double2*)ycn1.p,
                                                                     M, 1, t.max_leaf);
    BEM_CK(cudaGetLastError());
    return h2_down_scatter(op, (double2*)yh1.p, (const double2*)ycn1.p, (double2*)w, 1, st);
  };
  GmresWs ws;
  int imax = 0, isum = 0;
  double rmax = 0.0;
  int nunc = 0;
  for (int n = 0; n < L; ++n) {
    bem_status rs = BEM_OK;
    if (n > 0)
      rs = conv_launch(op, (const double2*)XH.p, (const double2*)Q.p, L, n, 1, n - 1, (double2*)yh1.p,
                       (double2*)ycn1.p, (double2*)r1.p, st);
    if (rs != BEM_OK) return rs;
    rhs_kernel<<<nb(M), 256, 0, st>>>(g_time + (int64_t)n * M, (const double2*)r1.p, (double2*)b1.p, M, n > 0);
    BEM_CK(cudaGetLastError());
    std::vector<int> hit;
    std::vector<double> hrel;
    rs = gmres_fn(M, 1, v0, (const double2*)b1.p, (double2*)x1.p, tol, restart, max_iter, st, hit, hrel, ws);
    if (rs != BEM_OK) return rs;
    isum += hit[0];
    imax = std::max(imax, hit[0]);
    rmax = std::max(rmax, hrel[0]);
    if (hrel[0] > tol) ++nunc;
    // q_n: output (input order, real), history (cluster order) and its cluster-basis coefficients
    store_step_kernel<<<nb(M), 256, 0, st>>>((const double2*)x1.p, phi_time + (int64_t)n * M, (double2*)xr1.p, M);
    BEM_CK(cudaGetLastError());
    rs = h2_gather(op, (const double2*)xr1.p, (double2*)Q.p + (int64_t)n * M, 1, st);
    if (rs == BEM_OK && far) {
      rs = h2_up(op, (const double2*)Q.p + (int64_t)n * M, (double2*)xh1.p, 1, st);
      if (rs == BEM_OK) {
        copy_column_kernel<<<nb((int64_t)C * p), 256, 0, st>>>((const double2*)xh1.p, (double2*)XH.p, C, L, n, p);
        BEM_CK(cudaGetLastError());
      }
    }
    if (rs != BEM_OK) return rs;
  }
  BEM_CK(cudaStreamSynchronize(st));
  if (stats) {
    stats->iters_max = imax; stats->iters_sum = isum; stats->n_unconverged = nunc;
    stats->resid_max = rmax; stats->imag_rel_max = 0.0;
  }
  if (nunc > 0) {
    set_error("cqm_mot_solve: %d time steps did not converge within max_iter=%d", nunc, max_iter);
    return BEM_ENOCONV;
  }
  return BEM_OK;
}
