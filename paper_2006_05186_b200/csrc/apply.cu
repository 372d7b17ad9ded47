// bem_apply_multifreq: y_t = V(s_{l_t}) x_t for all local frequencies at once
// (eq:lrfinal P:1404-1410; H^2 matvec P:1106-1107 / P:938-944):
//   a2 gather x into cluster order
//   a3 K1  near field, evaluated on the fly (collocation + 7-pt rule, self
//          panels analytic 1/r + rule on (e^{-sr}-1)/r), conjugate pairs
//          (l, L-l) share one exp/sincos
//   a4 K2^ upward pass: leaves xhat = W^T x, parents xhat = sum E^T xhat_son
//   a5 K3  coupling: yhat_r = sum_{b=(r,c)} sum_l Z_b[l,t] S_b(s_{k_l}) xhat_c
//          with the pivot slices S_b(s_{k_l}) regenerated from the kernel
//   a6 K2v downward pass: yhat_son += E yhat_parent; leaves y += U yhat
//   a7 scatter to input order
#include <algorithm>
#include <cmath>

#include "common.cuh"
#include "near_common.cuh"

namespace bem {
namespace {

// ------------------------------------------------------------------ gather
__global__ void gather_kernel(const double2* __restrict__ x, double2* __restrict__ xc, const int32_t* __restrict__ perm,
                              int64_t M, int nl) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= M * nl) return;
  const int64_t t = i / M, k = i - t * M;
  xc[i] = x[t * M + perm[k]];
}

// ------------------------------------------------------------------- K2
constexpr int kPassThreads = 256;
constexpr int kPassT = 16;  // frequencies per CTA

__global__ void __launch_bounds__(kPassThreads) up_leaf_kernel(const int32_t* __restrict__ leaves,
                                                               const int32_t* __restrict__ cb,
                                                               const int32_t* __restrict__ ce,
                                                               const double* __restrict__ W,
                                                               const double2* __restrict__ xc,
                                                               double2* __restrict__ xhat, int64_t M, int nl, int p) {
  const int c = leaves[blockIdx.x];
  const int b = cb[c], e = ce[c];
  const int t0 = blockIdx.y * kPassT;
  for (int idx = threadIdx.x; idx < kPassT * p; idx += blockDim.x) {
    const int t = t0 + idx / p, nu = idx % p;
    if (t >= nl) break;
    double2 acc = make_double2(0.0, 0.0);
    const double2* xt = xc + (int64_t)t * M;
    for (int k = b; k < e; ++k) {
      const double w = W[(int64_t)k * p + nu];
      const double2 v = xt[k];
      acc.x = fma(w, v.x, acc.x);
      acc.y = fma(w, v.y, acc.y);
    }
    xhat[((int64_t)c * nl + t) * p + nu] = acc;
  }
}

__global__ void __launch_bounds__(kPassThreads) up_transfer_kernel(const int32_t* __restrict__ list,
                                                                   const int32_t* __restrict__ son0,
                                                                   const int32_t* __restrict__ son1,
                                                                   const double* __restrict__ E,
                                                                   double2* __restrict__ xhat, int nl, int p) {
  const int c = list[blockIdx.x];
  const int s0 = son0[c], s1 = son1[c];
  const int t0 = blockIdx.y * kPassT;
  for (int idx = threadIdx.x; idx < kPassT * p; idx += blockDim.x) {
    const int t = t0 + idx / p, mu = idx % p;
    if (t >= nl) break;
    double2 acc = make_double2(0.0, 0.0);
    for (int sidx = 0; sidx < 2; ++sidx) {
      const int sc = sidx ? s1 : s0;
      const double* Es = E + (int64_t)sc * p * p;
      const double2* xs = xhat + ((int64_t)sc * nl + t) * p;
      for (int lam = 0; lam < p; ++lam) {
        const double w = Es[lam * p + mu];
        acc.x = fma(w, xs[lam].x, acc.x);
        acc.y = fma(w, xs[lam].y, acc.y);
      }
    }
    xhat[((int64_t)c * nl + t) * p + mu] = acc;
  }
}

__global__ void __launch_bounds__(kPassThreads) down_transfer_kernel(const int32_t* __restrict__ list,
                                                                     const int32_t* __restrict__ son0,
                                                                     const int32_t* __restrict__ son1,
                                                                     const double* __restrict__ E,
                                                                     double2* __restrict__ yhat, int nl, int p) {
  const int c = list[blockIdx.x];
  const int t0 = blockIdx.y * kPassT;
  for (int idx = threadIdx.x; idx < 2 * kPassT * p; idx += blockDim.x) {
    const int sidx = idx / (kPassT * p);
    const int rem = idx - sidx * kPassT * p;
    const int t = t0 + rem / p, lam = rem % p;
    if (t >= nl) continue;
    const int sc = sidx ? son1[c] : son0[c];
    const double* Es = E + (int64_t)sc * p * p + lam;  // E^T[sc][mu][lam]: coalesced over lam
    const double2* yp = yhat + ((int64_t)c * nl + t) * p;
    double2 acc = yhat[((int64_t)sc * nl + t) * p + lam];
    for (int mu = 0; mu < p; ++mu) {
      const double e = Es[(int64_t)mu * p];
      acc.x = fma(e, yp[mu].x, acc.x);
      acc.y = fma(e, yp[mu].y, acc.y);
    }
    yhat[((int64_t)sc * nl + t) * p + lam] = acc;
  }
}

__global__ void __launch_bounds__(kPassThreads) down_leaf_kernel(const int32_t* __restrict__ leaves,
                                                                 const int32_t* __restrict__ cb,
                                                                 const int32_t* __restrict__ ce,
                                                                 const double* __restrict__ U,
                                                                 const double2* __restrict__ yhat,
                                                                 const double2* __restrict__ yc,
                                                                 const int32_t* __restrict__ perm,
                                                                 double2* __restrict__ y, int64_t M, int nl, int p,
                                                                 int has_far, const double2* __restrict__ xc,
                                                                 double alpha) {
  const int c = leaves[blockIdx.x];
  const int b = cb[c], e = ce[c], n = e - b;
  const int t0 = blockIdx.y * kPassT;
  for (int idx = threadIdx.x; idx < kPassT * n; idx += blockDim.x) {
    const int t = t0 + idx / n, k = b + idx % n;
    if (t >= nl) break;
    double2 acc = yc[(int64_t)t * M + k];
    if (has_far) {
      const double2* yh = yhat + ((int64_t)c * nl + t) * p;
      const double* Uk = U + k;  // U^T[mu][k]: coalesced over k
      for (int mu = 0; mu < p; ++mu) {
        const double u = Uk[(int64_t)mu * M];
        acc.x = fma(u, yh[mu].x, acc.x);
        acc.y = fma(u, yh[mu].y, acc.y);
      }
    }
    if (alpha != 0.0) {  // (alpha I + K) x for the double layer
      const double2 xv = xc[(int64_t)t * M + k];
      acc.x = fma(alpha, xv.x, acc.x);
      acc.y = fma(alpha, xv.y, acc.y);
    }
    y[(int64_t)t * M + perm[k]] = acc;
  }
}

// Shared-memory staged variants (used when the tiles fit): the basis / transfer
// matrix and the coefficient tile are loaded once with coalesced loads, then every
// thread's dot product runs from shared memory (the unstaged kernels above chain
// ~2p dependent global loads per output; r01: K2 at 6 % of its roofline).
__global__ void __launch_bounds__(kPassThreads) up_leaf_s_kernel(const int32_t* __restrict__ leaves,
                                                                 const int32_t* __restrict__ cb,
                                                                 const int32_t* __restrict__ ce,
                                                                 const double* __restrict__ W,
                                                                 const double2* __restrict__ xc,
                                                                 double2* __restrict__ xhat, int64_t M, int nl, int p) {
  extern __shared__ double2 smx[];
  const int c = leaves[blockIdx.x];
  const int b = cb[c], n = ce[c] - b;
  const int t0 = blockIdx.y * kPassT;
  double2* xs = smx;                      // kPassT x n
  double* Ws = (double*)(smx + kPassT * n);  // n x p
  for (int idx = threadIdx.x; idx < n * p; idx += blockDim.x) Ws[idx] = W[(int64_t)b * p + idx];
  for (int idx = threadIdx.x; idx < kPassT * n; idx += blockDim.x) {
    const int tl = idx / n, k = idx - tl * n;
    xs[idx] = t0 + tl < nl ? xc[(int64_t)(t0 + tl) * M + b + k] : make_double2(0.0, 0.0);
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < kPassT * p; idx += blockDim.x) {
    const int tl = idx / p, nu = idx - tl * p;
    if (t0 + tl >= nl) break;
    double2 acc = make_double2(0.0, 0.0);
    for (int k = 0; k < n; ++k) {
      const double w = Ws[k * p + nu];
      const double2 v = xs[tl * n + k];
      acc.x = fma(w, v.x, acc.x);
      acc.y = fma(w, v.y, acc.y);
    }
    xhat[((int64_t)c * nl + t0 + tl) * p + nu] = acc;
  }
}

__global__ void __launch_bounds__(kPassThreads) up_transfer_s_kernel(const int32_t* __restrict__ list,
                                                                     const int32_t* __restrict__ son0,
                                                                     const int32_t* __restrict__ son1,
                                                                     const double* __restrict__ E,
                                                                     double2* __restrict__ xhat, int nl, int p) {
  extern __shared__ double2 smx[];
  const int c = list[blockIdx.x];
  const int sons[2] = {son0[c], son1[c]};
  const int t0 = blockIdx.y * kPassT;
  double2* xs = smx;                           // 2 x kPassT x p
  double* Es = (double*)(smx + 2 * kPassT * p);  // 2 x p x p
  for (int idx = threadIdx.x; idx < 2 * p * p; idx += blockDim.x) {
    const int sidx = idx / (p * p), e = idx - sidx * p * p;
    Es[idx] = E[(int64_t)sons[sidx] * p * p + e];
  }
  for (int idx = threadIdx.x; idx < 2 * kPassT * p; idx += blockDim.x) {
    const int sidx = idx / (kPassT * p), e = idx - sidx * kPassT * p;
    const int tl = e / p;
    xs[idx] = t0 + tl < nl ? xhat[((int64_t)sons[sidx] * nl + t0) * p + e] : make_double2(0.0, 0.0);
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < kPassT * p; idx += blockDim.x) {
    const int tl = idx / p, mu = idx - tl * p;
    if (t0 + tl >= nl) break;
    double2 acc = make_double2(0.0, 0.0);
    for (int sidx = 0; sidx < 2; ++sidx) {
      const double* Em = Es + sidx * p * p + mu;
      const double2* x = xs + (sidx * kPassT + tl) * p;
      for (int lam = 0; lam < p; ++lam) {
        const double w = Em[lam * p];
        acc.x = fma(w, x[lam].x, acc.x);
        acc.y = fma(w, x[lam].y, acc.y);
      }
    }
    xhat[((int64_t)c * nl + t0 + tl) * p + mu] = acc;
  }
}

__global__ void __launch_bounds__(kPassThreads) down_transfer_s_kernel(const int32_t* __restrict__ list,
                                                                       const int32_t* __restrict__ son0,
                                                                       const int32_t* __restrict__ son1,
                                                                       const double* __restrict__ ET,
                                                                       double2* __restrict__ yhat, int nl, int p) {
  extern __shared__ double2 smx[];
  const int c = list[blockIdx.x];
  const int sons[2] = {son0[c], son1[c]};
  const int t0 = blockIdx.y * kPassT;
  double2* ys = smx;                      // kPassT x p (parent)
  double* Es = (double*)(smx + kPassT * p);  // 2 x p x p, E^T[son][mu][lam]
  for (int idx = threadIdx.x; idx < 2 * p * p; idx += blockDim.x) {
    const int sidx = idx / (p * p), e = idx - sidx * p * p;
    Es[idx] = ET[(int64_t)sons[sidx] * p * p + e];
  }
  for (int idx = threadIdx.x; idx < kPassT * p; idx += blockDim.x) {
    const int tl = idx / p;
    ys[idx] = t0 + tl < nl ? yhat[((int64_t)c * nl + t0) * p + idx] : make_double2(0.0, 0.0);
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < 2 * kPassT * p; idx += blockDim.x) {
    const int sidx = idx / (kPassT * p), e = idx - sidx * kPassT * p;
    const int tl = e / p, lam = e - tl * p;
    if (t0 + tl >= nl) continue;
    const int sc = sons[sidx];
    const double* Em = Es + sidx * p * p + lam;
    const double2* yp = ys + tl * p;
    double2 acc = yhat[((int64_t)sc * nl + t0 + tl) * p + lam];
    for (int mu = 0; mu < p; ++mu) {
      const double w = Em[mu * p];
      acc.x = fma(w, yp[mu].x, acc.x);
      acc.y = fma(w, yp[mu].y, acc.y);
    }
    yhat[((int64_t)sc * nl + t0 + tl) * p + lam] = acc;
  }
}

__global__ void __launch_bounds__(kPassThreads) down_leaf_s_kernel(const int32_t* __restrict__ leaves,
                                                                   const int32_t* __restrict__ cb,
                                                                   const int32_t* __restrict__ ce,
                                                                   const double* __restrict__ UT,
                                                                   const double2* __restrict__ yhat,
                                                                   const double2* __restrict__ yc,
                                                                   const int32_t* __restrict__ perm,
                                                                   double2* __restrict__ y, int64_t M, int nl, int p,
                                                                   const double2* __restrict__ xc, double alpha) {
  extern __shared__ double2 smx[];
  const int c = leaves[blockIdx.x];
  const int b = cb[c], n = ce[c] - b;
  const int t0 = blockIdx.y * kPassT;
  double2* ys = smx;                      // kPassT x p
  double* Us = (double*)(smx + kPassT * p);  // p x n (U^T rows of the leaf's panels)
  for (int idx = threadIdx.x; idx < p * n; idx += blockDim.x) {
    const int mu = idx / n, k = idx - mu * n;
    Us[idx] = UT[(int64_t)mu * M + b + k];
  }
  for (int idx = threadIdx.x; idx < kPassT * p; idx += blockDim.x) {
    const int tl = idx / p;
    ys[idx] = t0 + tl < nl ? yhat[((int64_t)c * nl + t0) * p + idx] : make_double2(0.0, 0.0);
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < kPassT * n; idx += blockDim.x) {
    const int tl = idx / n, k = idx - tl * n;
    const int t = t0 + tl;
    if (t >= nl) break;
    double2 acc = yc[(int64_t)t * M + b + k];
    const double2* yh = ys + tl * p;
    for (int mu = 0; mu < p; ++mu) {
      const double u = Us[mu * n + k];
      acc.x = fma(u, yh[mu].x, acc.x);
      acc.y = fma(u, yh[mu].y, acc.y);
    }
    if (alpha != 0.0) {
      const double2 xv = xc[(int64_t)t * M + b + k];
      acc.x = fma(alpha, xv.x, acc.x);
      acc.y = fma(alpha, xv.y, acc.y);
    }
    y[(int64_t)t * M + perm[b + k]] = acc;
  }
}

// Leaf products on the FP64 tensor cores (mma.sync m8n8k4 f64, SASS DMMA): with the 16
// frequencies of a tile as 32 interleaved real columns,
//   up:   xhat_c[t][nu] = sum_k W[k][nu] x[t][k]         = (W^T)(p x n) . X(n x 32)
//   down: y[t][k]  = yc[t][k] + sum_mu U[k][mu] yhat[t][mu] = U(n x p) . Y(p x 32)
// A fragments from the basis tile, B fragments from the transposed coefficient tile
// (both in shared memory, row strides = 8 mod 16 doubles: two wavefronts per fragment
// load); each warp owns 8 x 8 output tiles, K = n (up) / p (down) in steps of 4.
constexpr int kLeafT = 16;  // frequencies per CTA (32 real columns = 4 DMMA column tiles)

__device__ __forceinline__ void dmma_k2(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

__host__ __device__ __forceinline__ int pad8(int n) { return (n + 15) / 16 * 16 + 8; }  // row stride = 8 (mod 16)

__global__ void __launch_bounds__(kPassThreads) up_leaf_d_kernel(const int32_t* __restrict__ leaves,
                                                                 const int32_t* __restrict__ cb,
                                                                 const int32_t* __restrict__ ce,
                                                                 const double* __restrict__ W,
                                                                 const double2* __restrict__ xc,
                                                                 double2* __restrict__ xhat, int64_t M, int nl, int p) {
  extern __shared__ double smd[];
  const int c = leaves[blockIdx.x];
  const int b = cb[c], n = ce[c] - b;
  const int n4 = (n + 3) & ~3;
  const int t0 = blockIdx.y * kLeafT;
  const int nt = min(kLeafT, nl - t0);
  const int WS = pad8(p), XS = pad8(2 * kLeafT);
  double* Ws = smd;              // [n4][WS]: W[k][nu]
  double* Xs = Ws + n4 * WS;     // [n4][XS]: x[t][k] as Xs[k][2t + re/im]
  for (int i = threadIdx.x; i < n4 * p; i += blockDim.x) {
    const int k = i / p, nu = i - k * p;
    Ws[k * WS + nu] = k < n ? W[(int64_t)(b + k) * p + nu] : 0.0;
  }
  for (int i = threadIdx.x; i < n4 * kLeafT; i += blockDim.x) {
    const int tl = i / n4, k = i - tl * n4;  // consecutive threads: consecutive panels (coalesced)
    const double2 v = (k < n && tl < nt) ? xc[(int64_t)(t0 + tl) * M + b + k] : make_double2(0.0, 0.0);
    BEM_DASSERT(k < n4 && 2 * tl + 1 < XS);
    Xs[k * XS + 2 * tl] = v.x;
    Xs[k * XS + 2 * tl + 1] = v.y;
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, q = lane & 3;
  const int nvt = (p + 7) / 8;
  for (int tile = warp; tile < nvt * 4; tile += blockDim.x >> 5) {
    const int v0 = (tile >> 2) * 8, n0 = (tile & 3) * 8;
    const int nu = v0 + g;
    double c0 = 0.0, c1 = 0.0;
    for (int k0 = 0; k0 < n4; k0 += 4) {
      const double a = nu < p ? Ws[(k0 + q) * WS + nu] : 0.0;
      const double bb = Xs[(k0 + q) * XS + n0 + g];
      dmma_k2(c0, c1, a, bb);
    }
    const int tl = (n0 >> 1) + q;  // columns n0 + 2q, n0 + 2q + 1 = (re, im) of frequency tl
    if (nu < p && tl < nt) xhat[((int64_t)c * nl + t0 + tl) * p + nu] = make_double2(c0, c1);
  }
}

__global__ void __launch_bounds__(kPassThreads) down_leaf_d_kernel(const int32_t* __restrict__ leaves,
                                                                   const int32_t* __restrict__ cb,
                                                                   const int32_t* __restrict__ ce,
                                                                   const double* __restrict__ U,
                                                                   const double2* __restrict__ yhat,
                                                                   const double2* __restrict__ yc,
                                                                   const int32_t* __restrict__ perm,
                                                                   double2* __restrict__ y, int64_t M, int nl, int p,
                                                                   const double2* __restrict__ xc, double alpha) {
  extern __shared__ double smd[];
  const int c = leaves[blockIdx.x];
  const int b = cb[c], n = ce[c] - b;
  const int p4 = (p + 3) & ~3;
  const int t0 = blockIdx.y * kLeafT;
  const int nt = min(kLeafT, nl - t0);
  const int US = pad8(p4), YS = pad8(2 * kLeafT);
  const int n8 = (n + 7) & ~7;
  double* Us = smd;              // [n8][US]: U[k][mu]
  double* Ys = Us + n8 * US;     // [p4][YS]: yhat[t][mu] as Ys[mu][2t + re/im]
  for (int i = threadIdx.x; i < n8 * p4; i += blockDim.x) {
    const int k = i / p4, mu = i - k * p4;
    Us[k * US + mu] = (k < n && mu < p) ? U[(int64_t)(b + k) * p + mu] : 0.0;
  }
  for (int i = threadIdx.x; i < kLeafT * p4; i += blockDim.x) {
    const int tl = i / p4, mu = i - tl * p4;
    const double2 v = (mu < p && tl < nt) ? yhat[((int64_t)c * nl + t0 + tl) * p + mu] : make_double2(0.0, 0.0);
    BEM_DASSERT(mu < p4 && 2 * tl + 1 < YS);
    Ys[mu * YS + 2 * tl] = v.x;
    Ys[mu * YS + 2 * tl + 1] = v.y;
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, q = lane & 3;
  const int nkt = n8 / 8;
  for (int tile = warp; tile < nkt * 4; tile += blockDim.x >> 5) {
    const int k0r = (tile >> 2) * 8, n0 = (tile & 3) * 8;
    double c0 = 0.0, c1 = 0.0;
    for (int m0 = 0; m0 < p4; m0 += 4) {
      const double a = Us[(k0r + g) * US + m0 + q];
      const double bb = Ys[(m0 + q) * YS + n0 + g];
      dmma_k2(c0, c1, a, bb);
    }
    const int k = k0r + g, tl = (n0 >> 1) + q;
    if (k < n && tl < nt) {
      const int64_t row = (int64_t)(t0 + tl) * M;
      BEM_DASSERT(b + k < M && perm[b + k] >= 0 && perm[b + k] < M);
      double2 acc = yc[row + b + k];
      acc.x += c0;
      acc.y += c1;
      if (alpha != 0.0) {
        const double2 xv = xc[row + b + k];
        acc.x = fma(alpha, xv.x, acc.x);
        acc.y = fma(alpha, xv.y, acc.y);
      }
      y[row + perm[b + k]] = acc;
    }
  }
}

// Pipelined leaf products: CTA = (leaf, chunk of FT frequencies).  The leaf's basis tile
// is staged once and reused for every 16-frequency sub-tile of the chunk; the next
// sub-tile's coefficients stream in (cp.async, one 16-byte complex per copy, directly
// into the transposed [k][2t + re/im] layout) while the current one is contracted on the
// tensor cores.  r2: the one-shot kernels (one sub-tile per CTA) spent most of their time
// waiting on the staging loads.
__global__ void __launch_bounds__(kPassThreads) up_leaf_p_kernel(const int32_t* __restrict__ leaves,
                                                                 const int32_t* __restrict__ cb,
                                                                 const int32_t* __restrict__ ce,
                                                                 const double* __restrict__ W,
                                                                 const double2* __restrict__ xc,
                                                                 double2* __restrict__ xhat, int64_t M, int nl, int p,
                                                                 int FT) {
  extern __shared__ double smd[];
  const int c = leaves[blockIdx.x];
  const int b = cb[c], n = ce[c] - b;
  const int n4 = (n + 3) & ~3;
  const int f0 = blockIdx.y * FT, f1 = min(nl, f0 + FT);
  const int WS = pad8(p), XS = pad8(2 * kLeafT);
  double* Ws = smd;                       // [n4][WS]: W[k][nu]
  double* X0 = Ws + n4 * WS;              // 2 x [n4][XS]: x[t][k] as X[k][2t + re/im]
  const size_t xsz = (size_t)n4 * XS;
  for (int i = threadIdx.x; i < n4 * p; i += blockDim.x) {
    const int k = i / p, nu = i - k * p;
    Ws[k * WS + nu] = k < n ? W[(int64_t)(b + k) * p + nu] : 0.0;
  }
  auto issue = [&](int t0, double* X) {
    const int nt = min(kLeafT, f1 - t0);
    for (int i = threadIdx.x; i < n4 * kLeafT; i += blockDim.x) {
      const int tl = i / n4, k = i - tl * n4;  // consecutive threads: consecutive panels (coalesced)
      double* d = X + k * XS + 2 * tl;
      if (k < n && tl < nt) cp_async16(d, xc + (int64_t)(t0 + tl) * M + b + k);
      else { d[0] = 0.0; d[1] = 0.0; }
    }
    cp_async_commit();
  };
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, q = lane & 3;
  const int nvt = (p + 7) / 8;
  int buf = 0;
  if (f0 < f1) issue(f0, X0);
  for (int t0 = f0; t0 < f1; t0 += kLeafT) {
    if (t0 + kLeafT < f1) issue(t0 + kLeafT, X0 + (buf ^ 1) * xsz);
    else cp_async_commit();
    cp_async_wait1();
    __syncthreads();
    const double* Xs = X0 + buf * xsz;
    const int nt = min(kLeafT, f1 - t0);
    for (int tile = warp; tile < nvt * 4; tile += blockDim.x >> 5) {
      const int v0 = (tile >> 2) * 8, n0 = (tile & 3) * 8;
      const int nu = v0 + g;
      double c0 = 0.0, c1 = 0.0;
      for (int k0 = 0; k0 < n4; k0 += 4) {
        const double a = nu < p ? Ws[(k0 + q) * WS + nu] : 0.0;
        const double bb = Xs[(k0 + q) * XS + n0 + g];
        dmma_k2(c0, c1, a, bb);
      }
      const int tl = (n0 >> 1) + q;
      if (nu < p && tl < nt) xhat[((int64_t)c * nl + t0 + tl) * p + nu] = make_double2(c0, c1);
    }
    __syncthreads();
    buf ^= 1;
  }
  cp_async_wait1();
}

__global__ void __launch_bounds__(kPassThreads) down_leaf_p_kernel(const int32_t* __restrict__ leaves,
                                                                   const int32_t* __restrict__ cb,
                                                                   const int32_t* __restrict__ ce,
                                                                   const double* __restrict__ U,
                                                                   const double2* __restrict__ yhat,
                                                                   const double2* __restrict__ yc,
                                                                   const int32_t* __restrict__ perm,
                                                                   double2* __restrict__ y, int64_t M, int nl, int p,
                                                                   const double2* __restrict__ xc, double alpha, int FT) {
  extern __shared__ double smd[];
  const int c = leaves[blockIdx.x];
  const int b = cb[c], n = ce[c] - b;
  const int p4 = (p + 3) & ~3;
  const int f0 = blockIdx.y * FT, f1 = min(nl, f0 + FT);
  const int US = pad8(p4), YS = pad8(2 * kLeafT);
  const int n8 = (n + 7) & ~7;
  double* Us = smd;              // [n8][US]: U[k][mu]
  double* Y0 = Us + n8 * US;     // 2 x [p4][YS]: yhat[t][mu] as Y[mu][2t + re/im]
  const size_t ysz = (size_t)p4 * YS;
  for (int i = threadIdx.x; i < n8 * p4; i += blockDim.x) {
    const int k = i / p4, mu = i - k * p4;
    Us[k * US + mu] = (k < n && mu < p) ? U[(int64_t)(b + k) * p + mu] : 0.0;
  }
  auto issue = [&](int t0, double* Y) {
    const int nt = min(kLeafT, f1 - t0);
    for (int i = threadIdx.x; i < kLeafT * p4; i += blockDim.x) {
      const int tl = i / p4, mu = i - tl * p4;
      double* d = Y + mu * YS + 2 * tl;
      if (mu < p && tl < nt) cp_async16(d, yhat + ((int64_t)c * nl + t0 + tl) * p + mu);
      else { d[0] = 0.0; d[1] = 0.0; }
    }
    cp_async_commit();
  };
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, q = lane & 3;
  const int nkt = n8 / 8;
  int buf = 0;
  if (f0 < f1) issue(f0, Y0);
  for (int t0 = f0; t0 < f1; t0 += kLeafT) {
    if (t0 + kLeafT < f1) issue(t0 + kLeafT, Y0 + (buf ^ 1) * ysz);
    else cp_async_commit();
    cp_async_wait1();
    __syncthreads();
    const double* Ys = Y0 + buf * ysz;
    const int nt = min(kLeafT, f1 - t0);
    for (int tile = warp; tile < nkt * 4; tile += blockDim.x >> 5) {
      const int k0r = (tile >> 2) * 8, n0 = (tile & 3) * 8;
      double c0 = 0.0, c1 = 0.0;
      for (int m0 = 0; m0 < p4; m0 += 4) {
        const double a = Us[(k0r + g) * US + m0 + q];
        const double bb = Ys[(m0 + q) * YS + n0 + g];
        dmma_k2(c0, c1, a, bb);
      }
      const int k = k0r + g, tl = (n0 >> 1) + q;
      if (k < n && tl < nt) {
        const int64_t row = (int64_t)(t0 + tl) * M;
        BEM_DASSERT(b + k < M && perm[b + k] >= 0 && perm[b + k] < M);
        double2 acc = yc[row + b + k];
        acc.x += c0;
        acc.y += c1;
        if (alpha != 0.0) {
          const double2 xv = xc[row + b + k];
          acc.x = fma(alpha, xv.x, acc.x);
          acc.y = fma(alpha, xv.y, acc.y);
        }
        y[row + perm[b + k]] = acc;
      }
    }
    __syncthreads();
    buf ^= 1;
  }
  cp_async_wait1();
}

// frequencies per CTA of the pipelined leaf kernels: about eight 16-frequency sub-tiles
inline int leaf_chunk(int nl) {
  static const int per = [] { const char* e = getenv("BEM_LEAF_SUB"); return e ? std::max(1, atoi(e)) : 8; }();
  const int nsub = (nl + kLeafT - 1) / kLeafT;
  const int nch = (nsub + per - 1) / per;  // CTAs per leaf, each pipelining <= per 16-column sub-tiles
  return kLeafT * ((nsub + nch - 1) / nch);
}
inline bool leaf_pipe() {
  static const bool on = [] { const char* e = getenv("BEM_LEAF_PIPE"); return e ? atoi(e) != 0 : true; }();
  return on;
}

// Kronecker transfers (tensor Chebyshev interpolation): E = E_z (x) E_y (x) E_x,
// so E^T x (upward) and E y (downward) are three m x m mode products on the m x m x m
// coefficient tensor (index mu = mx + m my + m^2 mz): 3 m p multiply-adds per (cluster,
// frequency) instead of p^2.  CTA = (parent cluster, tile of TF frequencies); the tiles of
// both sons / the parent are staged in shared memory and contracted axis by axis.
template <int MC>  // m at compile time (0: runtime m): constant index arithmetic
__global__ void __launch_bounds__(kPassThreads) up_transfer_k_kernel(const int32_t* __restrict__ list,
                                                                     const int32_t* __restrict__ son0,
                                                                     const int32_t* __restrict__ son1,
                                                                     const double* __restrict__ E1,
                                                                     double2* __restrict__ xhat, int nl, int m_, int TF) {
  extern __shared__ double2 smk[];
  const int m = MC > 0 ? MC : m_;
  const int p = m * m * m, mm = m * m;
  const int c = list[blockIdx.x];
  const int sons[2] = {son0[c], son1[c]};
  const int t0 = blockIdx.y * TF;
  const int nt = min(TF, nl - t0);
  double2* A = smk;                      // [2][TF][p]
  double2* B = A + 2 * TF * p;           // [2][TF][p]
  double* Es = (double*)(B + 2 * TF * p);  // [2][3][m][m]
  for (int i = threadIdx.x; i < 2 * 3 * mm; i += blockDim.x) {
    const int sidx = i / (3 * mm);
    Es[i] = E1[(size_t)sons[sidx] * 3 * mm + (i - sidx * 3 * mm)];
  }
  const int TP = TF * p;
  for (int i = threadIdx.x; i < 2 * TP; i += blockDim.x) {
    const int sidx = i / TP, r = i - sidx * TP;
    A[i] = r < nt * p ? xhat[((int64_t)sons[sidx] * nl + t0) * p + r] : make_double2(0.0, 0.0);
  }
  __syncthreads();
  // x: B[s][t][lz][ly][mx] = sum_lx Ex[lx][mx] A[s][t][lz][ly][lx]
  for (int i = threadIdx.x; i < 2 * TP; i += blockDim.x) {
    const int sidx = i / TP, e = i % p;
    const int mx = e % m, rest = e - mx;
    const double* Ex = Es + sidx * 3 * mm;
    const double2* a = A + (i - e) + rest;
    double2 acc = make_double2(0.0, 0.0);
    for (int l = 0; l < m; ++l) {
      const double w = Ex[l * m + mx];
      acc.x = fma(w, a[l].x, acc.x);
      acc.y = fma(w, a[l].y, acc.y);
    }
    B[i] = acc;
  }
  __syncthreads();
  // y: A[s][t][lz][my][mx] = sum_ly Ey[ly][my] B[s][t][lz][ly][mx]
  for (int i = threadIdx.x; i < 2 * TP; i += blockDim.x) {
    const int sidx = i / TP, e = i % p;
    const int mx = e % m, my = (e / m) % m, lz = e / mm;
    const double* Ey = Es + sidx * 3 * mm + mm;
    const double2* b = B + (i - e) + lz * mm + mx;
    double2 acc = make_double2(0.0, 0.0);
    for (int l = 0; l < m; ++l) {
      const double w = Ey[l * m + my];
      acc.x = fma(w, b[l * m].x, acc.x);
      acc.y = fma(w, b[l * m].y, acc.y);
    }
    A[i] = acc;
  }
  __syncthreads();
  // z and the sum over both sons: out[t][mz][my][mx] = sum_s sum_lz Ez_s[lz][mz] A[s][t][lz][my][mx]
  for (int i = threadIdx.x; i < nt * p; i += blockDim.x) {
    const int e = i % p;
    const int mz = e / mm, rest = e - mz * mm;
    double2 acc = make_double2(0.0, 0.0);
    for (int sidx = 0; sidx < 2; ++sidx) {
      const double* Ez = Es + sidx * 3 * mm + 2 * mm;
      const double2* a = A + sidx * TP + (i - e) + rest;
      for (int l = 0; l < m; ++l) {
        const double w = Ez[l * m + mz];
        acc.x = fma(w, a[l * mm].x, acc.x);
        acc.y = fma(w, a[l * mm].y, acc.y);
      }
    }
    xhat[((int64_t)c * nl + t0) * p + i] = acc;
  }
}

template <int MC>  // m at compile time (0: runtime m): constant index arithmetic
__global__ void __launch_bounds__(kPassThreads) down_transfer_k_kernel(const int32_t* __restrict__ list,
                                                                       const int32_t* __restrict__ son0,
                                                                       const int32_t* __restrict__ son1,
                                                                       const double* __restrict__ E1,
                                                                       double2* __restrict__ yhat, int nl, int m_, int TF) {
  extern __shared__ double2 smk[];
  const int m = MC > 0 ? MC : m_;
  const int p = m * m * m, mm = m * m;
  const int c = list[blockIdx.x];
  const int sons[2] = {son0[c], son1[c]};
  const int t0 = blockIdx.y * TF;
  const int nt = min(TF, nl - t0);
  const int TP = TF * p;
  double2* P = smk;                      // [TF][p] parent tile
  double2* B = P + TP;                   // [2][TF][p]
  double2* C2 = B + 2 * TP;              // [2][TF][p]
  double* Es = (double*)(C2 + 2 * TP);   // [2][3][m][m]
  for (int i = threadIdx.x; i < 2 * 3 * mm; i += blockDim.x) {
    const int sidx = i / (3 * mm);
    Es[i] = E1[(size_t)sons[sidx] * 3 * mm + (i - sidx * 3 * mm)];
  }
  for (int i = threadIdx.x; i < TP; i += blockDim.x)
    P[i] = i < nt * p ? yhat[((int64_t)c * nl + t0) * p + i] : make_double2(0.0, 0.0);
  __syncthreads();
  // x: B[s][t][mz][my][lx] = sum_mx Ex_s[lx][mx] P[t][mz][my][mx]
  for (int i = threadIdx.x; i < 2 * TP; i += blockDim.x) {
    const int sidx = i / TP, r = i - sidx * TP, e = r % p;
    const int lx = e % m, rest = e - lx;
    const double* Ex = Es + sidx * 3 * mm;
    const double2* a = P + (r - e) + rest;
    double2 acc = make_double2(0.0, 0.0);
    for (int u = 0; u < m; ++u) {
      const double w = Ex[lx * m + u];
      acc.x = fma(w, a[u].x, acc.x);
      acc.y = fma(w, a[u].y, acc.y);
    }
    B[i] = acc;
  }
  __syncthreads();
  // y: C[s][t][mz][ly][lx] = sum_my Ey_s[ly][my] B[s][t][mz][my][lx]
  for (int i = threadIdx.x; i < 2 * TP; i += blockDim.x) {
    const int sidx = i / TP, e = i % p;
    const int lx = e % m, ly = (e / m) % m, mz = e / mm;
    const double* Ey = Es + sidx * 3 * mm + mm;
    const double2* b = B + (i - e) + mz * mm + lx;
    double2 acc = make_double2(0.0, 0.0);
    for (int u = 0; u < m; ++u) {
      const double w = Ey[ly * m + u];
      acc.x = fma(w, b[u * m].x, acc.x);
      acc.y = fma(w, b[u * m].y, acc.y);
    }
    C2[i] = acc;
  }
  __syncthreads();
  // z: yhat_s[t][lz][ly][lx] += sum_mz Ez_s[lz][mz] C[s][t][mz][ly][lx]
  for (int i = threadIdx.x; i < 2 * TP; i += blockDim.x) {
    const int sidx = i / TP, r = i - sidx * TP, e = r % p;
    if (r >= nt * p) continue;
    const int lz = e / mm, rest = e - lz * mm;
    const double* Ez = Es + sidx * 3 * mm + 2 * mm;
    const double2* cc = C2 + (i - e) + rest;
    double2* out = yhat + ((int64_t)sons[sidx] * nl + t0) * p + r;
    double2 acc = *out;
    for (int u = 0; u < m; ++u) {
      const double w = Ez[lz * m + u];
      acc.x = fma(w, cc[u * mm].x, acc.x);
      acc.y = fma(w, cc[u * mm].y, acc.y);
    }
    *out = acc;
  }
}

constexpr size_t kPassSmemMax = 100 * 1024;

template <int MC>
cudaError_t launch_upk(unsigned n, unsigned ttk, size_t sm, cudaStream_t st, const int32_t* list, const int32_t* s0,
                       const int32_t* s1, const double* E1, double2* xhat, int nl, int m, int TF, bool down) {
  auto k = down ? down_transfer_k_kernel<MC> : up_transfer_k_kernel<MC>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  if (e != cudaSuccess) return e;
  k<<<dim3(n, ttk), kPassThreads, sm, st>>>(list, s0, s1, E1, xhat, nl, m, TF);
  return cudaGetLastError();
}

cudaError_t launch_transfer_k(unsigned n, unsigned ttk, size_t sm, cudaStream_t st, const int32_t* list,
                              const int32_t* s0, const int32_t* s1, const double* E1, double2* xy, int nl, int m,
                              int TF, bool down) {
  switch (m) {
    case 3: return launch_upk<3>(n, ttk, sm, st, list, s0, s1, E1, xy, nl, m, TF, down);
    case 4: return launch_upk<4>(n, ttk, sm, st, list, s0, s1, E1, xy, nl, m, TF, down);
    case 5: return launch_upk<5>(n, ttk, sm, st, list, s0, s1, E1, xy, nl, m, TF, down);
    default: return launch_upk<0>(n, ttk, sm, st, list, s0, s1, E1, xy, nl, m, TF, down);
  }
}


constexpr size_t kLeafSmemMax = 160 * 1024;
constexpr size_t kTransferSmem = 56 * 1024;  // Kronecker transfers: 4 CTAs per SM  // DMMA leaf kernels (p = 125: one CTA per SM)

__global__ void scatter_kernel(const double2* __restrict__ yc, double2* __restrict__ y,
                               const int32_t* __restrict__ perm, int64_t M, int nl, const double2* __restrict__ xc, double alpha) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= M * nl) return;
  const int64_t t = i / M, k = i - t * M;
  double2 v = yc[i];
  if (alpha != 0.0) {
    v.x = fma(alpha, xc[i].x, v.x);
    v.y = fma(alpha, xc[i].y, v.y);
  }
  y[t * M + perm[k]] = v;
}

// K2 up / down passes over nl columns, staged kernels when their tiles fit
bem_status run_up(Tree& t, const double* W, const double2* xc, double2* xhat, int nl, cudaStream_t st) {
  const int p = t.p;
  const unsigned tt = (unsigned)((nl + kPassT - 1) / kPassT);
  const int n4 = (t.max_leaf + 3) & ~3;
  const size_t sm_d = sizeof(double) * (size_t)n4 * (pad8(p) + pad8(2 * kLeafT));
  const size_t sm_leaf = sizeof(double2) * kPassT * t.max_leaf + sizeof(double) * (size_t)t.max_leaf * p;
  const size_t sm_p = sizeof(double) * (size_t)n4 * (pad8(p) + 2 * pad8(2 * kLeafT));
  if (leaf_pipe() && sm_p <= kLeafSmemMax) {
    const int FT = leaf_chunk(nl);
    BEM_CK(cudaFuncSetAttribute(up_leaf_p_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm_p));
    up_leaf_p_kernel<<<dim3((unsigned)t.n_leaves, (unsigned)((nl + FT - 1) / FT)), kPassThreads, sm_p, st>>>(
        t.d_leaves.p, t.d_begin.p, t.d_end.p, W, xc, xhat, t.M, nl, p, FT);
  } else if (sm_d <= kLeafSmemMax) {
    BEM_CK(cudaFuncSetAttribute(up_leaf_d_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm_d));
    up_leaf_d_kernel<<<dim3((unsigned)t.n_leaves, (unsigned)((nl + kLeafT - 1) / kLeafT)), kPassThreads, sm_d, st>>>(
        t.d_leaves.p, t.d_begin.p, t.d_end.p, W, xc, xhat, t.M, nl, p);
  } else if (sm_leaf <= kPassSmemMax) {
    BEM_CK(cudaFuncSetAttribute(up_leaf_s_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm_leaf));
    up_leaf_s_kernel<<<dim3((unsigned)t.n_leaves, tt), kPassThreads, sm_leaf, st>>>(t.d_leaves.p, t.d_begin.p,
                                                                                   t.d_end.p, W, xc, xhat, t.M, nl, p);
  } else {
    up_leaf_kernel<<<dim3((unsigned)t.n_leaves, tt), kPassThreads, 0, st>>>(t.d_leaves.p, t.d_begin.p, t.d_end.p, W,
                                                                             xc, xhat, t.M, nl, p);
  }
  BEM_CK(cudaGetLastError());
  // Kronecker transfers: TF frequencies per CTA with four [TF][p] tiles in shared memory
  static const int tf_env = [] { const char* e = getenv("BEM_K2_TF"); return e ? atoi(e) : 0; }();
  // r3g sweep (config 4, up / down ms): TF 13 (56 KB budget) 2.62 / 3.05, TF 4 2.28 / 2.77, TF 8 2.27 / 2.88
  const int TF = tf_env > 0 ? tf_env : std::min(4, std::max(1, (int)(kTransferSmem / (sizeof(double2) * 4 * p))));
  const size_t sm_k = sizeof(double2) * 4 * (size_t)TF * p + sizeof(double) * 6 * t.m * t.m;
  const unsigned ttk = (unsigned)((nl + TF - 1) / TF);
  if (t.d_E1.p) {
    for (int lv = t.depth - 1; lv >= 0; --lv) {
      const int n = (int)t.level_nonleaf[lv].size();
      if (n == 0) continue;
      BEM_CK(launch_transfer_k((unsigned)n, ttk, sm_k, st, t.d_level_nonleaf[lv].p, t.d_son0.p, t.d_son1.p, t.d_E1.p,
                               xhat, nl, t.m, TF, false));
    }
    return BEM_OK;
  }
  const size_t sm_tr = sizeof(double2) * 2 * kPassT * p + sizeof(double) * 2 * (size_t)p * p;
  const bool staged = sm_tr <= kPassSmemMax;
  if (staged)
    BEM_CK(cudaFuncSetAttribute(up_transfer_s_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm_tr));
  for (int lv = t.depth - 1; lv >= 0; --lv) {
    const int n = (int)t.level_nonleaf[lv].size();
    if (n == 0) continue;
    if (staged)
      up_transfer_s_kernel<<<dim3((unsigned)n, tt), kPassThreads, sm_tr, st>>>(t.d_level_nonleaf[lv].p, t.d_son0.p,
                                                                               t.d_son1.p, t.d_E.p, xhat, nl, p);
    else
      up_transfer_kernel<<<dim3((unsigned)n, tt), kPassThreads, 0, st>>>(t.d_level_nonleaf[lv].p, t.d_son0.p,
                                                                         t.d_son1.p, t.d_E.p, xhat, nl, p);
    BEM_CK(cudaGetLastError());
  }
  return BEM_OK;
}

bem_status run_down(Tree& t, double2* yhat, const double2* yc, double2* y, int nl, const double2* xc, double alpha,
                    cudaStream_t st, cudaEvent_t wait_before_leaf = nullptr) {
  const int p = t.p;
  const unsigned tt = (unsigned)((nl + kPassT - 1) / kPassT);
  static const int tf_env = [] { const char* e = getenv("BEM_K2_TF"); return e ? atoi(e) : 0; }();
  const int TF = tf_env > 0 ? tf_env : std::min(4, std::max(1, (int)(kTransferSmem / (sizeof(double2) * 5 * p))));
  const size_t sm_k = sizeof(double2) * 5 * (size_t)TF * p + sizeof(double) * 6 * t.m * t.m;
  const unsigned ttk = (unsigned)((nl + TF - 1) / TF);
  const size_t sm_tr = sizeof(double2) * kPassT * p + sizeof(double) * 2 * (size_t)p * p;
  const bool kron = t.d_E1.p != nullptr;
  const bool staged = sm_tr <= kPassSmemMax;
  if (!kron && staged)
    BEM_CK(cudaFuncSetAttribute(down_transfer_s_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm_tr));
  for (int lv = 0; lv < t.depth; ++lv) {
    const int n = (int)t.level_nonleaf[lv].size();
    if (n == 0) continue;
    if (kron)
      BEM_CK(launch_transfer_k((unsigned)n, ttk, sm_k, st, t.d_level_nonleaf[lv].p, t.d_son0.p, t.d_son1.p, t.d_E1.p,
                               yhat, nl, t.m, TF, true));
    else if (staged)
      down_transfer_s_kernel<<<dim3((unsigned)n, tt), kPassThreads, sm_tr, st>>>(t.d_level_nonleaf[lv].p, t.d_son0.p,
                                                                                 t.d_son1.p, t.d_ET.p, yhat, nl, p);
    else
      down_transfer_kernel<<<dim3((unsigned)n, tt), kPassThreads, 0, st>>>(t.d_level_nonleaf[lv].p, t.d_son0.p,
                                                                           t.d_son1.p, t.d_ET.p, yhat, nl, p);
    BEM_CK(cudaGetLastError());
  }
  if (wait_before_leaf) BEM_CK(cudaStreamWaitEvent(st, wait_before_leaf, 0));
  const int p4 = (p + 3) & ~3, n8 = (t.max_leaf + 7) & ~7;
  const size_t sm_d = sizeof(double) * ((size_t)n8 * pad8(p4) + (size_t)p4 * pad8(2 * kLeafT));
  const size_t sm_leaf = sizeof(double2) * kPassT * p + sizeof(double) * (size_t)p * t.max_leaf;
  const size_t sm_p = sizeof(double) * ((size_t)n8 * pad8(p4) + 2 * (size_t)p4 * pad8(2 * kLeafT));
  if (leaf_pipe() && sm_p <= kLeafSmemMax) {
    const int FT = leaf_chunk(nl);
    BEM_CK(cudaFuncSetAttribute(down_leaf_p_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm_p));
    down_leaf_p_kernel<<<dim3((unsigned)t.n_leaves, (unsigned)((nl + FT - 1) / FT)), kPassThreads, sm_p, st>>>(
        t.d_leaves.p, t.d_begin.p, t.d_end.p, t.d_U.p, yhat, yc, t.d_perm.p, y, t.M, nl, p, xc, alpha, FT);
  } else if (sm_d <= kLeafSmemMax) {
    BEM_CK(cudaFuncSetAttribute(down_leaf_d_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm_d));
    down_leaf_d_kernel<<<dim3((unsigned)t.n_leaves, (unsigned)((nl + kLeafT - 1) / kLeafT)), kPassThreads, sm_d,
                         st>>>(t.d_leaves.p, t.d_begin.p, t.d_end.p, t.d_U.p, yhat, yc, t.d_perm.p, y, t.M, nl, p, xc,
                               alpha);
  } else if (sm_leaf <= kPassSmemMax) {
    BEM_CK(cudaFuncSetAttribute(down_leaf_s_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm_leaf));
    down_leaf_s_kernel<<<dim3((unsigned)t.n_leaves, tt), kPassThreads, sm_leaf, st>>>(
        t.d_leaves.p, t.d_begin.p, t.d_end.p, t.d_UT.p, yhat, yc, t.d_perm.p, y, t.M, nl, p, xc, alpha);
  } else {
    down_leaf_kernel<<<dim3((unsigned)t.n_leaves, tt), kPassThreads, 0, st>>>(
        t.d_leaves.p, t.d_begin.p, t.d_end.p, t.d_UT.p, yhat, yc, t.d_perm.p, y, t.M, nl, p, 1, xc, alpha);
  }
  BEM_CK(cudaGetLastError());
  return BEM_OK;
}

}  // namespace

// y = V x (dl = false) or y = (alpha I + K) x (dl = true, double layer, NEXT-1): the
// same coupling tensors / ACA skeleton, K's near field and column basis W^K
bem_status apply_launch(Op& op, const double* xin, double* yout, cudaStream_t st, bool dl, double alpha) {
  Tree& t = *op.tree;
  const int64_t M = t.M;
  const int nl = op.n_local;
  const double2* x = (const double2*)xin;
  double2* y = (double2*)yout;
  double2* xc = (double2*)op.d_xc.p;
  double2* yc = (double2*)op.d_yc.p;
  double2* xhat = (double2*)op.d_xhat.p;
  double2* yhat = (double2*)op.d_yhat.p;
  const bool prof = op.profile;
  if (prof) {
    for (auto& e : op.ev)
      if (!e) BEM_CK(cudaEventCreate(&e));
    BEM_CK(cudaEventRecord(op.ev[0], st));
    if (op.d_near_evals.p) BEM_CK(cudaMemsetAsync(op.d_near_evals.p, 0, sizeof(unsigned long long), st));
  }
  Nvtx nv_apply(dl ? "apply_double_layer" : "apply_multifreq");
  const int64_t tot = M * nl;
  {
    Nvtx nv("a2 gather");
    gather_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(x, xc, t.d_perm.p, M, nl);
  }
  BEM_CK(cudaGetLastError());
  const bool dense = op.mode == BEM_MODE_DENSE;
  const bool has_far = !dense && !t.far_r.empty();
  // K1 (near field) and the far branch (K2 up, K3, K2 down transfers) are independent until
  // the leaf-level scatter: unless per-kernel timers are on, K1 runs on a side stream forked
  // from st (event fork/join, graph-capturable) so both kernels share the SMs' FP64 pipes
  // K1 fused into the far10 launch (near-field warps beside the coupling work, then a tail
  // kernel for the items they left) where far10 runs; per-kernel timers keep the kernels apart
  const bool fuse = !dl && has_far && !prof && far_fuses_near(op);
  const bool overlap = op.overlap && has_far && !prof && !fuse;
  NearArgs fna;
  if (fuse) {
    int F = 4;
    near_args(op, xc, yc, fna, F);
  }
  cudaStream_t sk1 = st;
  if (overlap) {
    if (!op.side) {
      int lo = 0, hi = 0;
      BEM_CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
      BEM_CK(cudaStreamCreateWithPriority(&op.side, cudaStreamNonBlocking, lo));  // K1: lowest priority
      BEM_CK(cudaEventCreateWithFlags(&op.ev_fork, cudaEventDisableTiming));
      BEM_CK(cudaEventCreateWithFlags(&op.ev_join, cudaEventDisableTiming));
    }
    BEM_CK(cudaEventRecord(op.ev_fork, st));
    BEM_CK(cudaStreamWaitEvent(op.side, op.ev_fork, 0));
    sk1 = op.side;
  }
  if (!fuse) {
    Nvtx nv("a3 K1 near field");
    bem_status rs = launch_near(op, xc, yc, sk1, dl);
    if (rs != BEM_OK) return rs;
  }
  if (overlap) BEM_CK(cudaEventRecord(op.ev_join, sk1));
  if (prof) BEM_CK(cudaEventRecord(op.ev[1], st));
  if (has_far) {
    {
      Nvtx nv("a4 K2 up");
      bem_status rs = run_up(t, dl ? t.d_WK.p : t.d_W.p, xc, xhat, nl, st);
      if (rs != BEM_OK) return rs;
    }
    if (prof) BEM_CK(cudaEventRecord(op.ev[2], st));
    bem_status rs;
    {
      Nvtx nv(fuse ? "a5 K3 coupling + a3 K1 near field (fused)" : "a5 K3 coupling");
      rs = launch_far(op, xhat, yhat, st, fuse ? &fna : nullptr);
    }
    if (rs != BEM_OK) return rs;
    if (prof) BEM_CK(cudaEventRecord(op.ev[3], st));
    {
      // the down transfers do not read yc: only the leaf scatter waits for K1
      Nvtx nv("a6-a7 K2 down + scatter");
      bem_status rs = run_down(t, yhat, yc, y, nl, xc, dl ? alpha : 0.0, st, overlap ? op.ev_join : nullptr);
      if (rs != BEM_OK) return rs;
    }
  } else {
    if (prof) { BEM_CK(cudaEventRecord(op.ev[2], st)); BEM_CK(cudaEventRecord(op.ev[3], st)); }
    scatter_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(yc, y, t.d_perm.p, M, nl, xc, dl ? alpha : 0.0);
    BEM_CK(cudaGetLastError());
  }
  if (prof) BEM_CK(cudaEventRecord(op.ev[4], st));
  return BEM_OK;
}

// Building blocks for the time-domain path (mot.cu): ncols columns, [ncols][M] layout.
bem_status h2_gather(Op& op, const double2* x, double2* xc, int ncols, cudaStream_t st) {
  const int64_t tot = op.tree->M * ncols;
  gather_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(x, xc, op.tree->d_perm.p, op.tree->M, ncols);
  BEM_CK(cudaGetLastError());
  return BEM_OK;
}

bem_status h2_up(Op& op, const double2* xc, double2* xhat, int ncols, cudaStream_t st) {
  return run_up(*op.tree, op.tree->d_W.p, xc, xhat, ncols, st);
}

// y (input order) = ycn + U-side of the downward pass of yhat
bem_status h2_down_scatter(Op& op, double2* yhat, const double2* ycn, double2* y, int ncols, cudaStream_t st) {
  Tree& t = *op.tree;
  if (t.far_r.empty()) {
    const int64_t tot = t.M * ncols;
    scatter_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(ycn, y, t.d_perm.p, t.M, ncols, ycn, 0.0);
    BEM_CK(cudaGetLastError());
    return BEM_OK;
  }
  return run_down(t, yhat, ycn, y, ncols, ycn, 0.0, st);
}

}  // namespace bem

using namespace bem;

extern "C" bem_status bem_apply_multifreq(bem_op oh, const bem_c128* x, bem_c128* y, void* cuda_stream) {
  BEM_REQ(oh && x && y, "bem_apply_multifreq: NULL argument");
  BEM_REQ(((uintptr_t)x & 15) == 0 && ((uintptr_t)y & 15) == 0, "bem_apply_multifreq: pointers must be 16-byte aligned");
  Op& op = oh->o;
  const size_t bytes = (size_t)op.n_local * op.tree->M * 16;
  BEM_REQ((const char*)x + bytes <= (const char*)y || (const char*)y + bytes <= (const char*)x,
          "bem_apply_multifreq: x and y overlap");
  cudaPointerAttributes at;
  BEM_CK(cudaPointerGetAttributes(&at, x));
  BEM_REQ(at.type == cudaMemoryTypeDevice && at.device == op.tree->device,
          "bem_apply_multifreq: x must be device memory on device %d", op.tree->device);
  BEM_CK(cudaPointerGetAttributes(&at, y));
  BEM_REQ(at.type == cudaMemoryTypeDevice && at.device == op.tree->device,
          "bem_apply_multifreq: y must be device memory on device %d", op.tree->device);
  DeviceGuard dg(op.tree->device);
  return apply_launch(op, (const double*)x, (double*)y, (cudaStream_t)cuda_stream, false, 0.0);
}

extern "C" bem_status bem_apply_double_layer(bem_op oh, const bem_c128* x, bem_c128* y, double alpha,
                                             void* cuda_stream) {
  BEM_REQ(oh && x && y, "bem_apply_double_layer: NULL argument");
  BEM_REQ(((uintptr_t)x & 15) == 0 && ((uintptr_t)y & 15) == 0,
          "bem_apply_double_layer: pointers must be 16-byte aligned");
  Op& op = oh->o;
  const size_t bytes = (size_t)op.n_local * op.tree->M * 16;
  BEM_REQ((const char*)x + bytes <= (const char*)y || (const char*)y + bytes <= (const char*)x,
          "bem_apply_double_layer: x and y overlap");
  cudaPointerAttributes at;
  BEM_CK(cudaPointerGetAttributes(&at, x));
  BEM_REQ(at.type == cudaMemoryTypeDevice && at.device == op.tree->device,
          "bem_apply_double_layer: x must be device memory on device %d", op.tree->device);
  BEM_CK(cudaPointerGetAttributes(&at, y));
  BEM_REQ(at.type == cudaMemoryTypeDevice && at.device == op.tree->device,
          "bem_apply_double_layer: y must be device memory on device %d", op.tree->device);
  DeviceGuard dg(op.tree->device);
  return apply_launch(op, (const double*)x, (double*)y, (cudaStream_t)cuda_stream, true, alpha);
}

extern "C" bem_status bem_op_launch_count(bem_op oh, int32_t* n) {
  BEM_REQ(oh && n, "bem_op_launch_count: NULL argument");
  const Op& op = oh->o;
  const Tree& t = *op.tree;
  int c = 3;  // gather, K1, scatter / down-leaf
  if (op.mode != BEM_MODE_DENSE && !t.far_r.empty()) {
    c += 2;  // up-leaf, K3
    for (int lv = 0; lv < t.depth; ++lv) c += t.level_nonleaf[lv].empty() ? 0 : 2;
  }
  *n = c;
  return BEM_OK;
}

extern "C" bem_status bem_op_set_profiling(bem_op oh, int32_t enable) {
  BEM_REQ(oh, "bem_op_set_profiling: NULL op");
  Op& op = oh->o;
  op.profile = enable != 0;
  if (op.profile && op.d_near_evals.p == nullptr) {
    DeviceGuard dg(op.tree->device);
    BEM_CK(op.d_near_evals.alloc(1));
    BEM_CK(cudaMemset(op.d_near_evals.p, 0, sizeof(unsigned long long)));
  }
  return BEM_OK;
}

extern "C" bem_status bem_op_get_work(bem_op oh, bem_op_work* out) {
  BEM_REQ(oh && out, "bem_op_get_work: NULL argument");
  Op& op = oh->o;
  DeviceGuard dg(op.tree->device);
  BEM_CK(cudaDeviceSynchronize());
  const bool aca = op.mode == BEM_MODE_H2ACA || op.mode == BEM_MODE_COMBINED;
  out->far_rank_cols_run = out->far_rank_cols_total = 0;
  if (aca) far10_work(op, &out->far_rank_cols_run, &out->far_rank_cols_total);
  const int64_t nnz = op.mode == BEM_MODE_DENSE ? op.tree->M * op.tree->M : op.tree->nnz_near;
  out->near_evals_total = 7 * nnz * op.n_class;
  out->near_evals_run = -1;
  if (op.d_near_evals.p != nullptr) {
    unsigned long long v = 0;
    BEM_CK(cudaMemcpy(&v, op.d_near_evals.p, sizeof(v), cudaMemcpyDeviceToHost));
    out->near_evals_run = (int64_t)v;
  }
  out->near_tau = op.near_tau;
  out->far_delta = op.d_skip.p != nullptr ? op.far_delta : 0.0;
  return BEM_OK;
}

extern "C" bem_status bem_op_get_timings(bem_op oh, double* ms5) {
  BEM_REQ(oh && ms5, "bem_op_get_timings: NULL argument");
  Op& op = oh->o;
  if (!op.profile || !op.ev[4]) {
    set_error("bem_op_get_timings: profiling was not enabled for the last apply");
    return BEM_ESTATE;
  }
  DeviceGuard dg(op.tree->device);
  BEM_CK(cudaEventSynchronize(op.ev[4]));
  float ms[4];
  for (int i = 0; i < 4; ++i) BEM_CK(cudaEventElapsedTime(&ms[i], op.ev[i], op.ev[i + 1]));
  // K1 (incl. gather), K2 up, K3, K2 down (incl. scatter), other
  ms5[0] = ms[0]; ms5[1] = ms[1]; ms5[2] = ms[2]; ms5[3] = ms[3]; ms5[4] = 0.0;
  return BEM_OK;
}
