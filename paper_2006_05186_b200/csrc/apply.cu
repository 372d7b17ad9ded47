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
#include <cmath>

#include "common.cuh"

namespace bem {
namespace {

constexpr double kInv4Pi = 0.079577471545947667884;  // 1/(4 pi)

__device__ __forceinline__ double2 cmadd(double2 acc, double2 a, double2 b) {
  acc.x = fma(a.x, b.x, acc.x);
  acc.x = fma(-a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y);
  acc.y = fma(a.y, b.x, acc.y);
  return acc;
}
__device__ __forceinline__ double2 cmadd_conj(double2 acc, double2 a, double2 b) {  // acc + conj(a) b
  acc.x = fma(a.x, b.x, acc.x);
  acc.x = fma(a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y);
  acc.y = fma(-a.y, b.x, acc.y);
  return acc;
}

// ------------------------------------------------------------------ gather
__global__ void gather_kernel(const double2* __restrict__ x, double2* __restrict__ xc, const int32_t* __restrict__ perm,
                              int64_t M, int nl) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= M * nl) return;
  const int64_t t = i / M, k = i - t * M;
  xc[i] = x[t * M + perm[k]];
}

// -------------------------------------------------------------------- K1
struct NearArgs {
  int64_t M;
  int nl, n_class;
  const int32_t* leaf_of;
  const int32_t* near_ptr;
  const int32_t* near_cb;
  const int32_t* near_ce;
  const double* cen;
  const double* qn;
  const double* qw;
  const double* selfJ;
  const double2* s;
  const int32_t* local_l;
  const int32_t* class_t1;
  const int32_t* class_t2;
  const double2* xc;
  double2* yc;
};

constexpr int kNearWarps = 4;
constexpr int kNearF = 8;

__global__ void __launch_bounds__(kNearWarps * 32) near_kernel(NearArgs a) {
  const int lane = threadIdx.x & 31;
  const int64_t k = (int64_t)blockIdx.x * kNearWarps + (threadIdx.x >> 5);
  if (k >= a.M) return;
  const int c0 = blockIdx.y * kNearF;
  const int nf = min(kNearF, a.n_class - c0);
  double sre[kNearF], sim[kNearF];
  int t1[kNearF], t2[kNearF];
#pragma unroll
  for (int f = 0; f < kNearF; ++f) {
    if (f < nf) {
      t1[f] = a.class_t1[c0 + f];
      t2[f] = a.class_t2[c0 + f];
      const double2 sv = a.s[a.local_l[t1[f]]];
      sre[f] = sv.x; sim[f] = sv.y;
    } else {
      t1[f] = -1; t2[f] = -1; sre[f] = 0.0; sim[f] = 0.0;
    }
  }
  double2 acc1[kNearF], acc2[kNearF];
#pragma unroll
  for (int f = 0; f < kNearF; ++f) { acc1[f] = make_double2(0.0, 0.0); acc2[f] = make_double2(0.0, 0.0); }
  const double cx = a.cen[3 * k], cy = a.cen[3 * k + 1], cz = a.cen[3 * k + 2];
  const int li = a.leaf_of[k];
  for (int rg = a.near_ptr[li]; rg < a.near_ptr[li + 1]; ++rg) {
    const int jb = a.near_cb[rg], je = a.near_ce[rg];
    for (int j = jb + lane; j < je; j += 32) {
      double rq[7], wq[7];
#pragma unroll
      for (int q = 0; q < 7; ++q) {
        const double dx = cx - a.qn[21 * (int64_t)j + 3 * q];
        const double dy = cy - a.qn[21 * (int64_t)j + 3 * q + 1];
        const double dz = cz - a.qn[21 * (int64_t)j + 3 * q + 2];
        rq[q] = sqrt(dx * dx + dy * dy + dz * dz);
        wq[q] = a.qw[7 * (int64_t)j + q];
      }
      const bool self = (j == k);
#pragma unroll
      for (int f = 0; f < kNearF; ++f) {
        if (f >= nf) break;
        double vr = 0.0, vi = 0.0;
        if (!self) {
#pragma unroll
          for (int q = 0; q < 7; ++q) {
            const double e = exp(-sre[f] * rq[q]) * (wq[q] / rq[q]);
            double sn, cs;
            sincos(sim[f] * rq[q], &sn, &cs);
            vr = fma(e, cs, vr);
            vi = fma(-e, sn, vi);
          }
        } else {
          // (1/4pi)[J + |T| sum_q w_q phi(s, r_q)], phi(s,0) = -s
          vr = a.selfJ[j] - wq[0] * sre[f];
          vi = -wq[0] * sim[f];
#pragma unroll
          for (int q = 1; q < 7; ++q) {
            const double xr = -sre[f] * rq[q], yr = -sim[f] * rq[q];
            double sn, cs, sh, ch;
            sincos(yr, &sn, &cs);
            sincos(0.5 * yr, &sh, &ch);
            const double re = expm1(xr) * cs - 2.0 * sh * sh;
            const double im = exp(xr) * sn;
            vr = fma(wq[q] / rq[q], re, vr);
            vi = fma(wq[q] / rq[q], im, vi);
          }
        }
        const double2 kv = make_double2(vr, vi);
        acc1[f] = cmadd(acc1[f], kv, a.xc[(int64_t)t1[f] * a.M + j]);
        if (t2[f] >= 0) acc2[f] = cmadd_conj(acc2[f], kv, a.xc[(int64_t)t2[f] * a.M + j]);
      }
    }
  }
#pragma unroll
  for (int f = 0; f < kNearF; ++f) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      acc1[f].x += __shfl_xor_sync(0xffffffffu, acc1[f].x, off);
      acc1[f].y += __shfl_xor_sync(0xffffffffu, acc1[f].y, off);
      acc2[f].x += __shfl_xor_sync(0xffffffffu, acc2[f].x, off);
      acc2[f].y += __shfl_xor_sync(0xffffffffu, acc2[f].y, off);
    }
  }
#pragma unroll
  for (int f = 0; f < kNearF; ++f) {
    if (f < nf && lane == 2 * f) a.yc[(int64_t)t1[f] * a.M + k] = acc1[f];
    if (f < nf && lane == 2 * f + 1 && t2[f] >= 0) a.yc[(int64_t)t2[f] * a.M + k] = acc2[f];
  }
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
    const double* Es = E + (int64_t)sc * p * p + (int64_t)lam * p;
    const double2* yp = yhat + ((int64_t)c * nl + t) * p;
    double2 acc = yhat[((int64_t)sc * nl + t) * p + lam];
    for (int mu = 0; mu < p; ++mu) {
      acc.x = fma(Es[mu], yp[mu].x, acc.x);
      acc.y = fma(Es[mu], yp[mu].y, acc.y);
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
                                                                 int has_far) {
  const int c = leaves[blockIdx.x];
  const int b = cb[c], e = ce[c], n = e - b;
  const int t0 = blockIdx.y * kPassT;
  for (int idx = threadIdx.x; idx < kPassT * n; idx += blockDim.x) {
    const int t = t0 + idx / n, k = b + idx % n;
    if (t >= nl) break;
    double2 acc = yc[(int64_t)t * M + k];
    if (has_far) {
      const double2* yh = yhat + ((int64_t)c * nl + t) * p;
      const double* Uk = U + (int64_t)k * p;
      for (int mu = 0; mu < p; ++mu) {
        acc.x = fma(Uk[mu], yh[mu].x, acc.x);
        acc.y = fma(Uk[mu], yh[mu].y, acc.y);
      }
    }
    y[(int64_t)t * M + perm[k]] = acc;
  }
}

__global__ void scatter_kernel(const double2* __restrict__ yc, double2* __restrict__ y,
                               const int32_t* __restrict__ perm, int64_t M, int nl) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= M * nl) return;
  const int64_t t = i / M, k = i - t * M;
  y[t * M + perm[k]] = yc[i];
}

// ------------------------------------------------------------------- K3
struct FarArgs {
  int C, nl, m, p, mode, rcap;
  const int32_t* far_ptr;
  const int32_t* far_sorted;
  const int32_t* far_c;
  const double* xi;
  const double2* s;
  const int32_t* local_l;
  const int32_t* rank;
  const int32_t* pivk;
  const int64_t* zoff;
  const double2* Z;
  const double2* xhat;
  double2* yhat;
};

constexpr int kFarThreads = 256;
constexpr int kFarT = 32;  // frequencies per CTA

__device__ __forceinline__ double2 kern(double r, double2 s) {
  const double e = exp(-s.x * r) / (12.566370614359172954 * r);
  double sn, cs;
  sincos(s.y * r, &sn, &cs);
  return make_double2(e * cs, -e * sn);
}

__global__ void __launch_bounds__(kFarThreads) far_kernel(FarArgs a) {
  extern __shared__ double2 sm[];
  const int p = a.p, m = a.m;
  const int r = blockIdx.x;
  const int t0 = blockIdx.y * kFarT;
  const int nt = min(kFarT, a.nl - t0);
  double* xr = (double*)sm;          // 3p
  double* xcn = xr + 3 * p;          // 3p
  double2* acc = (double2*)(xcn + 3 * p);  // p * kFarT
  double2* B = acc + p * kFarT;            // p * kFarT
  double2* S = B + p * kFarT;              // rb * p
  const int rb = max(1, min(p, 4096 / p));
  for (int i = threadIdx.x; i < p * kFarT; i += blockDim.x) acc[i] = make_double2(0.0, 0.0);
  for (int i = threadIdx.x; i < p; i += blockDim.x) {
    const double* x = a.xi + (int64_t)r * 3 * m;
    xr[3 * i] = x[i % m]; xr[3 * i + 1] = x[m + (i / m) % m]; xr[3 * i + 2] = x[2 * m + i / (m * m)];
  }
  __syncthreads();
  for (int bi = a.far_ptr[r]; bi < a.far_ptr[r + 1]; ++bi) {
    const int b = a.far_sorted[bi];
    const int c = a.far_c[b];
    for (int i = threadIdx.x; i < p; i += blockDim.x) {
      const double* x = a.xi + (int64_t)c * 3 * m;
      xcn[3 * i] = x[i % m]; xcn[3 * i + 1] = x[m + (i / m) % m]; xcn[3 * i + 2] = x[2 * m + i / (m * m)];
    }
    __syncthreads();
    const double2* xh = a.xhat + ((int64_t)c * a.nl + t0) * p;
    if (a.mode == BEM_MODE_H2ONLY) {
      // plain H^2: coupling S_b(s_l) evaluated per frequency
      for (int idx = threadIdx.x; idx < p * nt; idx += blockDim.x) {
        const int t = idx / p, mu = idx % p;
        const double2 sv = a.s[a.local_l[t0 + t]];
        double2 v = acc[mu * kFarT + t];
        for (int nu = 0; nu < p; ++nu) {
          const double dx = xcn[3 * nu] - xr[3 * mu], dy = xcn[3 * nu + 1] - xr[3 * mu + 1],
                       dz = xcn[3 * nu + 2] - xr[3 * mu + 2];
          v = cmadd(v, kern(sqrt(dx * dx + dy * dy + dz * dz), sv), xh[(int64_t)t * p + nu]);
        }
        acc[mu * kFarT + t] = v;
      }
      __syncthreads();
      continue;
    }
    const int rk = a.rank[b];
    const double2* Zb = a.Z + a.zoff[b];
    for (int l = 0; l < rk; ++l) {
      const double2 sv = a.s[a.pivk[(int64_t)b * a.rcap + l]];
      for (int idx = threadIdx.x; idx < p * kFarT; idx += blockDim.x) {
        const int nu = idx / kFarT, t = idx % kFarT;
        double2 v = make_double2(0.0, 0.0);
        if (t < nt) {
          const double2 z = Zb[(int64_t)l * a.nl + t0 + t];
          const double2 xv = xh[(int64_t)t * p + nu];
          v = make_double2(z.x * xv.x - z.y * xv.y, z.x * xv.y + z.y * xv.x);
        }
        B[idx] = v;
      }
      for (int mu0 = 0; mu0 < p; mu0 += rb) {
        const int nr = min(rb, p - mu0);
        __syncthreads();
        for (int idx = threadIdx.x; idx < nr * p; idx += blockDim.x) {
          const int mu = mu0 + idx / p, nu = idx % p;
          const double dx = xcn[3 * nu] - xr[3 * mu], dy = xcn[3 * nu + 1] - xr[3 * mu + 1],
                       dz = xcn[3 * nu + 2] - xr[3 * mu + 2];
          S[idx] = kern(sqrt(dx * dx + dy * dy + dz * dz), sv);
        }
        __syncthreads();
        for (int idx = threadIdx.x; idx < nr * kFarT; idx += blockDim.x) {
          const int mu = mu0 + idx / kFarT, t = idx % kFarT;
          double2 v = acc[mu * kFarT + t];
          const double2* Sr = S + (mu - mu0) * p;
          for (int nu = 0; nu < p; ++nu) v = cmadd(v, Sr[nu], B[nu * kFarT + t]);
          acc[mu * kFarT + t] = v;
        }
      }
      __syncthreads();
    }
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < p * nt; idx += blockDim.x) {
    const int t = idx / p, mu = idx % p;
    a.yhat[((int64_t)r * a.nl + t0 + t) * p + mu] = acc[mu * kFarT + t];
  }
}

}  // namespace

bem_status apply_launch(Op& op, const double* xin, double* yout, cudaStream_t st) {
  Tree& t = *op.tree;
  const int64_t M = t.M;
  const int nl = op.n_local, p = t.p;
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
  }
  const int64_t tot = M * nl;
  gather_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(x, xc, t.d_perm.p, M, nl);
  BEM_CK(cudaGetLastError());
  // K1
  NearArgs na;
  na.M = M; na.nl = nl; na.n_class = op.n_class; na.leaf_of = t.d_leaf_of.p;
  const bool dense = op.mode == BEM_MODE_DENSE;
  na.near_ptr = dense ? op.d_dn_ptr.p : t.d_near_ptr.p;
  na.near_cb = dense ? op.d_dn_cb.p : t.d_near_cb.p;
  na.near_ce = dense ? op.d_dn_ce.p : t.d_near_ce.p;
  na.cen = t.d_cen.p; na.qn = t.d_qn.p; na.qw = t.d_qw.p; na.selfJ = t.d_selfJ.p;
  na.s = (const double2*)op.d_s.p; na.local_l = op.d_local_l.p;
  na.class_t1 = op.d_class_t1.p; na.class_t2 = op.d_class_t2.p; na.xc = xc; na.yc = yc;
  dim3 ng((unsigned)((M + kNearWarps - 1) / kNearWarps), (unsigned)((op.n_class + kNearF - 1) / kNearF));
  near_kernel<<<ng, kNearWarps * 32, 0, st>>>(na);
  BEM_CK(cudaGetLastError());
  if (prof) BEM_CK(cudaEventRecord(op.ev[1], st));
  const bool has_far = !dense && !t.far_r.empty();
  const unsigned tt = (unsigned)((nl + kPassT - 1) / kPassT);
  if (has_far) {
    up_leaf_kernel<<<dim3((unsigned)t.n_leaves, tt), kPassThreads, 0, st>>>(t.d_leaves.p, t.d_begin.p, t.d_end.p,
                                                                             t.d_W.p, xc, xhat, M, nl, p);
    BEM_CK(cudaGetLastError());
    for (int lv = t.depth - 1; lv >= 0; --lv) {
      const int n = (int)t.level_nonleaf[lv].size();
      if (n == 0) continue;
      up_transfer_kernel<<<dim3((unsigned)n, tt), kPassThreads, 0, st>>>(t.d_level_nonleaf[lv].p, t.d_son0.p,
                                                                         t.d_son1.p, t.d_E.p, xhat, nl, p);
      BEM_CK(cudaGetLastError());
    }
    if (prof) BEM_CK(cudaEventRecord(op.ev[2], st));
    FarArgs fa;
    fa.C = t.C; fa.nl = nl; fa.m = t.m; fa.p = p; fa.mode = op.mode; fa.rcap = op.rcap;
    fa.far_ptr = t.d_far_ptr.p; fa.far_sorted = t.d_far_sorted.p; fa.far_c = t.d_far_c.p; fa.xi = t.d_xi.p;
    fa.s = (const double2*)op.d_s.p; fa.local_l = op.d_local_l.p; fa.rank = op.d_rank.p; fa.pivk = op.d_pivk.p;
    fa.zoff = op.d_zoff.p; fa.Z = (const double2*)op.d_Z.p; fa.xhat = xhat; fa.yhat = yhat;
    const int rb = std::max(1, std::min(p, 4096 / p));
    const size_t smem = sizeof(double) * 6 * p + sizeof(double2) * (2 * (size_t)p * kFarT + (size_t)rb * p);
    BEM_CK(cudaFuncSetAttribute(far_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    far_kernel<<<dim3((unsigned)t.C, (unsigned)((nl + kFarT - 1) / kFarT)), kFarThreads, smem, st>>>(fa);
    BEM_CK(cudaGetLastError());
    if (prof) BEM_CK(cudaEventRecord(op.ev[3], st));
    for (int lv = 0; lv < t.depth; ++lv) {
      const int n = (int)t.level_nonleaf[lv].size();
      if (n == 0) continue;
      down_transfer_kernel<<<dim3((unsigned)n, tt), kPassThreads, 0, st>>>(t.d_level_nonleaf[lv].p, t.d_son0.p,
                                                                           t.d_son1.p, t.d_E.p, yhat, nl, p);
      BEM_CK(cudaGetLastError());
    }
    down_leaf_kernel<<<dim3((unsigned)t.n_leaves, tt), kPassThreads, 0, st>>>(
        t.d_leaves.p, t.d_begin.p, t.d_end.p, t.d_U.p, yhat, yc, t.d_perm.p, y, M, nl, p, 1);
    BEM_CK(cudaGetLastError());
  } else {
    if (prof) { BEM_CK(cudaEventRecord(op.ev[2], st)); BEM_CK(cudaEventRecord(op.ev[3], st)); }
    scatter_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(yc, y, t.d_perm.p, M, nl);
    BEM_CK(cudaGetLastError());
  }
  if (prof) BEM_CK(cudaEventRecord(op.ev[4], st));
  return BEM_OK;
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
  return apply_launch(op, (const double*)x, (double*)y, (cudaStream_t)cuda_stream);
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
  oh->o.profile = enable != 0;
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
