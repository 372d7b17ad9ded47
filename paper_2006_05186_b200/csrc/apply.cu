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

}  // namespace

// y = V x (dl = false) or y = (alpha I + K) x (dl = true, double layer, NEXT-1): the
// same coupling tensors / ACA skeleton, K's near field and column basis W^K
bem_status apply_launch(Op& op, const double* xin, double* yout, cudaStream_t st, bool dl, double alpha) {
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
  const bool dense = op.mode == BEM_MODE_DENSE;
  const bool has_far = !dense && !t.far_r.empty();
  // K1 (near field) and the far branch (K2 up, K3, K2 down transfers) are independent until
  // the leaf-level scatter: unless per-kernel timers are on, K1 runs on a side stream forked
  // from st (event fork/join, graph-capturable) so both kernels share the SMs' FP64 pipes
  const bool overlap = op.overlap && has_far && !prof;
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
  {
    bem_status rs = launch_near(op, xc, yc, sk1, dl);
    if (rs != BEM_OK) return rs;
  }
  if (overlap) BEM_CK(cudaEventRecord(op.ev_join, sk1));
  if (prof) BEM_CK(cudaEventRecord(op.ev[1], st));
  const unsigned tt = (unsigned)((nl + kPassT - 1) / kPassT);
  if (has_far) {
    up_leaf_kernel<<<dim3((unsigned)t.n_leaves, tt), kPassThreads, 0, st>>>(t.d_leaves.p, t.d_begin.p, t.d_end.p,
                                                                             dl ? t.d_WK.p : t.d_W.p, xc, xhat, M, nl, p);
    BEM_CK(cudaGetLastError());
    for (int lv = t.depth - 1; lv >= 0; --lv) {
      const int n = (int)t.level_nonleaf[lv].size();
      if (n == 0) continue;
      up_transfer_kernel<<<dim3((unsigned)n, tt), kPassThreads, 0, st>>>(t.d_level_nonleaf[lv].p, t.d_son0.p,
                                                                         t.d_son1.p, t.d_E.p, xhat, nl, p);
      BEM_CK(cudaGetLastError());
    }
    if (prof) BEM_CK(cudaEventRecord(op.ev[2], st));
    bem_status rs = launch_far(op, xhat, yhat, st);
    if (rs != BEM_OK) return rs;
    if (prof) BEM_CK(cudaEventRecord(op.ev[3], st));
    for (int lv = 0; lv < t.depth; ++lv) {
      const int n = (int)t.level_nonleaf[lv].size();
      if (n == 0) continue;
      down_transfer_kernel<<<dim3((unsigned)n, tt), kPassThreads, 0, st>>>(t.d_level_nonleaf[lv].p, t.d_son0.p,
                                                                           t.d_son1.p, t.d_ET.p, yhat, nl, p);
      BEM_CK(cudaGetLastError());
    }
    if (overlap) BEM_CK(cudaStreamWaitEvent(st, op.ev_join, 0));
    down_leaf_kernel<<<dim3((unsigned)t.n_leaves, tt), kPassThreads, 0, st>>>(
        t.d_leaves.p, t.d_begin.p, t.d_end.p, t.d_UT.p, yhat, yc, t.d_perm.p, y, M, nl, p, 1, xc, dl ? alpha : 0.0);
    BEM_CK(cudaGetLastError());
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
  Tree& t = *op.tree;
  const unsigned tt = (unsigned)((ncols + kPassT - 1) / kPassT);
  up_leaf_kernel<<<dim3((unsigned)t.n_leaves, tt), kPassThreads, 0, st>>>(t.d_leaves.p, t.d_begin.p, t.d_end.p, t.d_W.p,
                                                                           xc, xhat, t.M, ncols, t.p);
  BEM_CK(cudaGetLastError());
  for (int lv = t.depth - 1; lv >= 0; --lv) {
    const int n = (int)t.level_nonleaf[lv].size();
    if (n == 0) continue;
    up_transfer_kernel<<<dim3((unsigned)n, tt), kPassThreads, 0, st>>>(t.d_level_nonleaf[lv].p, t.d_son0.p,
                                                                       t.d_son1.p, t.d_E.p, xhat, ncols, t.p);
    BEM_CK(cudaGetLastError());
  }
  return BEM_OK;
}

// y (input order) = ycn + U-side of the downward pass of yhat
bem_status h2_down_scatter(Op& op, double2* yhat, const double2* ycn, double2* y, int ncols, cudaStream_t st) {
  Tree& t = *op.tree;
  const unsigned tt = (unsigned)((ncols + kPassT - 1) / kPassT);
  if (t.far_r.empty()) {
    const int64_t tot = t.M * ncols;
    scatter_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(ycn, y, t.d_perm.p, t.M, ncols, ycn, 0.0);
    BEM_CK(cudaGetLastError());
    return BEM_OK;
  }
  for (int lv = 0; lv < t.depth; ++lv) {
    const int n = (int)t.level_nonleaf[lv].size();
    if (n == 0) continue;
    down_transfer_kernel<<<dim3((unsigned)n, tt), kPassThreads, 0, st>>>(t.d_level_nonleaf[lv].p, t.d_son0.p,
                                                                         t.d_son1.p, t.d_ET.p, yhat, ncols, t.p);
    BEM_CK(cudaGetLastError());
  }
  down_leaf_kernel<<<dim3((unsigned)t.n_leaves, tt), kPassThreads, 0, st>>>(
      t.d_leaves.p, t.d_begin.p, t.d_end.p, t.d_UT.p, yhat, ycn, t.d_perm.p, y, t.M, ncols, t.p, 1, ycn, 0.0);
  BEM_CK(cudaGetLastError());
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
