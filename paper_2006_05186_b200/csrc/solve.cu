// cqm_solve: frequency-decoupled CQM solve of V phi = g (Remark P:1607-1614;
// reading D10).  All local frequencies iterate in lockstep through one
// multi-frequency apply per inner iteration; converged frequencies are masked.
// GMRES(restart) from x0 = 0, classical Gram-Schmidt with one
// re-orthogonalisation, complex Givens rotations, per-frequency stop
// ||b - A x|| <= tol ||b||.  BLAS-1 work runs in the kernels below (one CTA per
// (frequency, basis vector) reduction, deterministic tree order); the host
// only reads a per-frequency "still active" count each iteration.
#include <cmath>
#include <vector>

#include <functional>

#include "common.cuh"

namespace bem {
namespace {

constexpr int kRed = 256;

__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 cmulk(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 cconjmul(double2 a, double2 b) {  // conj(a) b
  return make_double2(a.x * b.x + a.y * b.y, a.x * b.y - a.y * b.x);
}

template <class T>
__device__ T block_sum(T v, T* sh) {
  sh[threadIdx.x] = v;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) sh[threadIdx.x] = sh[threadIdx.x] + sh[threadIdx.x + s];
    __syncthreads();
  }
  T r = sh[0];
  __syncthreads();
  return r;
}

struct D2 {
  double x, y;
  __device__ D2 operator+(const D2& o) const { return D2{x + o.x, y + o.y}; }
};

// h[t][i] = <V_i[t], w[t]> for i < ni ; grid (nl, ni)
__global__ void __launch_bounds__(kRed) dots_kernel(const double2* __restrict__ V, const double2* __restrict__ w,
                                                    double2* __restrict__ h, int64_t M, int nl, int ldh) {
  __shared__ D2 sh[kRed];
  const int t = blockIdx.x, i = blockIdx.y;
  const double2* v = V + ((int64_t)i * nl + t) * M;
  const double2* ww = w + (int64_t)t * M;
  D2 acc{0.0, 0.0};
  for (int64_t k = threadIdx.x; k < M; k += blockDim.x) {
    const double2 p = cconjmul(v[k], ww[k]);
    acc.x += p.x; acc.y += p.y;
  }
  acc = block_sum(acc, sh);
  if (threadIdx.x == 0) h[(int64_t)t * ldh + i] = make_double2(acc.x, acc.y);
}

// w[t] -= sum_i h[t][i] V_i[t]; Hacc[t][i*ldH + j] += h[t][i] (pass accumulation)
__global__ void orth_update_kernel(const double2* __restrict__ V, const double2* __restrict__ h, double2* __restrict__ w,
                                   int64_t M, int nl, int ni, int ldh) {
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= M * nl) return;
  const int t = (int)(idx / M);
  const int64_t k = idx - (int64_t)t * M;
  double2 acc = w[idx];
  for (int i = 0; i < ni; ++i) {
    const double2 hv = h[(int64_t)t * ldh + i];
    const double2 v = V[((int64_t)i * nl + t) * M + k];
    acc.x -= hv.x * v.x - hv.y * v.y;
    acc.y -= hv.x * v.y + hv.y * v.x;
  }
  w[idx] = acc;
}

__global__ void __launch_bounds__(kRed) norm_kernel(const double2* __restrict__ w, double* __restrict__ nrm, int64_t M) {
  __shared__ double sh[kRed];
  const int t = blockIdx.x;
  double acc = 0.0;
  for (int64_t k = threadIdx.x; k < M; k += blockDim.x) {
    const double2 v = w[(int64_t)t * M + k];
    acc += v.x * v.x + v.y * v.y;
  }
  acc = block_sum(acc, sh);
  if (threadIdx.x == 0) nrm[t] = sqrt(acc);
}

__global__ void scale_kernel(const double2* __restrict__ w, const double* __restrict__ nrm, double2* __restrict__ out,
                             int64_t M, int nl) {
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= M * nl) return;
  const int t = (int)(idx / M);
  const double n = nrm[t];
  const double2 v = w[idx];
  out[idx] = n > 0.0 ? make_double2(v.x / n, v.y / n) : make_double2(0.0, 0.0);
}

__global__ void axpby_kernel(const double2* __restrict__ b, const double2* __restrict__ ax, double2* __restrict__ r,
                             int64_t n) {  // r = b - ax
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) r[i] = make_double2(b[i].x - ax[i].x, b[i].y - ax[i].y);
}

// cycle start: g[t] = (beta, 0...), jt = 0, cyc_active = active && beta > tol*bnorm
__global__ void cycle_init_kernel(const double* __restrict__ beta, const double* __restrict__ bnorm, double tol,
                                  int* __restrict__ active, int* __restrict__ cyc, int* __restrict__ jt,
                                  double2* __restrict__ g, double2* __restrict__ H, int nl, int restart,
                                  int* __restrict__ n_active) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nl) return;
  if (active[t] && beta[t] <= tol * bnorm[t]) active[t] = 0;
  cyc[t] = active[t];
  jt[t] = 0;
  for (int i = 0; i <= restart; ++i) g[(int64_t)t * (restart + 1) + i] = make_double2(i == 0 ? beta[t] : 0.0, 0.0);
  for (int i = 0; i < (restart + 1) * restart; ++i) H[(int64_t)t * (restart + 1) * restart + i] = make_double2(0.0, 0.0);
  if (active[t]) atomicAdd(n_active, 1);
}

// add the two CGS passes into column j of H
__global__ void hacc_kernel(const double2* __restrict__ h, double2* __restrict__ H, int nl, int ni, int ldh, int j,
                            int restart) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nl) return;
  for (int i = 0; i < ni; ++i) {
    double2& Hij = H[(int64_t)t * (restart + 1) * restart + (int64_t)i * restart + j];
    Hij = cadd(Hij, h[(int64_t)t * ldh + i]);
  }
}

__global__ void givens_kernel(double2* __restrict__ H, double2* __restrict__ g, double2* __restrict__ cs,
                              double2* __restrict__ sn, const double* __restrict__ hn, const double* __restrict__ bnorm,
                              int* __restrict__ cyc, int* __restrict__ jt, int* __restrict__ iters, double tol, int j,
                              int restart, int nl, int* __restrict__ n_active) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nl || !cyc[t]) return;
  double2* Ht = H + (int64_t)t * (restart + 1) * restart;
  double2* gt = g + (int64_t)t * (restart + 1);
  double2* ct = cs + (int64_t)t * restart;
  double2* st = sn + (int64_t)t * restart;
  Ht[(int64_t)(j + 1) * restart + j] = make_double2(hn[t], 0.0);
  for (int i = 0; i < j; ++i) {
    const double2 a = Ht[(int64_t)i * restart + j], b = Ht[(int64_t)(i + 1) * restart + j];
    const double2 c = ct[i], s = st[i];
    // [c s; -conj(s) c] with real c
    Ht[(int64_t)i * restart + j] = cadd(make_double2(c.x * a.x, c.x * a.y), cmulk(s, b));
    const double2 ms = make_double2(-s.x, s.y);  // -conj(s)
    Ht[(int64_t)(i + 1) * restart + j] = cadd(cmulk(ms, a), make_double2(c.x * b.x, c.x * b.y));
  }
  const double2 a = Ht[(int64_t)j * restart + j], b = Ht[(int64_t)(j + 1) * restart + j];
  const double na = hypot(a.x, a.y), nb = hypot(b.x, b.y);
  const double den = hypot(na, nb);
  double2 c, s;
  if (den == 0.0) { c = make_double2(1.0, 0.0); s = make_double2(0.0, 0.0); }
  else if (na == 0.0) { c = make_double2(0.0, 0.0); s = make_double2(b.x / nb, -b.y / nb); }
  else {
    c = make_double2(na / den, 0.0);
    const double2 ua = make_double2(a.x / na, a.y / na);
    s = cmulk(ua, make_double2(b.x / den, -b.y / den));
  }
  ct[j] = c; st[j] = s;
  Ht[(int64_t)j * restart + j] = cadd(make_double2(c.x * a.x, c.x * a.y), cmulk(s, b));
  Ht[(int64_t)(j + 1) * restart + j] = make_double2(0.0, 0.0);
  const double2 gj = gt[j];
  gt[j + 1] = cmulk(make_double2(-s.x, s.y), gj);
  gt[j] = make_double2(c.x * gj.x, c.x * gj.y);
  jt[t] = j + 1;
  iters[t] += 1;
  const double res = hypot(gt[j + 1].x, gt[j + 1].y);
  if (res <= tol * bnorm[t]) cyc[t] = 0;
  else atomicAdd(n_active, 1);
}

// y = H^{-1} g (upper triangular, jt[t] columns), then x += V y
__global__ void trisolve_kernel(const double2* __restrict__ H, const double2* __restrict__ g, double2* __restrict__ y,
                                const int* __restrict__ jt, int restart, int nl) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nl) return;
  const double2* Ht = H + (int64_t)t * (restart + 1) * restart;
  const double2* gt = g + (int64_t)t * (restart + 1);
  double2* yt = y + (int64_t)t * restart;
  const int n = jt[t];
  for (int i = restart - 1; i >= n; --i) yt[i] = make_double2(0.0, 0.0);
  for (int i = n - 1; i >= 0; --i) {
    double2 acc = gt[i];
    for (int k = i + 1; k < n; ++k) {
      const double2 p = cmulk(Ht[(int64_t)i * restart + k], yt[k]);
      acc.x -= p.x; acc.y -= p.y;
    }
    const double2 d = Ht[(int64_t)i * restart + i];
    const double dd = d.x * d.x + d.y * d.y;
    yt[i] = make_double2((acc.x * d.x + acc.y * d.y) / dd, (acc.y * d.x - acc.x * d.y) / dd);
  }
}

__global__ void xupdate_kernel(const double2* __restrict__ V, const double2* __restrict__ y, const int* __restrict__ jt,
                               double2* __restrict__ x, int64_t M, int nl, int restart) {
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= M * nl) return;
  const int t = (int)(idx / M);
  const int64_t k = idx - (int64_t)t * M;
  double2 acc = x[idx];
  for (int i = 0; i < jt[t]; ++i) {
    const double2 p = cmulk(y[(int64_t)t * restart + i], V[((int64_t)i * nl + t) * M + k]);
    acc.x += p.x; acc.y += p.y;
  }
  x[idx] = acc;
}

__global__ void real_to_complex_kernel(const double* __restrict__ a, double2* __restrict__ b, int64_t n) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) b[i] = make_double2(a[i], 0.0);
}

__global__ void __launch_bounds__(kRed) complex_to_real_kernel(const double2* __restrict__ a, double* __restrict__ b,
                                                               int64_t n, double* __restrict__ mx) {
  __shared__ double sh[2 * kRed];
  double mi = 0.0, mr = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double2 v = a[i];
    b[i] = v.x;
    mi = fmax(mi, fabs(v.y));
    mr = fmax(mr, hypot(v.x, v.y));
  }
  sh[threadIdx.x] = mi;
  sh[kRed + threadIdx.x] = mr;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      sh[threadIdx.x] = fmax(sh[threadIdx.x], sh[threadIdx.x + s]);
      sh[kRed + threadIdx.x] = fmax(sh[kRed + threadIdx.x], sh[kRed + threadIdx.x + s]);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    atomicMax((unsigned long long*)&mx[0], __double_as_longlong(sh[0]));
    atomicMax((unsigned long long*)&mx[1], __double_as_longlong(sh[kRed]));
  }
}

inline unsigned nblk(int64_t n) { return (unsigned)((n + 255) / 256); }

}  // namespace
}  // namespace bem

using namespace bem;

namespace bem {
namespace {

// Batched restarted GMRES over the op's local frequencies (frequency domain,
// input panel order): solves V(s_l) X_t = B_t for every local t.  B, X:
// device [n_local][M] complex.  Writes per-frequency iteration counts and the
// final relative residuals (host vectors).
// Generic batched GMRES core: apply(x, w) computes w = A_t x_t for all nl columns
// ([nl][M] complex); set_mask(mask) tells the operator which columns may skip work.
template <class ApplyFn, class MaskFn>
bem_status gmres_core(int64_t M, int nl, ApplyFn apply, MaskFn set_mask, bool use_mask, const double2* B, double2* X,
                      double tol, int restart, int max_iter, cudaStream_t st, std::vector<int>& hit,
                      std::vector<double>& hrel, GmresWs& ws) {
  Nvtx nv("a9 GMRES");
  const int64_t n = M * nl;
  if (ws.n != n || ws.nl != nl || ws.restart != restart) {  // (re)allocate the workspace
    BEM_CK(ws.r.alloc(2 * n));
    BEM_CK(ws.w.alloc(2 * n)); BEM_CK(ws.V.alloc(2 * n * (restart + 1)));
    BEM_CK(ws.h.alloc(2 * (size_t)nl * (restart + 1))); BEM_CK(ws.H.alloc(2 * (size_t)nl * (restart + 1) * restart));
    BEM_CK(ws.g.alloc(2 * (size_t)nl * (restart + 1))); BEM_CK(ws.cs.alloc(2 * (size_t)nl * restart));
    BEM_CK(ws.sn.alloc(2 * (size_t)nl * restart)); BEM_CK(ws.y.alloc(2 * (size_t)nl * restart));
    BEM_CK(ws.beta.alloc(nl)); BEM_CK(ws.bnorm.alloc(nl)); BEM_CK(ws.hn.alloc(nl));
    BEM_CK(ws.active.alloc(nl)); BEM_CK(ws.cyc.alloc(nl)); BEM_CK(ws.jt.alloc(nl)); BEM_CK(ws.iters.alloc(nl));
    BEM_CK(ws.cnt.alloc(1));
    ws.n = n; ws.nl = nl; ws.restart = restart;
  }
  DBuf<double>&r = ws.r, &w = ws.w, &V = ws.V, &h = ws.h, &H = ws.H, &g = ws.g, &cs = ws.cs, &sn = ws.sn, &y = ws.y;
  DBuf<double>&beta = ws.beta, &bnorm = ws.bnorm, &hn = ws.hn;
  DBuf<int>&active = ws.active, &cyc = ws.cyc, &jt = ws.jt, &iters = ws.iters, &cnt = ws.cnt;
  double2* Rr = (double2*)r.p; double2* Wv = (double2*)w.p;
  double2* VV = (double2*)V.p;
  // converged frequencies skip the K1 / K3 work of later applies (mask)
  struct MaskGuard {
    MaskFn& f;
    ~MaskGuard() { f(nullptr); }
  } mask_guard{set_mask};
  norm_kernel<<<nl, kRed, 0, st>>>(B, bnorm.p, M);
  BEM_CK(cudaMemsetAsync(X, 0, sizeof(double2) * n, st));
  BEM_CK(cudaMemsetAsync(iters.p, 0, sizeof(int) * nl, st));
  {
    std::vector<int> ones(nl, 1);
    BEM_CK(cudaMemcpyAsync(active.p, ones.data(), sizeof(int) * nl, cudaMemcpyHostToDevice, st));
    BEM_CK(cudaStreamSynchronize(st));
  }
  int total = 0;
  bem_status rs;
  for (;;) {
    // r = b - A x ; beta = ||r||
    set_mask(use_mask ? active.p : nullptr);
    rs = apply((const double*)X, w.p);
    if (rs != BEM_OK) return rs;
    axpby_kernel<<<nblk(n), 256, 0, st>>>(B, Wv, Rr, n);
    norm_kernel<<<nl, kRed, 0, st>>>(Rr, beta.p, M);
    BEM_CK(cudaMemsetAsync(cnt.p, 0, sizeof(int), st));
    cycle_init_kernel<<<nblk(nl), 256, 0, st>>>(beta.p, bnorm.p, tol, active.p, cyc.p, jt.p, (double2*)g.p,
                                                (double2*)H.p, nl, restart, cnt.p);
    BEM_CK(cudaGetLastError());
    int hcnt = 0;
    BEM_CK(cudaMemcpyAsync(&hcnt, cnt.p, sizeof(int), cudaMemcpyDeviceToHost, st));
    BEM_CK(cudaStreamSynchronize(st));
    if (hcnt == 0 || total >= max_iter) break;
    scale_kernel<<<nblk(n), 256, 0, st>>>(Rr, beta.p, VV, M, nl);
    for (int j = 0; j < restart && total < max_iter; ++j) {
      set_mask(use_mask ? cyc.p : nullptr);
      rs = apply((const double*)(VV + (int64_t)j * n), w.p);
      if (rs != BEM_OK) return rs;
      ++total;
      for (int pass = 0; pass < 2; ++pass) {
        dots_kernel<<<dim3(nl, j + 1), kRed, 0, st>>>(VV, Wv, (double2*)h.p, M, nl, restart + 1);
        orth_update_kernel<<<nblk(n), 256, 0, st>>>(VV, (double2*)h.p, Wv, M, nl, j + 1, restart + 1);
        hacc_kernel<<<nblk(nl), 256, 0, st>>>((double2*)h.p, (double2*)H.p, nl, j + 1, restart + 1, j, restart);
      }
      norm_kernel<<<nl, kRed, 0, st>>>(Wv, hn.p, M);
      scale_kernel<<<nblk(n), 256, 0, st>>>(Wv, hn.p, VV + (int64_t)(j + 1) * n, M, nl);
      BEM_CK(cudaMemsetAsync(cnt.p, 0, sizeof(int), st));
      givens_kernel<<<nblk(nl), 256, 0, st>>>((double2*)H.p, (double2*)g.p, (double2*)cs.p, (double2*)sn.p, hn.p,
                                              bnorm.p, cyc.p, jt.p, iters.p, tol, j, restart, nl, cnt.p);
      BEM_CK(cudaGetLastError());
      BEM_CK(cudaMemcpyAsync(&hcnt, cnt.p, sizeof(int), cudaMemcpyDeviceToHost, st));
      BEM_CK(cudaStreamSynchronize(st));
      if (hcnt == 0) break;
    }
    trisolve_kernel<<<nblk(nl), 256, 0, st>>>((double2*)H.p, (double2*)g.p, (double2*)y.p, jt.p, restart, nl);
    xupdate_kernel<<<nblk(n), 256, 0, st>>>(VV, (double2*)y.p, jt.p, X, M, nl, restart);
    BEM_CK(cudaGetLastError());
  }
  if (use_mask) {  // true final residuals of every frequency (the last masked apply zeroed converged ones)
    set_mask(nullptr);
    rs = apply((const double*)X, w.p);
    if (rs != BEM_OK) return rs;
    axpby_kernel<<<nblk(n), 256, 0, st>>>(B, Wv, Rr, n);
    norm_kernel<<<nl, kRed, 0, st>>>(Rr, beta.p, M);
    BEM_CK(cudaGetLastError());
  }
  std::vector<double> hb(nl), hbn(nl);
  hit.assign(nl, 0);
  hrel.assign(nl, 0.0);
  BEM_CK(cudaMemcpy(hb.data(), beta.p, sizeof(double) * nl, cudaMemcpyDeviceToHost));
  BEM_CK(cudaMemcpy(hbn.data(), bnorm.p, sizeof(double) * nl, cudaMemcpyDeviceToHost));
  BEM_CK(cudaMemcpy(hit.data(), iters.p, sizeof(int) * nl, cudaMemcpyDeviceToHost));
  for (int t = 0; t < nl; ++t) hrel[t] = hbn[t] > 0.0 ? hb[t] / hbn[t] : 0.0;
  return BEM_OK;
}

bem_status gmres_multifreq(Op& op, const double2* B, double2* X, double tol, int restart, int max_iter,
                           cudaStream_t st, std::vector<int>& hit, std::vector<double>& hrel) {
  auto apply = [&](const double* x, double* w) { return apply_launch(op, x, w, st); };
  auto set_mask = [&](const int32_t* m) { op.d_mask = m; };
  GmresWs ws;
  return gmres_core(op.tree->M, op.n_local, apply, set_mask, op.use_solve_mask, B, X, tol, restart, max_iter, st, hit,
                    hrel, ws);
}

bem_status finish_stats(const std::vector<int>& hit, const std::vector<double>& hrel, double tol, int max_iter,
                        double imag_rel, bem_solve_stats* stats) {
  int nunc = 0, imax = 0, isum = 0;
  double rmax = 0.0;
  for (size_t t = 0; t < hit.size(); ++t) {
    rmax = std::max(rmax, hrel[t]);
    if (hrel[t] > tol) ++nunc;
    imax = std::max(imax, hit[t]);
    isum += hit[t];
  }
  if (stats) {
    stats->iters_max = imax; stats->iters_sum = isum; stats->n_unconverged = nunc;
    stats->resid_max = rmax; stats->imag_rel_max = imag_rel;
  }
  if (nunc > 0) {
    set_error("GMRES: %d frequencies did not converge within max_iter=%d", nunc, max_iter);
    return BEM_ENOCONV;
  }
  return BEM_OK;
}

}  // namespace

bem_status gmres_fn(int64_t M, int nl, const std::function<bem_status(const double*, double*)>& apply,
                    const double2* B, double2* X, double tol, int restart, int max_iter, cudaStream_t st,
                    std::vector<int>& hit, std::vector<double>& hrel, GmresWs& ws) {
  auto set_mask = [](const int32_t*) {};
  return gmres_core(M, nl, apply, set_mask, false, B, X, tol, restart, max_iter, st, hit, hrel, ws);
}

bem_status solve_stats(const std::vector<int>& hit, const std::vector<double>& hrel, double tol, int max_iter,
                       double imag_rel, bem_solve_stats* stats) {
  return finish_stats(hit, hrel, tol, max_iter, imag_rel, stats);
}

// cqm_solve on G ranks: this rank's DOF shard g_time [L][M_loc] -> forward K4 + NCCL
// all-to-all -> batched GMRES on this rank's frequencies -> all-to-all + inverse K4.
bem_status solve_sharded(Op& op, const double* g_time, double* phi_time, int64_t M_loc, double R, double tol,
                         int restart, int max_iter, bem_comm c, cudaStream_t st, bem_solve_stats* stats) {
  BEM_REQ(tol > 0.0 && restart >= 1 && max_iter >= 1, "cqm_solve: bad tol/restart/max_iter");
  BEM_REQ(R > 0.0 && R < 1.0, "cqm_solve: R must lie in (0,1)");
  bem_status rs = comm_check(c, op, M_loc);
  if (rs != BEM_OK) return rs;
  DeviceGuard dg(op.tree->device);
  const int N = op.L - 1;
  const int64_t nt = M_loc * op.L, nf = op.tree->M * op.n_local;
  DBuf<double> tmpc, x, mx;
  BEM_CK(tmpc.alloc(2 * std::max<int64_t>(nt, 1))); BEM_CK(x.alloc(2 * std::max<int64_t>(nf, 1)));
  BEM_CK(mx.alloc(2));
  real_to_complex_kernel<<<nblk(nt), 256, 0, st>>>(g_time, (double2*)tmpc.p, nt);
  BEM_CK(cudaGetLastError());
  double2* gf = nullptr;
  rs = shard_forward(op, c, tmpc.p, R, &gf, st);
  if (rs != BEM_OK) return rs;
  std::vector<int> hit;
  std::vector<double> hrel;
  rs = gmres_multifreq(op, gf, (double2*)x.p, tol, restart, max_iter, st, hit, hrel);
  if (rs != BEM_OK) return rs;
  rs = shard_inverse(op, c, (const double2*)x.p, R, tmpc.p, st);
  if (rs != BEM_OK) return rs;
  BEM_CK(cudaMemsetAsync(mx.p, 0, sizeof(double) * 2, st));
  complex_to_real_kernel<<<1024, kRed, 0, st>>>((const double2*)tmpc.p, phi_time, nt, mx.p);
  BEM_CK(cudaGetLastError());
  // statistics over the ranks: max (iters_max, resid_max, max |Im|, max |phi|), sum (unconverged, iters)
  int nunc = 0, imax = 0;
  long long isum = 0;
  double rmax = 0.0;
  for (size_t t = 0; t < hit.size(); ++t) {
    rmax = std::max(rmax, hrel[t]);
    if (hrel[t] > tol) ++nunc;
    imax = std::max(imax, hit[t]);
    isum += hit[t];
  }
  double* red = comm_scratch(c);
  const double loc[6] = {(double)imax, rmax, 0.0, 0.0, (double)nunc, (double)isum};
  BEM_CK(cudaMemcpyAsync(red, loc, sizeof(loc), cudaMemcpyHostToDevice, st));
  BEM_CK(cudaMemcpyAsync(red + 2, mx.p, 2 * sizeof(double), cudaMemcpyDeviceToDevice, st));
  rs = comm_allreduce(c, red, 4, 2, st);
  if (rs != BEM_OK) return rs;
  double glob[6];
  BEM_CK(cudaMemcpyAsync(glob, red, sizeof(glob), cudaMemcpyDeviceToHost, st));
  BEM_CK(cudaStreamSynchronize(st));
  if (stats) {
    stats->iters_max = (int32_t)glob[0]; stats->resid_max = glob[1];
    stats->imag_rel_max = glob[3] > 0.0 ? glob[2] / glob[3] : 0.0;
    stats->n_unconverged = (int32_t)glob[4]; stats->iters_sum = (int32_t)glob[5];
  }
  if (glob[4] > 0) {
    set_error("cqm_solve: %d frequencies (all ranks) did not converge within max_iter=%d", (int)glob[4], max_iter);
    return BEM_ENOCONV;
  }
  return BEM_OK;
}

}  // namespace bem

extern "C" bem_status bem_solve_multifreq(bem_op oh, const bem_c128* g_freq, bem_c128* phi_freq, double tol,
                                          int32_t restart, int32_t max_iter, void* cuda_stream,
                                          bem_solve_stats* stats) {
  BEM_REQ(oh && g_freq && phi_freq, "bem_solve_multifreq: NULL argument");
  BEM_REQ(g_freq != phi_freq, "bem_solve_multifreq: in-place is not allowed");
  BEM_REQ(tol > 0.0 && restart >= 1 && max_iter >= 1, "bem_solve_multifreq: bad tol/restart/max_iter");
  Op& op = oh->o;
  DeviceGuard dg(op.tree->device);
  std::vector<int> hit;
  std::vector<double> hrel;
  bem_status rs = gmres_multifreq(op, (const double2*)g_freq, (double2*)phi_freq, tol, restart, max_iter,
                                  (cudaStream_t)cuda_stream, hit, hrel);
  if (rs != BEM_OK) return rs;
  return finish_stats(hit, hrel, tol, max_iter, 0.0, stats);
}

extern "C" bem_status cqm_solve(bem_op oh, const double* g_time, double* phi_time, int64_t M_loc, double R, double tol,
                                int32_t restart, int32_t max_iter, void* nccl_comm, void* cuda_stream,
                                bem_solve_stats* stats) {
  BEM_REQ(oh && g_time && phi_time, "cqm_solve: NULL argument");
  Op& op = oh->o;
  Tree& tr = *op.tree;
  if (nccl_comm != nullptr) return solve_sharded(op, g_time, phi_time, M_loc, R, tol, restart, max_iter,
                                                 (bem_comm)nccl_comm, (cudaStream_t)cuda_stream, stats);
  BEM_REQ(M_loc == tr.M, "cqm_solve: M_loc must equal the number of panels on a single device");
  BEM_REQ(op.n_local == op.L, "cqm_solve: the operator must hold all L frequencies");
  for (int t = 0; t < op.n_local; ++t) BEM_REQ(op.local_l[t] == t, "cqm_solve: local_l must be 0..L-1 in order");
  BEM_REQ(tol > 0.0 && restart >= 1 && max_iter >= 1, "cqm_solve: bad tol/restart/max_iter");
  BEM_REQ(R > 0.0 && R < 1.0, "cqm_solve: R must lie in (0,1)");
  DeviceGuard dg(tr.device);
  cudaStream_t st = (cudaStream_t)cuda_stream;
  const int64_t M = tr.M;
  const int nl = op.n_local, N = op.L - 1;
  const int64_t n = M * nl;
  DBuf<double> tmpc, b, x, mx;
  BEM_CK(tmpc.alloc(2 * n)); BEM_CK(b.alloc(2 * n)); BEM_CK(x.alloc(2 * n)); BEM_CK(mx.alloc(2));
  // g^ = forward(g)
  real_to_complex_kernel<<<nblk(n), 256, 0, st>>>(g_time, (double2*)tmpc.p, n);
  BEM_CK(cudaGetLastError());
  bem_status rs = fft_transform(tmpc.p, b.p, M, N, R, false, st);
  if (rs != BEM_OK) return rs;
  std::vector<int> hit;
  std::vector<double> hrel;
  rs = gmres_multifreq(op, (const double2*)b.p, (double2*)x.p, tol, restart, max_iter, st, hit, hrel);
  if (rs != BEM_OK) return rs;
  // phi = Re inverse(phi^)
  rs = fft_transform(x.p, tmpc.p, M, N, R, true, st);
  if (rs != BEM_OK) return rs;
  BEM_CK(cudaMemsetAsync(mx.p, 0, sizeof(double) * 2, st));
  complex_to_real_kernel<<<1024, kRed, 0, st>>>((const double2*)tmpc.p, phi_time, n, mx.p);
  BEM_CK(cudaGetLastError());
  double hmx[2] = {0, 0};
  BEM_CK(cudaMemcpyAsync(hmx, mx.p, sizeof(double) * 2, cudaMemcpyDeviceToHost, st));
  BEM_CK(cudaStreamSynchronize(st));
  return finish_stats(hit, hrel, tol, max_iter, hmx[1] > 0.0 ? hmx[0] / hmx[1] : 0.0, stats);
}
