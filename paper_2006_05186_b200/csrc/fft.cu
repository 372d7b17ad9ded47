// K4: batched R-scaled CQM transforms along the time/frequency axis
// (eq:omega_n P:436-441, eq:slphelm P:529-540; reading D2):
//   forward  X_l = sum_n R^n x_n w^{nl},             w = e^{-2 pi i/L}
//   inverse  y_n = R^{-n}/L sum_l Y_l w^{-nl}
// L = N+1 has large prime factors (33, 129, 257, 513, 1025), so each column
// is transformed by Bluestein's chirp-z identity nl = (n^2 + l^2 - (l-n)^2)/2:
//   out_j = post_j sum_i (in_i pre_i) h_{j-i}
// with chirp c_k = e^{-pi i (k^2 mod 2L)/L} (index reduced in integers), and
//   forward: pre_i = R^i c_i,   h_k = conj(c_k), post_j = c_j
//   inverse: pre_i = conj(c_i), h_k = c_k,       post_j = R^{-j} conj(c_j)/L.
// The length-L linear convolution runs as a power-of-two P >= 2L-1 radix-2
// FFT in shared memory, one CTA per group of DOF columns (coalesced row loads).
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <tuple>

#include "common.cuh"

namespace bem {
namespace {

struct Plan {
  int L = 0, P = 0, logP = 0;
  DBuf<double> pre, post, hhat, tw;  // complex arrays (interleaved)
};

std::mutex g_plan_mu;
std::map<std::tuple<int, int, uint64_t, int>, std::unique_ptr<Plan>> g_plans;

// host radix-2 FFT (plan construction only), sign = -1 forward
void host_fft(std::vector<double>& re, std::vector<double>& im, int sign) {
  const int n = (int)re.size();
  for (int i = 1, j = 0; i < n; ++i) {
    int bit = n >> 1;
    for (; j & bit; bit >>= 1) j ^= bit;
    j ^= bit;
    if (i < j) { std::swap(re[i], re[j]); std::swap(im[i], im[j]); }
  }
  for (int len = 2; len <= n; len <<= 1) {
    for (int i = 0; i < n; i += len)
      for (int k = 0; k < len / 2; ++k) {
        const double ang = sign * 2.0 * M_PI * (double)k / (double)len;
        const double wr = std::cos(ang), wi = std::sin(ang);
        const double ur = re[i + k], ui = im[i + k];
        const double vr = re[i + k + len / 2] * wr - im[i + k + len / 2] * wi;
        const double vi = re[i + k + len / 2] * wi + im[i + k + len / 2] * wr;
        re[i + k] = ur + vr; im[i + k] = ui + vi;
        re[i + k + len / 2] = ur - vr; im[i + k + len / 2] = ui - vi;
      }
  }
}

bem_status get_plan(int N, double R, bool inverse, Plan** out) {
  int dev = 0;
  cudaGetDevice(&dev);
  uint64_t rbits;
  std::memcpy(&rbits, &R, 8);
  auto key = std::make_tuple(dev, N, rbits, inverse ? 1 : 0);
  std::lock_guard<std::mutex> lk(g_plan_mu);
  auto it = g_plans.find(key);
  if (it != g_plans.end()) { *out = it->second.get(); return BEM_OK; }
  auto pl = std::make_unique<Plan>();
  const int L = N + 1;
  int P = 1, logP = 0;
  while (P < 2 * L - 1) { P <<= 1; ++logP; }
  pl->L = L; pl->P = P; pl->logP = logP;
  std::vector<double> cre(L), cim(L);
  for (int k = 0; k < L; ++k) {
    const long long k2 = ((long long)k * k) % (2LL * L);
    const double ang = M_PI * (double)k2 / (double)L;
    cre[k] = std::cos(ang); cim[k] = -std::sin(ang);
  }
  std::vector<double> pre(2 * L), post(2 * L), hr(P, 0.0), hi(P, 0.0), tw(P);
  for (int k = 0; k < L; ++k) {
    if (!inverse) {
      const double rk = std::pow(R, (double)k);
      pre[2 * k] = rk * cre[k]; pre[2 * k + 1] = rk * cim[k];
      post[2 * k] = cre[k]; post[2 * k + 1] = cim[k];
    } else {
      const double sc = std::pow(R, -(double)k) / (double)L;
      pre[2 * k] = cre[k]; pre[2 * k + 1] = -cim[k];
      post[2 * k] = sc * cre[k]; post[2 * k + 1] = -sc * cim[k];
    }
    const double h_re = cre[k], h_im = inverse ? cim[k] : -cim[k];
    hr[k] = h_re; hi[k] = h_im;
    if (k > 0) { hr[P - k] = h_re; hi[P - k] = h_im; }
  }
  host_fft(hr, hi, -1);
  std::vector<double> hh(2 * P);
  for (int k = 0; k < P; ++k) { hh[2 * k] = hr[k] / (double)P; hh[2 * k + 1] = hi[k] / (double)P; }
  for (int k = 0; k < P / 2; ++k) {
    const double ang = -2.0 * M_PI * (double)k / (double)P;
    tw[2 * k] = std::cos(ang); tw[2 * k + 1] = std::sin(ang);
  }
  BEM_CK(pl->pre.upload(pre));
  BEM_CK(pl->post.upload(post));
  BEM_CK(pl->hhat.upload(hh));
  BEM_CK(pl->tw.upload(tw));
  *out = pl.get();
  g_plans[key] = std::move(pl);
  return BEM_OK;
}

constexpr int kFftThreads = 256;

__device__ __forceinline__ double2 cm(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}

// in-place radix-2 DIT FFT of NC columns (bit-reversed input order assumed), up to three
// radix-2 stages per shared-memory pass: a thread loads the 8 (or 4 / 2) elements
// i0 + m * 2^s of one group, applies stages s, s+1, s+2 in registers and stores them
// back (stage s pairs (m, m+1), s+1 pairs (m, m+2), s+2 pairs (m, m+4)), so a
// P = 512 transform takes 3 passes and barriers instead of 9 (r01: K4 was bound by the
// per-stage shared-memory round trips).
// Shared-memory element swizzle within a column: bits 0-2 XOR bits 3-5. Every 8 threads
// of a radix-8 pass (h0 = 1, 8, 64) then touch 8 different 16-byte bank groups.
__device__ __forceinline__ int sw(int i) { return i ^ ((i >> 3) & 7); }

template <int G>  // elements per thread-group = 2^stages in this pass
__device__ __forceinline__ void fft_pass(double2* buf, int P, int s, int NC, const double2* __restrict__ tw,
                                         bool inv, const double2* __restrict__ post_mul) {
  const int h0 = 1 << s;                     // half-width of the first stage
  const int ngrp = NC * (P / G);
  for (int g = threadIdx.x; g < ngrp; g += blockDim.x) {
    const int col = g / (P / G), r = g - col * (P / G);
    const int pos0 = r & (h0 - 1), blk = r >> s;   // group = blk-th run of G*h0 elements
    double2* b = buf + (size_t)col * P;
    const int i0 = blk * (G * h0) + pos0;
    double2 e[G];
#pragma unroll
    for (int m = 0; m < G; ++m) e[m] = b[sw(i0 + m * h0)];
#pragma unroll
    for (int st = 0, span = 1; span < G; ++st, span <<= 1) {
      const int tstride = P >> (s + st + 1);
#pragma unroll
      for (int m = 0; m < G; ++m) {
        if (m & span) continue;                   // m is the upper element of its pair
        const int pos = pos0 + (m & (span - 1)) * h0;
        double2 w = tw[pos * tstride];
        if (inv) w.y = -w.y;
        const double2 u = e[m], v = cm(e[m + span], w);
        e[m] = make_double2(u.x + v.x, u.y + v.y);
        e[m + span] = make_double2(u.x - v.x, u.y - v.y);
      }
    }
    if (post_mul) {  // last pass of the forward transform: the filter spectrum, fused
#pragma unroll
      for (int m = 0; m < G; ++m) e[m] = cm(e[m], post_mul[i0 + m * h0]);
    }
#pragma unroll
    for (int m = 0; m < G; ++m) b[sw(i0 + m * h0)] = e[m];
  }
}

// post_mul (nullable): pointwise factor applied to the natural-order result in the last pass
__device__ void smem_fft(double2* buf, int P, int logP, int NC, const double2* __restrict__ tw, bool inv,
                         const double2* __restrict__ post_mul = nullptr) {
  int s = 0;
  for (; s + 3 <= logP; s += 3) {
    fft_pass<8>(buf, P, s, NC, tw, inv, s + 3 == logP ? post_mul : nullptr);
    __syncthreads();
  }
  if (logP - s == 2) {
    fft_pass<4>(buf, P, s, NC, tw, inv, post_mul);
    __syncthreads();
  } else if (logP - s == 1) {
    fft_pass<2>(buf, P, s, NC, tw, inv, post_mul);
    __syncthreads();
  }
}

// Decimation-in-frequency counterpart (natural-order input, bit-reversed output) for the
// inverse FFT of the convolution: the same element groups as fft_pass, stages from the
// largest half-width down, butterfly (u, v) -> (u + v, (u - v) w). Its bit-reversed output
// is read through the bit-reversed index in the store phase, so the convolution needs no
// permutation pass.
template <int G>
__device__ __forceinline__ void fft_pass_dif(double2* buf, int P, int s, int NC, const double2* __restrict__ tw,
                                             bool inv) {
  const int h0 = 1 << s;
  const int ngrp = NC * (P / G);
  for (int g = threadIdx.x; g < ngrp; g += blockDim.x) {
    const int col = g / (P / G), r = g - col * (P / G);
    const int pos0 = r & (h0 - 1), blk = r >> s;
    double2* b = buf + (size_t)col * P;
    const int i0 = blk * (G * h0) + pos0;
    double2 e[G];
#pragma unroll
    for (int m = 0; m < G; ++m) e[m] = b[sw(i0 + m * h0)];
#pragma unroll
    for (int span = G / 2; span >= 1; span >>= 1) {
      const int tstride = P / (2 * span * h0);
#pragma unroll
      for (int m = 0; m < G; ++m) {
        if (m & span) continue;
        const int pos = pos0 + (m & (span - 1)) * h0;
        double2 w = tw[pos * tstride];
        if (inv) w.y = -w.y;
        const double2 u = e[m], v = e[m + span];
        e[m] = make_double2(u.x + v.x, u.y + v.y);
        e[m + span] = cm(make_double2(u.x - v.x, u.y - v.y), w);
      }
    }
#pragma unroll
    for (int m = 0; m < G; ++m) b[sw(i0 + m * h0)] = e[m];
  }
}

__device__ void smem_fft_dif(double2* buf, int P, int logP, int NC, const double2* __restrict__ tw, bool inv) {
  const int full = logP / 3, rem = logP - 3 * full;
  if (rem == 2) {
    fft_pass_dif<4>(buf, P, 3 * full, NC, tw, inv);
    __syncthreads();
  } else if (rem == 1) {
    fft_pass_dif<2>(buf, P, 3 * full, NC, tw, inv);
    __syncthreads();
  }
  for (int k = full - 1; k >= 0; --k) {
    fft_pass_dif<8>(buf, P, 3 * k, NC, tw, inv);
    __syncthreads();
  }
}

// Row addressing of the transform's input and output: row r of the input is
// in_rows.p[r] (or in + r*M when in_rows == nullptr), likewise for the output.
// With row pointers into OTHER ranks' buffers (CUDA IPC / NVLink peer memory)
// the kernel performs the time<->frequency transform and the all-to-all
// transpose in one pass: the forward transform stores frequency row l of this
// rank's DOF columns straight into the owner of l (cqm_forward_rows), the
// inverse reads them back from the owners (cqm_inverse_rows).
constexpr int kMaxRows = 2048;
struct RowPtrs {
  double2* p[kMaxRows];
};

__global__ void __launch_bounds__(kFftThreads) bluestein_kernel(const double2* __restrict__ in, double2* __restrict__ out,
                                                               int64_t M, int L, int P, int logP, int NC,
                                                               const double2* __restrict__ pre,
                                                               const double2* __restrict__ post,
                                                               const double2* __restrict__ hhat,
                                                               const double2* __restrict__ tw,
                                                               const RowPtrs* __restrict__ in_rows,
                                                               const RowPtrs* __restrict__ out_rows) {
  extern __shared__ double2 buf[];
  const int64_t c0 = (int64_t)blockIdx.x * NC;
  const int nc = (int)min((int64_t)NC, M - c0);
  // load with pre-chirp into bit-reversed positions; zero padding
  for (int idx = threadIdx.x; idx < NC * P; idx += blockDim.x) {
    const int n = idx / NC, col = idx % NC;
    double2 v = make_double2(0.0, 0.0);
    if (n < L && col < nc) {
      const double2* row = in_rows ? in_rows->p[n] : in + (int64_t)n * M;
      v = cm(row[c0 + col], pre[n]);
    }
    const int rv = (int)(__brev((unsigned)n) >> (32 - logP));
    if (n < P) buf[(size_t)col * P + sw(rv)] = v;
  }
  __syncthreads();
  // forward FFT, then the filter spectrum (already scaled by 1/P), fused into its last pass
  smem_fft(buf, P, logP, NC, tw, false, hhat);
  smem_fft_dif(buf, P, logP, NC, tw, true);  // output in bit-reversed order
  for (int idx = threadIdx.x; idx < NC * L; idx += blockDim.x) {
    const int j = idx / NC, col = idx % NC;
    if (col < nc) {
      double2* row = out_rows ? out_rows->p[j] : out + (int64_t)j * M;
      const int jr = (int)(__brev((unsigned)j) >> (32 - logP));
      row[c0 + col] = cm(buf[(size_t)col * P + sw(jr)], post[j]);
    }
  }
}

}  // namespace

bem_status fft_transform_rows(const double* in, double* out, int64_t M, int N, double R, bool inverse, cudaStream_t st,
                              const RowPtrs* in_rows, const RowPtrs* out_rows) {
  Plan* pl = nullptr;
  bem_status rs = get_plan(N, R, inverse, &pl);
  if (rs != BEM_OK) return rs;
  static const int nc_elems = [] {  // columns x points per CTA (env BEM_FFT_ELEMS; r01 sweep: 2048 best)
    const char* e = getenv("BEM_FFT_ELEMS");
    return e ? std::max(64, atoi(e)) : 2048;
  }();
  const int NC = std::max(1, nc_elems / pl->P);
  const size_t smem = sizeof(double2) * (size_t)NC * pl->P;
  BEM_CK(cudaFuncSetAttribute(bluestein_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const unsigned grid = (unsigned)((M + NC - 1) / NC);
  bluestein_kernel<<<grid, kFftThreads, smem, st>>>((const double2*)in, (double2*)out, M, pl->L, pl->P, pl->logP, NC,
                                                    (const double2*)pl->pre.p, (const double2*)pl->post.p,
                                                    (const double2*)pl->hhat.p, (const double2*)pl->tw.p, in_rows,
                                                    out_rows);
  BEM_CK(cudaGetLastError());
  return BEM_OK;
}

bem_status fft_transform(const double* in, double* out, int64_t M, int N, double R, bool inverse, cudaStream_t st) {
  return fft_transform_rows(in, out, M, N, R, inverse, st, nullptr, nullptr);
}

// row tables live in device memory owned by a small per-thread cache (graph-safe:
// the table is written with cudaMemcpyAsync on the caller's stream before the kernel)
struct RowTable {
  DBuf<double> buf;  // sizeof(RowPtrs) bytes
};
static thread_local RowTable g_rows[2];

}  // namespace bem

using namespace bem;

static bem_status transform_entry(const bem_c128* in, bem_c128* out, int64_t M, int32_t N, double R, void* stream,
                                  bool inverse) {
  BEM_REQ(in && out, "cqm transform: NULL pointer");
  BEM_REQ(M >= 1 && N >= 1, "cqm transform: need M_loc >= 1 and N >= 1");
  BEM_REQ(R > 0.0 && R <= 1.0, "cqm transform: R must lie in (0,1]");
  const size_t bytes = (size_t)(N + 1) * M * 16;
  BEM_REQ((const char*)in + bytes <= (const char*)out || (const char*)out + bytes <= (const char*)in,
          "cqm transform: in-place / overlapping buffers are not supported");
  cudaPointerAttributes at;
  BEM_CK(cudaPointerGetAttributes(&at, in));
  BEM_REQ(at.type == cudaMemoryTypeDevice, "cqm transform: input must be device memory");
  DeviceGuard dg(at.device);
  BEM_CK(cudaPointerGetAttributes(&at, out));
  BEM_REQ(at.type == cudaMemoryTypeDevice, "cqm transform: output must be device memory");
  return fft_transform((const double*)in, (double*)out, M, N, R, inverse, (cudaStream_t)stream);
}

extern "C" bem_status cqm_forward(const bem_c128* x_time, bem_c128* x_freq, int64_t M_loc, int32_t N, double R,
                                  void* cuda_stream) {
  return transform_entry(x_time, x_freq, M_loc, N, R, cuda_stream, false);
}

extern "C" bem_status cqm_inverse(const bem_c128* y_freq, bem_c128* y_time, int64_t M_loc, int32_t N, double R,
                                  void* cuda_stream) {
  return transform_entry(y_freq, y_time, M_loc, N, R, cuda_stream, true);
}

// host pointer table -> device table (async on the stream; the host array is copied into
// pinned staging first, so the caller may reuse it immediately)
static bem_status upload_rows(int which, bem_c128* const* rows, int L, cudaStream_t st, const RowPtrs** dev) {
  static thread_local RowPtrs* staging[2] = {nullptr, nullptr};
  RowTable& tb = g_rows[which];
  if (!tb.buf.p) BEM_CK(tb.buf.alloc((sizeof(RowPtrs) + 7) / 8));
  if (!staging[which]) BEM_CK(cudaMallocHost((void**)&staging[which], sizeof(RowPtrs)));
  BEM_CK(cudaStreamSynchronize(st));  // the previous use of this staging slot has been consumed
  for (int r = 0; r < L; ++r) staging[which]->p[r] = (double2*)rows[r];
  BEM_CK(cudaMemcpyAsync(tb.buf.p, staging[which], sizeof(double2*) * (size_t)L, cudaMemcpyHostToDevice, st));
  *dev = (const RowPtrs*)tb.buf.p;
  return BEM_OK;
}

extern "C" bem_status cqm_forward_rows(const bem_c128* x_time, int64_t M_loc, bem_c128* const* out_rows, int32_t N,
                                       double R, void* cuda_stream) {
  BEM_REQ(x_time && out_rows, "cqm_forward_rows: NULL pointer");
  BEM_REQ(M_loc >= 1 && N >= 1 && N + 1 <= kMaxRows, "cqm_forward_rows: need M_loc >= 1 and 1 <= N < %d", kMaxRows);
  BEM_REQ(R > 0.0 && R <= 1.0, "cqm_forward_rows: R must lie in (0,1]");
  for (int r = 0; r <= N; ++r) BEM_REQ(out_rows[r] != nullptr, "cqm_forward_rows: row %d is NULL", r);
  cudaPointerAttributes at;
  BEM_CK(cudaPointerGetAttributes(&at, x_time));
  BEM_REQ(at.type == cudaMemoryTypeDevice, "cqm_forward_rows: input must be device memory");
  DeviceGuard dg(at.device);
  const RowPtrs* dev = nullptr;
  bem_status rs = upload_rows(0, out_rows, N + 1, (cudaStream_t)cuda_stream, &dev);
  if (rs != BEM_OK) return rs;
  return fft_transform_rows((const double*)x_time, nullptr, M_loc, N, R, false, (cudaStream_t)cuda_stream, nullptr, dev);
}

extern "C" bem_status cqm_inverse_rows(bem_c128* const* in_rows, bem_c128* y_time, int64_t M_loc, int32_t N, double R,
                                       void* cuda_stream) {
  BEM_REQ(y_time && in_rows, "cqm_inverse_rows: NULL pointer");
  BEM_REQ(M_loc >= 1 && N >= 1 && N + 1 <= kMaxRows, "cqm_inverse_rows: need M_loc >= 1 and 1 <= N < %d", kMaxRows);
  BEM_REQ(R > 0.0 && R <= 1.0, "cqm_inverse_rows: R must lie in (0,1]");
  for (int r = 0; r <= N; ++r) BEM_REQ(in_rows[r] != nullptr, "cqm_inverse_rows: row %d is NULL", r);
  cudaPointerAttributes at;
  BEM_CK(cudaPointerGetAttributes(&at, y_time));
  BEM_REQ(at.type == cudaMemoryTypeDevice, "cqm_inverse_rows: output must be device memory");
  DeviceGuard dg(at.device);
  const RowPtrs* dev = nullptr;
  bem_status rs = upload_rows(1, in_rows, N + 1, (cudaStream_t)cuda_stream, &dev);
  if (rs != BEM_OK) return rs;
  return fft_transform_rows(nullptr, (double*)y_time, M_loc, N, R, true, (cudaStream_t)cuda_stream, dev, nullptr);
}

// CUDA IPC helpers for the peer row tables (multi-GPU transposes without NCCL)
extern "C" bem_status bem_ipc_get_handle(void* dev_ptr, void* handle_out /* 64 bytes */) {
  BEM_REQ(dev_ptr && handle_out, "bem_ipc_get_handle: NULL argument");
  cudaIpcMemHandle_t h;
  BEM_CK(cudaIpcGetMemHandle(&h, dev_ptr));
  static_assert(sizeof(h) == 64, "CUDA IPC handle size");
  memcpy(handle_out, &h, sizeof(h));
  return BEM_OK;
}

extern "C" bem_status bem_ipc_open_handle(const void* handle, int32_t device, void** dev_ptr_out) {
  BEM_REQ(handle && dev_ptr_out, "bem_ipc_open_handle: NULL argument");
  DeviceGuard dg(device);
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  BEM_CK(cudaIpcOpenMemHandle(dev_ptr_out, h, cudaIpcMemLazyEnablePeerAccess));
  return BEM_OK;
}

// raw device allocations (own cudaMalloc, so an IPC handle maps exactly this buffer)
extern "C" bem_status bem_device_alloc(int64_t bytes, int32_t device, void** out) {
  BEM_REQ(out && bytes > 0, "bem_device_alloc: bad arguments");
  DeviceGuard dg(device);
  BEM_CK(cudaMalloc(out, (size_t)bytes));
  return BEM_OK;
}

extern "C" bem_status bem_device_free(void* ptr) {
  if (ptr) BEM_CK(cudaFree(ptr));
  return BEM_OK;
}

extern "C" bem_status bem_ipc_close(void* dev_ptr) {
  BEM_REQ(dev_ptr, "bem_ipc_close: NULL argument");
  BEM_CK(cudaIpcCloseMemHandle(dev_ptr));
  return BEM_OK;
}
