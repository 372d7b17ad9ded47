// K4: batched R-scaled CQM transforms along the time/frequency axis
// (eq:omega_n P:436-441, eq:slphelm P:529-540; reading D2):
//   forward  X_l = sum_n R^n x_n w^{nl},             w = e^{-2 pi i/L}
//   inverse  y_n = R^{-n}/L sum_l Y_l w^{-nl}
// One CTA transforms a group of NC DOF columns entirely in shared memory: the
// [L][NC] tile is loaded with coalesced row segments (R^n folded into the load),
// transformed, and stored (R^{-n}/L folded into the store).
//  * L whose prime factors are all <= 64 (33 = 3*11, 129 = 3*43, 513 = 3^3*19,
//    1025 = 5^2*41): a self-sorting mixed-radix Stockham FFT -- radix-2/3/4/5/7
//    butterflies in registers, larger prime factors as a direct DFT whose
//    outputs are spread over threads (every input read is a shared-memory
//    broadcast); twiddles and roots from one table of the L-th roots of unity.
//  * otherwise (257 is prime): Bluestein's chirp-z identity
//    nl = (n^2 + l^2 - (l-n)^2)/2 with a power-of-two P >= 2L-1 FFT:
//      out_j = post_j sum_i (in_i pre_i) h_{j-i},  c_k = e^{-pi i (k^2 mod 2L)/L},
//      forward: pre_i = R^i c_i, h_k = conj(c_k), post_j = c_j;
//      inverse: pre_i = conj(c_i), h_k = c_k, post_j = R^{-j} conj(c_j)/L.
// Rows may be addressed through a table of row pointers passed BY VALUE in the
// kernel parameters (16 KB, graph-capturable, no staging): the transforms fused
// with the multi-GPU time<->frequency transpose (cqm_*_rows, bem_comm.cu).
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
  DBuf<double> pre, post, hhat, tw;  // Bluestein: complex arrays (interleaved)
  bool stock = false;                // mixed-radix Stockham (every prime factor <= kMaxRadix)
  int nst = 0, rad[24] = {};
  DBuf<double> roots, scale;         // Stockham: e^{sign 2 pi i k/L} (k < L); R^n or R^{-n}/L
};

constexpr int kMaxRadix = 64;

// radices of L: 4s, 2s, 3s, 5s, 7s, then the remaining primes; empty if a prime > kMaxRadix
std::vector<int> factor_radices(int L) {
  std::vector<int> f;
  int n = L;
  for (int q : {4, 2, 3, 5, 7})
    while (n % q == 0) { f.push_back(q); n /= q; }
  for (int q = 11; n > 1 && q <= kMaxRadix; q += 2)
    while (n % q == 0) { f.push_back(q); n /= q; }
  if (n > 1) f.clear();
  return f;
}

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
  const std::vector<int> rad = factor_radices(L);
  if (!rad.empty() && (int)rad.size() <= 24) {
    pl->L = L;
    pl->stock = true;
    pl->nst = (int)rad.size();
    for (int i = 0; i < pl->nst; ++i) pl->rad[i] = rad[i];
    const double sg = inverse ? 1.0 : -1.0;
    std::vector<double> ro(2 * L), sc(L);
    for (int k = 0; k < L; ++k) {
      const double ang = 2.0 * M_PI * (double)k / (double)L;
      ro[2 * k] = std::cos(ang);
      ro[2 * k + 1] = sg * std::sin(ang);
      sc[k] = inverse ? std::pow(R, -(double)k) / (double)L : std::pow(R, (double)k);
    }
    BEM_CK(pl->roots.upload(ro));
    BEM_CK(pl->scale.upload(sc));
    *out = pl.get();
    g_plans[key] = std::move(pl);
    return BEM_OK;
  }
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

// Row addressing: mode 0 = row r at in/out + r*M; mode 1 = input row r at tab.p[r];
// mode 2 = output row r at tab.p[r].  With row pointers into OTHER ranks' buffers
// (CUDA IPC peer memory) or into the packed send / receive buffers of an NCCL
// all-to-all (bem_comm.cu), the kernel performs the transform and the
// time<->frequency transpose's (un)packing in one pass.
struct K4Args {
  const double2* in;
  double2* out;
  int64_t M;
  int L, NC, mode, inverse;
  // Stockham
  int nst;
  int rad[24];
  const double2* roots;
  const double* scale;
  // Bluestein
  int P, logP;
  const double2 *pre, *post, *hhat, *tw;
};

__device__ __forceinline__ double2 cfma(double2 acc, double2 a, double2 b) {  // acc + a b
  acc.x = fma(a.x, b.x, fma(-a.y, b.y, acc.x));
  acc.y = fma(a.x, b.y, fma(a.y, b.x, acc.y));
  return acc;
}

// radix-R Stockham stage (R <= 8, butterflies in registers), A -> B:
//   j < T = L/R, jm = j mod Ns:  v_r = A[j + r T] w^{jm r L/(Ns R)},
//   B[(j - jm) R + jm + k Ns] = sum_r v_r w^{(r k mod R) L/R}
template <int R>
__device__ __forceinline__ void stage_small(const double2* __restrict__ A, double2* __restrict__ B, int L, int Ns,
                                            int NC, const double2* __restrict__ W) {
  const int T = L / R, tstep = L / (Ns * R), rstep = L / R;
  for (int it = threadIdx.x; it < T * NC; it += blockDim.x) {
    const int j = it / NC, c = it - j * NC;
    const int jm = j % Ns;
    double2 v[R];
#pragma unroll
    for (int r = 0; r < R; ++r) v[r] = A[(j + r * T) * NC + c];
#pragma unroll
    for (int r = 1; r < R; ++r) v[r] = cm(v[r], W[jm * r * tstep]);
    const int base = (j - jm) * R + jm;
    if constexpr (R == 2) {
      B[base * NC + c] = make_double2(v[0].x + v[1].x, v[0].y + v[1].y);
      B[(base + Ns) * NC + c] = make_double2(v[0].x - v[1].x, v[0].y - v[1].y);
    } else {
#pragma unroll
      for (int k = 0; k < R; ++k) {
        double2 acc = v[0];
#pragma unroll
        for (int r = 1; r < R; ++r) acc = cfma(acc, v[r], W[((r * k) % R) * rstep]);
        BEM_DASSERT((base + k * Ns) * NC + c < L * NC);
        B[(base + k * Ns) * NC + c] = acc;
      }
    }
  }
}

// prime radix R > 8: twiddle pass A -> B, then a direct R-point DFT, B -> A (the result
// stays in A).  One thread per output pair (k, R - k): with v_r = a_r + i b_r and
// w^{rk} = c + i d, X_k = (sum ac - sum bd) + i (sum ad + sum bc) and X_{R-k} =
// (sum ac + sum bd) + i (sum bc - sum ad), so the pair costs four FMAs and two
// shared-memory loads per r (k = 0: the plain sum); the inputs are broadcasts.
__device__ __forceinline__ void stage_large(double2* __restrict__ A, double2* __restrict__ B, int L, int R, int Ns,
                                            int NC, const double2* __restrict__ W) {
  const int T = L / R, tstep = L / (Ns * R), rstep = L / R;
  for (int e = threadIdx.x; e < L * NC; e += blockDim.x) {
    const int row = e / NC;
    const int r = row / T, j = row - r * T;
    B[e] = cm(A[e], W[(j % Ns) * r * tstep]);
  }
  __syncthreads();
  const int H = (R + 1) / 2;  // k = 0 and the pairs (k, R - k), k = 1..(R-1)/2 (R odd)
  for (int it = threadIdx.x; it < T * H * NC; it += blockDim.x) {
    const int c = it % NC, q = it / NC;
    const int j = q / H, k = q - j * H;
    const int jm = j % Ns;
    const double2* b = B + j * NC + c;
    double2* out = A + ((j - jm) * R + jm) * NC + c;
    if (k == 0) {
      double2 acc = b[0];
      for (int r = 1; r < R; ++r) {
        const double2 v = b[r * T * NC];
        acc.x += v.x;
        acc.y += v.y;
      }
      out[0] = acc;
      continue;
    }
    const double2 v0 = b[0];
    double sac = v0.x, sbd = 0.0, sad = 0.0, sbc = v0.y;
    int idx = k;
    for (int r = 1; r < R; ++r) {
      const double2 v = b[r * T * NC], w = W[idx * rstep];
      sac = fma(v.x, w.x, sac);
      sbd = fma(v.y, w.y, sbd);
      sad = fma(v.x, w.y, sad);
      sbc = fma(v.y, w.x, sbc);
      idx += k;
      if (idx >= R) idx -= R;
    }
    BEM_DASSERT((out - A) + (int64_t)(R - k) * Ns * NC < (int64_t)L * NC);
    out[(int64_t)k * Ns * NC] = make_double2(sac - sbd, sad + sbc);
    out[(int64_t)(R - k) * Ns * NC] = make_double2(sac + sbd, sbc - sad);
  }
}

__device__ __forceinline__ void stockham_body(const K4Args& a, const double2* const* tab) {
  extern __shared__ double2 sm2[];
  const int L = a.L, NC = a.NC;
  double2* A = sm2;
  double2* B = A + (size_t)L * NC;
  double2* W = B + (size_t)L * NC;
  const int64_t c0 = (int64_t)blockIdx.x * NC;
  const int nc = (int)min((int64_t)NC, a.M - c0);
  for (int i = threadIdx.x; i < L; i += blockDim.x) W[i] = a.roots[i];
  for (int idx = threadIdx.x; idx < L * NC; idx += blockDim.x) {
    const int n = idx / NC, c = idx - n * NC;
    double2 v = make_double2(0.0, 0.0);
    if (c < nc) {
      const double2* row = a.mode == 1 ? tab[n] : a.in + (int64_t)n * a.M;
      v = row[c0 + c];
      if (!a.inverse) { const double sc = a.scale[n]; v.x *= sc; v.y *= sc; }
    }
    BEM_DASSERT(idx < L * NC);
    A[idx] = v;
  }
  __syncthreads();
  int Ns = 1;
  for (int st = 0; st < a.nst; ++st) {
    const int R = a.rad[st];
    switch (R) {
      case 2: stage_small<2>(A, B, L, Ns, NC, W); break;
      case 3: stage_small<3>(A, B, L, Ns, NC, W); break;
      case 4: stage_small<4>(A, B, L, Ns, NC, W); break;
      case 5: stage_small<5>(A, B, L, Ns, NC, W); break;
      case 7: stage_small<7>(A, B, L, Ns, NC, W); break;
      default: stage_large(A, B, L, R, Ns, NC, W); break;
    }
    if (R <= 8) { double2* t = A; A = B; B = t; }
    __syncthreads();
    Ns *= R;
  }
  for (int idx = threadIdx.x; idx < L * NC; idx += blockDim.x) {
    const int n = idx / NC, c = idx - n * NC;
    if (c < nc) {
      double2 v = A[idx];
      if (a.inverse) { const double sc = a.scale[n]; v.x *= sc; v.y *= sc; }
      double2* row = a.mode == 2 ? const_cast<double2*>(tab[n]) : a.out + (int64_t)n * a.M;
      row[c0 + c] = v;
    }
  }
}

__device__ __forceinline__ void bluestein_body(const K4Args& a, const double2* const* tab) {
  extern __shared__ double2 buf[];
  const int L = a.L, P = a.P, logP = a.logP, NC = a.NC;
  const int64_t c0 = (int64_t)blockIdx.x * NC;
  const int nc = (int)min((int64_t)NC, a.M - c0);
  // load with pre-chirp into bit-reversed positions; zero padding
  for (int idx = threadIdx.x; idx < NC * P; idx += blockDim.x) {
    const int n = idx / NC, col = idx % NC;
    double2 v = make_double2(0.0, 0.0);
    if (n < L && col < nc) {
      const double2* row = a.mode == 1 ? tab[n] : a.in + (int64_t)n * a.M;
      v = cm(row[c0 + col], a.pre[n]);
    }
    const int rv = (int)(__brev((unsigned)n) >> (32 - logP));
    if (n < P) buf[(size_t)col * P + sw(rv)] = v;
  }
  __syncthreads();
  // forward FFT, then the filter spectrum (already scaled by 1/P), fused into its last pass
  smem_fft(buf, P, logP, NC, a.tw, false, a.hhat);
  smem_fft_dif(buf, P, logP, NC, a.tw, true);  // output in bit-reversed order
  for (int idx = threadIdx.x; idx < NC * L; idx += blockDim.x) {
    const int j = idx / NC, col = idx % NC;
    if (col < nc) {
      double2* row = a.mode == 2 ? const_cast<double2*>(tab[j]) : a.out + (int64_t)j * a.M;
      const int jr = (int)(__brev((unsigned)j) >> (32 - logP));
      row[c0 + col] = cm(buf[(size_t)col * P + sw(jr)], a.post[j]);
    }
  }
}

// Persistent, software-pipelined Stockham: each CTA walks column groups blockIdx.x,
// blockIdx.x + gridDim.x, ...; while a group is transformed in shared memory the next
// group's [L][NC] tile is already in flight (cp.async, 16-byte elements straight into the
// second staging buffer), so the HBM reads overlap the butterflies instead of alternating
// with them (r2: the one-shot kernel was long-scoreboard bound at 1.2 TB/s).
// Shared memory: In[0], In[1], B ([L][NC] each) and the root table W [L].
__device__ __forceinline__ void stockham_pipe_body(const K4Args& a, const double2* const* tab) {
  extern __shared__ double2 sm2[];
  const int L = a.L, NC = a.NC;
  const size_t tile = (size_t)L * NC;  // staging buffers at sm2 and sm2 + tile
  double2* Bw = sm2 + (size_t)2 * L * NC;
  double2* W = Bw + (size_t)L * NC;
  const int64_t ngrp = (a.M + NC - 1) / NC;
  for (int i = threadIdx.x; i < L; i += blockDim.x) W[i] = a.roots[i];
  auto issue = [&](int64_t grp, double2* dst) {
    const int64_t c0 = grp * NC;
    const int nc = (int)min((int64_t)NC, a.M - c0);
    for (int idx = threadIdx.x; idx < L * NC; idx += blockDim.x) {
      const int n = idx / NC, c = idx - n * NC;
      if (c < nc) {
        const double2* row = a.mode == 1 ? tab[n] : a.in + (int64_t)n * a.M;
        cp_async16(dst + idx, row + c0 + c);
      } else {
        dst[idx] = make_double2(0.0, 0.0);
      }
    }
    cp_async_commit();
  };
  int cur = 0;
  if ((int64_t)blockIdx.x < ngrp) issue(blockIdx.x, sm2);
  for (int64_t grp = blockIdx.x; grp < ngrp; grp += gridDim.x) {
    const int64_t nxt = grp + gridDim.x;
    if (nxt < ngrp) issue(nxt, sm2 + (cur ^ 1) * tile);
    else cp_async_commit();  // empty group: wait_group 1 below still means "current tile landed"
    cp_async_wait1();
    __syncthreads();
    double2* A = sm2 + cur * tile;
    double2* B = Bw;
    if (!a.inverse) {
      for (int idx = threadIdx.x; idx < L * NC; idx += blockDim.x) {
        const double sc = a.scale[idx / NC];
        A[idx].x *= sc;
        A[idx].y *= sc;
      }
      __syncthreads();
    }
    int Ns = 1;
    for (int st = 0; st < a.nst; ++st) {
      const int R = a.rad[st];
      switch (R) {
        case 2: stage_small<2>(A, B, L, Ns, NC, W); break;
        case 3: stage_small<3>(A, B, L, Ns, NC, W); break;
        case 4: stage_small<4>(A, B, L, Ns, NC, W); break;
        case 5: stage_small<5>(A, B, L, Ns, NC, W); break;
        case 7: stage_small<7>(A, B, L, Ns, NC, W); break;
        default: stage_large(A, B, L, R, Ns, NC, W); break;
      }
      if (R <= 8) { double2* t = A; A = B; B = t; }
      __syncthreads();
      Ns *= R;
    }
    const int64_t c0 = grp * NC;
    const int nc = (int)min((int64_t)NC, a.M - c0);
    for (int idx = threadIdx.x; idx < L * NC; idx += blockDim.x) {
      const int n = idx / NC, c = idx - n * NC;
      if (c < nc) {
        double2 v = A[idx];
        if (a.inverse) { const double sc = a.scale[n]; v.x *= sc; v.y *= sc; }
        double2* row = a.mode == 2 ? const_cast<double2*>(tab[n]) : a.out + (int64_t)n * a.M;
        row[c0 + c] = v;
      }
    }
    __syncthreads();  // In[cur] and B are free before the next iteration refills In[cur]
    cur ^= 1;
  }
  cp_async_wait1();  // nothing outstanding at exit (the trailing group is empty)
}

// ---- L = 513 = 27 * 19 (config 4): the whole transform of a column in registers, two
// passes through shared memory instead of one per radix stage (the generic Stockham kernel
// above is shared-memory bound: ~40 wavefronts per element at L = 513).  Cooley-Tukey with
// n = 19 n1 + n2, k = k1 + 27 k2:
//   X[k1 + 27 k2] = sum_{n2} W19^{n2 k2} W513^{n2 k1} sum_{n1} x[19 n1 + n2] W27^{n1 k1};
// pass 1: thread (n2, column) reads its 27 inputs from global memory (R^n folded in), does
// the 27-point DFT (3 x 3 x 3) in registers and the W513 twiddle, writes T[k1][n2] to shared
// memory; pass 2: thread (k1, column) reads 19 values, does the 19-point DFT (output pairs
// (k, 19 - k) share inputs and roots), writes its 19 output rows (R^{-n}/L folded in).
// Roots of 27 and 19 come from the constant bank (compile-time indices after unrolling).
__constant__ double2 kT27[2][27];  // e^{sign 2 pi i x / 27}: [0] forward (sign -1), [1] inverse
__constant__ double2 kT19[2][19];
constexpr int k513NC = 8;          // DOF columns per CTA (128-byte row segments)

template <int INV>
__device__ __forceinline__ void dft3(double2& a0, double2& a1, double2& a2) {
  constexpr double s = INV ? 0.86602540378443864676 : -0.86602540378443864676;  // sign * sqrt(3) / 2
  const double t1x = a1.x + a2.x, t1y = a1.y + a2.y, t2x = a1.x - a2.x, t2y = a1.y - a2.y;
  const double mx = fma(-0.5, t1x, a0.x), my = fma(-0.5, t1y, a0.y);
  a0 = make_double2(a0.x + t1x, a0.y + t1y);
  a1 = make_double2(fma(-s, t2y, mx), fma(s, t2x, my));
  a2 = make_double2(fma(s, t2y, mx), fma(-s, t2x, my));
}
__device__ __forceinline__ double2 cmulc(double2 a, double2 w) {
  return make_double2(fma(a.x, w.x, -a.y * w.y), fma(a.x, w.y, a.y * w.x));
}
// in-place 9-point DFT (n = 3 n1 + n2, k = k1 + 3 k2); twiddles W9^x = W27^{3x}
template <int INV>
__device__ __forceinline__ void dft9(double2 (&v)[9]) {
  double2 u[3][3];  // u[k1][n2]
#pragma unroll
  for (int n2 = 0; n2 < 3; ++n2) {
    double2 a0 = v[n2], a1 = v[3 + n2], a2 = v[6 + n2];
    dft3<INV>(a0, a1, a2);
    u[0][n2] = a0;
    u[1][n2] = n2 == 0 ? a1 : cmulc(a1, kT27[INV][(3 * n2) % 27]);
    u[2][n2] = n2 == 0 ? a2 : cmulc(a2, kT27[INV][(6 * n2) % 27]);
  }
#pragma unroll
  for (int k1 = 0; k1 < 3; ++k1) {
    dft3<INV>(u[k1][0], u[k1][1], u[k1][2]);
#pragma unroll
    for (int k2 = 0; k2 < 3; ++k2) v[k1 + 3 * k2] = u[k1][k2];
  }
}
// in-place 27-point DFT (n = 9 n1 + n2, k = k1 + 3 k2)
template <int INV>
__device__ __forceinline__ void dft27(double2 (&v)[27]) {
  double2 u[3][9];  // u[k1][n2]
#pragma unroll
  for (int n2 = 0; n2 < 9; ++n2) {
    double2 a0 = v[n2], a1 = v[9 + n2], a2 = v[18 + n2];
    dft3<INV>(a0, a1, a2);
    u[0][n2] = a0;
    u[1][n2] = n2 == 0 ? a1 : cmulc(a1, kT27[INV][n2 % 27]);
    u[2][n2] = n2 == 0 ? a2 : cmulc(a2, kT27[INV][(2 * n2) % 27]);
  }
#pragma unroll
  for (int k1 = 0; k1 < 3; ++k1) {
    dft9<INV>(u[k1]);
#pragma unroll
    for (int k2 = 0; k2 < 9; ++k2) v[k1 + 3 * k2] = u[k1][k2];
  }
}

template <int INV>
__global__ void __launch_bounds__(256, 2) k513_kernel(const double2* __restrict__ in, double2* __restrict__ out,
                                                      int64_t M, const double2* __restrict__ roots,
                                                      const double* __restrict__ scale) {
  constexpr int L = 513, NC = k513NC;
  extern __shared__ double2 sm513[];
  double2* T = sm513;          // [k1][n2][c]
  double2* W = T + L * NC;     // roots
  const int tid = threadIdx.x;
  const int64_t c0 = (int64_t)blockIdx.x * NC;
  for (int i = tid; i < L; i += blockDim.x) W[i] = roots[i];
  __syncthreads();
  if (tid < 19 * NC) {  // pass 1
    const int c = tid % NC, n2 = tid / NC;
    const bool ok = c0 + c < M;
    double2 v[27];
#pragma unroll
    for (int n1 = 0; n1 < 27; ++n1) {
      const int n = 19 * n1 + n2;
      double2 x = ok ? in[(int64_t)n * M + c0 + c] : make_double2(0.0, 0.0);
      if (!INV) { const double sc = scale[n]; x.x *= sc; x.y *= sc; }
      v[n1] = x;
    }
    dft27<INV>(v);
#pragma unroll
    for (int k1 = 0; k1 < 27; ++k1) T[(k1 * 19 + n2) * NC + c] = k1 == 0 ? v[0] : cmulc(v[k1], W[(n2 * k1) % L]);
  }
  __syncthreads();
  if (tid < 27 * NC) {  // pass 2
    const int c = tid % NC, k1 = tid / NC;
    double2 v[19];
#pragma unroll
    for (int n2 = 0; n2 < 19; ++n2) v[n2] = T[(k1 * 19 + n2) * NC + c];
    if (c0 + c < M) {
      double2* o = out + c0 + c;
      double sx = v[0].x, sy = v[0].y;
#pragma unroll
      for (int r = 1; r < 19; ++r) { sx += v[r].x; sy += v[r].y; }
      {
        double2 y = make_double2(sx, sy);
        if (INV) { const double sc = scale[k1]; y.x *= sc; y.y *= sc; }
        o[(int64_t)k1 * M] = y;
      }
#pragma unroll
      for (int k = 1; k <= 9; ++k) {
        double sac = v[0].x, sbd = 0.0, sad = 0.0, sbc = v[0].y;
#pragma unroll
        for (int r = 1; r < 19; ++r) {
          const double2 w = kT19[INV][(r * k) % 19];
          sac = fma(v[r].x, w.x, sac);
          sbd = fma(v[r].y, w.y, sbd);
          sad = fma(v[r].x, w.y, sad);
          sbc = fma(v[r].y, w.x, sbc);
        }
        const int ka = k1 + 27 * k, kb = k1 + 27 * (19 - k);
        double2 ya = make_double2(sac - sbd, sad + sbc), yb = make_double2(sac + sbd, sbc - sad);
        if (INV) {
          const double sa = scale[ka], sb = scale[kb];
          ya.x *= sa; ya.y *= sa; yb.x *= sb; yb.y *= sb;
        }
        o[(int64_t)ka * M] = ya;
        o[(int64_t)kb * M] = yb;
      }
    }
  }
}

bool k513_tables_ready[64] = {};
std::mutex k513_mu;
cudaError_t k513_tables() {  // constant tables of the current device (idempotent per device)
  int dev = 0;
  cudaError_t e0 = cudaGetDevice(&dev);
  if (e0 != cudaSuccess) return e0;
  if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
  std::lock_guard<std::mutex> lk(k513_mu);
  if (k513_tables_ready[dev]) return cudaSuccess;
  double2 t27[2][27], t19[2][19];
  for (int d = 0; d < 2; ++d) {
    const double sg = d ? 1.0 : -1.0;
    for (int x = 0; x < 27; ++x) t27[d][x] = make_double2(std::cos(2.0 * M_PI * x / 27.0), sg * std::sin(2.0 * M_PI * x / 27.0));
    for (int x = 0; x < 19; ++x) t19[d][x] = make_double2(std::cos(2.0 * M_PI * x / 19.0), sg * std::sin(2.0 * M_PI * x / 19.0));
  }
  cudaError_t e = cudaMemcpyToSymbol(kT27, t27, sizeof(t27));
  if (e == cudaSuccess) e = cudaMemcpyToSymbol(kT19, t19, sizeof(t19));
  if (e == cudaSuccess) k513_tables_ready[dev] = true;
  return e;
}

constexpr int kMaxRows = 2048;
struct RowTab {
  const double2* p[kMaxRows];
};

__global__ void __launch_bounds__(kFftThreads, 3) stockham_kernel(const K4Args a) { stockham_body(a, nullptr); }
__global__ void __launch_bounds__(kFftThreads, 3) stockham_rows_kernel(const K4Args a, const __grid_constant__ RowTab tab) {
  stockham_body(a, tab.p);
}
__global__ void __launch_bounds__(kFftThreads, 2) stockham_pipe_kernel(const K4Args a) { stockham_pipe_body(a, nullptr); }
__global__ void __launch_bounds__(kFftThreads, 2) stockham_pipe_rows_kernel(const K4Args a,
                                                                           const __grid_constant__ RowTab tab) {
  stockham_pipe_body(a, tab.p);
}
__global__ void __launch_bounds__(kFftThreads) bluestein_kernel(const K4Args a) { bluestein_body(a, nullptr); }
__global__ void __launch_bounds__(kFftThreads) bluestein_rows_kernel(const K4Args a, const __grid_constant__ RowTab tab) {
  bluestein_body(a, tab.p);
}

}  // namespace

// tab: host row table (mode 1: input rows, 2: output rows), copied into the kernel
// parameters at launch (nothing to keep alive, capturable in a CUDA graph)
bem_status fft_transform_rows(const double* in, double* out, int64_t M, int N, double R, bool inverse, cudaStream_t st,
                              const double2* const* tab, int mode) {
  Nvtx nv(inverse ? "a8 K4 cqm_inverse" : "a1 K4 cqm_forward");
  Plan* pl = nullptr;
  bem_status rs = get_plan(N, R, inverse, &pl);
  if (rs != BEM_OK) return rs;
  if (mode != 0 && N + 1 > kMaxRows) {
    set_error("cqm transform rows: L = %d exceeds %d", N + 1, kMaxRows);
    return BEM_EINVAL;
  }
  K4Args a{};
  a.in = (const double2*)in; a.out = (double2*)out; a.M = M; a.L = pl->L; a.mode = mode; a.inverse = inverse ? 1 : 0;
  RowTab* rt = nullptr;
  std::unique_ptr<RowTab> hold;
  if (mode != 0) {
    hold = std::make_unique<RowTab>();
    for (int r = 0; r <= N; ++r) hold->p[r] = tab[r];
    rt = hold.get();
  }
  size_t smem;
  bool pipe = false;
  if (pl->stock) {
    a.nst = pl->nst;
    for (int i = 0; i < pl->nst; ++i) a.rad[i] = pl->rad[i];
    a.roots = (const double2*)pl->roots.p; a.scale = pl->scale.p;
    // columns per CTA: the largest power of two keeping the two [L][NC] tiles and the root
    // table within ~74 KB (three CTAs per SM)
    int NC = 1;
    while (NC < 64 && (size_t)(2 * 2 * NC + 1) * pl->L * 16 <= 74 * 1024) NC *= 2;
    if (NC == 1 && (size_t)5 * pl->L * 16 <= 113 * 1024) NC = 2;  // >= 32-byte row segments (two CTAs per SM)
    static const int nc_env = [] { const char* e = getenv("BEM_FFT_NC"); return e ? atoi(e) : 0; }();
    if (nc_env > 0) NC = nc_env;  // tuning experiments
    // pipelined persistent kernel: three [L][NC] tiles + roots, two CTAs per SM, NC >= 2
    static const int pipe_env = [] { const char* e = getenv("BEM_FFT_PIPE"); return e ? atoi(e) : 0; }();
    int NCp = 8;
    while (NCp > 2 && (size_t)(3 * NCp + 1) * pl->L * 16 > 113 * 1024) NCp /= 2;
    if (nc_env > 0) NCp = nc_env;
    pipe = pipe_env != 0 && (size_t)(3 * NCp + 1) * pl->L * 16 <= 113 * 1024;
    if (pipe) NC = NCp;
    a.NC = NC;
    smem = sizeof(double2) * ((size_t)(pipe ? 3 : 2) * NC + 1) * pl->L;
  } else {
    static const int nc_elems = [] {  // columns x points per CTA (env BEM_FFT_ELEMS; r01 sweep: 2048 best)
      const char* e = getenv("BEM_FFT_ELEMS");
      return e ? std::max(64, atoi(e)) : 2048;
    }();
    a.NC = std::max(1, nc_elems / pl->P);
    a.P = pl->P; a.logP = pl->logP;
    a.pre = (const double2*)pl->pre.p; a.post = (const double2*)pl->post.p;
    a.hhat = (const double2*)pl->hhat.p; a.tw = (const double2*)pl->tw.p;
    smem = sizeof(double2) * (size_t)a.NC * pl->P;
  }
  unsigned grid = (unsigned)((M + a.NC - 1) / a.NC);
  static const int k513_env = [] { const char* e = getenv("BEM_FFT_513"); return e ? atoi(e) : 1; }();
  if (pl->stock && pl->L == 513 && mode == 0 && k513_env) {
    BEM_CK(k513_tables());
    const unsigned g = (unsigned)((M + k513NC - 1) / k513NC);
    const int sm = (int)sizeof(double2) * 513 * (k513NC + 1);
    auto kk = inverse ? k513_kernel<1> : k513_kernel<0>;
    BEM_CK(cudaFuncSetAttribute(kk, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
    kk<<<g, 256, sm, st>>>(a.in, a.out, M, a.roots, a.scale);
    BEM_CK(cudaGetLastError());
    return BEM_OK;
  }
  if (pipe) {
    auto k = rt ? (void*)stockham_pipe_rows_kernel : (void*)stockham_pipe_kernel;
    BEM_CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    static int nsm = 0;
    if (nsm == 0) {
      int dev = 0;
      BEM_CK(cudaGetDevice(&dev));
      BEM_CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    }
    int per = 0;
    BEM_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, (const void*)k, kFftThreads, smem));
    grid = std::min<unsigned>(grid, (unsigned)(std::max(per, 1) * nsm));
    if (rt) stockham_pipe_rows_kernel<<<grid, kFftThreads, smem, st>>>(a, *rt);
    else stockham_pipe_kernel<<<grid, kFftThreads, smem, st>>>(a);
  } else if (pl->stock) {
    if (rt) {
      BEM_CK(cudaFuncSetAttribute(stockham_rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      stockham_rows_kernel<<<grid, kFftThreads, smem, st>>>(a, *rt);
    } else {
      BEM_CK(cudaFuncSetAttribute(stockham_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      stockham_kernel<<<grid, kFftThreads, smem, st>>>(a);
    }
  } else {
    if (rt) {
      BEM_CK(cudaFuncSetAttribute(bluestein_rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      bluestein_rows_kernel<<<grid, kFftThreads, smem, st>>>(a, *rt);
    } else {
      BEM_CK(cudaFuncSetAttribute(bluestein_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      bluestein_kernel<<<grid, kFftThreads, smem, st>>>(a);
    }
  }
  BEM_CK(cudaGetLastError());
  return BEM_OK;
}

bem_status fft_transform(const double* in, double* out, int64_t M, int N, double R, bool inverse, cudaStream_t st) {
  return fft_transform_rows(in, out, M, N, R, inverse, st, nullptr, 0);
}

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
  return fft_transform_rows((const double*)x_time, nullptr, M_loc, N, R, false, (cudaStream_t)cuda_stream,
                            (const double2* const*)out_rows, 2);
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
  return fft_transform_rows(nullptr, (double*)y_time, M_loc, N, R, true, (cudaStream_t)cuda_stream,
                            (const double2* const*)in_rows, 1);
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
