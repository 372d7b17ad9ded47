// K3 on the INT8 tensor cores ("far10"): the MACA coupling step (eq:maca
// P:1314-1320 inside the H^2 matvec P:938-944)
//   yhat_r[:, t] += sum_b sum_j S_b(s_{k_j}) (Z_b[j, t] xhat_c[:, t])
// as complex FP64 products emulated exactly on tcgen05.mma kind::i8 (DESIGN.md §7,
// "far10").  B200's FP64 path (DMMA / DFMA) peaks at 37 TFLOP/s while its INT8 tensor
// cores run 8192 MACs per clock per SM; every FP64 operand is written as a 48-bit
// fixed-point number of six signed bytes (balanced digits: d_i = byte_i(v + 0x80..80) - 128),
// and the 21 byte-slice products with i + j <= 5 (weights 2^{8(10-i-j)}) are
// accumulated exactly in int32 tensor-memory accumulators, one per level i + j
// (dropped levels and the roundings to 48 bits: ~4e-13 relative per block product,
// far below the 1e-10 parity bar).
//
// Scaling (exact powers of two, so the integer sums are exact):
//   B (kernel slice S_j, regenerated from the kernel as in far8): S_j / sigma_j with
//     sigma_j = max |S_j| over this CTA's rows = max(f(r_min), f(r_max)), f(r) =
//     |e^{-s r}| / (4 pi r) (f has no interior maximum for any Re s);
//   A (Z_b[j, t] sigma_j xhat_c[nu, t]): per frequency column t the power of two above
//     max_j |Z_b[j, t]| sigma_j * max_nu |xhat_c[nu, t]|.
// Per block the six level accumulators are read out, recombined in int64 and
// added to FP64 register accumulators (readout after every block keeps every int32
// sum below 2^31 for ranks <= 160).
//
// GEMM per stage (one ACA term j, 16 nu): D[t][n] (M = 128 frequency columns,
// N = 64 = 32 mu rows x (Re, Im)) += A[t][k] B[n][k], K = 32 bytes = 16 nu x (Re, Im):
//   B[2 mu][(nu, re)] = Re S, B[2 mu][(nu, im)] = -Im S,
//   B[2 mu + 1][(nu, re)] = Im S, B[2 mu + 1][(nu, im)] = Re S.
// A lives in tensor memory (written by the producing threads with tcgen05.st, no
// shared-memory read bandwidth spent on it), B in shared memory (canonical K-major
// layout).  Two stages in flight: the threads build stage s + 1 while the tensor
// cores run stage s (completion through an mbarrier per stage buffer).
#include "common.cuh"
#include "far_common.cuh"
#include "fastmath.cuh"
#include "tc.cuh"

namespace bem {
namespace {

constexpr int kQT = kFar10Tile;       // frequency columns per CTA (MMA M)
constexpr int kQRW = 32;              // mu rows per CTA
constexpr int kQN = 2 * kQRW;         // MMA N: (mu, Re/Im output part)
constexpr int kQKC = 16;              // nu per stage (MMA K = 32 bytes)
constexpr int kQXP = kQT + 2;         // x^ chunk row: tile columns, then <= 2 leftover columns
constexpr int kQThreads = 256;
constexpr int kQSl = 6;               // byte slices per operand
constexpr int kQBSlice = kQN * 32;    // bytes of one B slice tile [64][32]
constexpr int kQBStage = kQSl * kQBSlice;
constexpr uint32_t kQCols = 512;      // TMEM: six level accumulators [0, 384), two A stages [384, 480)
constexpr uint32_t kQAcol = 384;
constexpr uint32_t kQIdesc = tc::idesc_i8(kQT, kQN);
constexpr unsigned long long kQBias = 0x808080808080ull;
constexpr size_t kQMinSmem = 116 * 1024;  // one CTA per SM (it owns all 512 TMEM columns)

// canonical K-major no-swizzle offset of (n, k) in a [64][32] int8 tile: 8-row x 16-byte
// core matrices, the two K halves 128 B apart (LBO), 8-row groups 256 B apart (SBO)
__device__ __forceinline__ uint32_t boff(int n, int k) {
  return (uint32_t)((n >> 3) * 256 + (k >> 4) * 128 + (n & 7) * 16 + (k & 15));
}

// balanced digit SI (0 = most significant of six) of four biased 48-bit values, packed
// little-endian into one word of signed bytes
template <int SI>
__device__ __forceinline__ uint32_t pack4(uint64_t w0, uint64_t w1, uint64_t w2, uint64_t w3) {
  constexpr int byte = 5 - SI;
  constexpr uint32_t bsel = byte & 3;
  const uint32_t a0 = byte >= 4 ? (uint32_t)(w0 >> 32) : (uint32_t)w0;
  const uint32_t a1 = byte >= 4 ? (uint32_t)(w1 >> 32) : (uint32_t)w1;
  const uint32_t a2 = byte >= 4 ? (uint32_t)(w2 >> 32) : (uint32_t)w2;
  const uint32_t a3 = byte >= 4 ? (uint32_t)(w3 >> 32) : (uint32_t)w3;
  const uint32_t lo = __byte_perm(a0, a1, bsel | ((bsel + 4) << 4));
  const uint32_t hi = __byte_perm(a2, a3, bsel | ((bsel + 4) << 4));
  return __byte_perm(lo, hi, 0x5410) ^ 0x80808080u;
}

__device__ __forceinline__ uint64_t biased(double v) {
  return (uint64_t)__double2ll_rn(v) + kQBias;
}

__device__ __forceinline__ double kmag(double r, double sre, const double* etab) {  // |e^{-s r}| / (4 pi r)
  return (sre >= 0.0 ? fast::exp_neg_tab(-sre * r, etab) : exp(-sre * r)) * (0.079577471545947667884 / r);
}

__global__ void __launch_bounds__(kQThreads, 1) far10_kernel(const Far10Args a) {
  extern __shared__ __align__(1024) uint8_t smq[];
  __shared__ uint32_t taddr_s;
  __shared__ __align__(8) uint64_t mbar[2];
  __shared__ double etab[64];
  __shared__ double2 sctab[64];
  __shared__ double xr[3 * kQRW];
  __shared__ double ascl[kQT], oscl[kQT];
  __shared__ double redmin[kQThreads / 32], redmax[kQThreads / 32];
  const int p = a.p, m = a.m;
  uint8_t* sB = smq;                                          // 2 x [6][64][32] int8
  double2* xs = (double2*)(smq + 2 * kQBStage);               // [16][kQXP]
  double2* dtab = xs + kQKC * kQXP;                           // [32][p] (r, 1/(4 pi r))
  double* sig = (double*)(dtab + (size_t)kQRW * p);           // [rcap] sigma_j
  double* isig = sig + a.rcap;                                // [rcap] 2^46 / sigma_j
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int4 sg = a.segs[blockIdx.x / a.nch];
  const int r = sg.x;
  const int tile = blockIdx.y + a.tile0;
  const int tc0 = a.tb + tile * kQT;
  const int ncol = min(kQT, a.tb + a.nd - tc0);
  const bool lead = tile == 0;
  const int ntb = lead ? a.tb : 0;  // leftover columns (FP64 path) handled by this CTA
  const int mu0 = (blockIdx.x % a.nch) * kQRW;
  const int nrow = min(kQRW, p - mu0);
  for (int i = tid; i < 64; i += kQThreads) {
    etab[i] = fast::kExp2Tab[i];
    sctab[i] = fast::kSinCosTab[i];
  }
  for (int i = tid; i < nrow; i += kQThreads) node(a.xi + (int64_t)r * 3 * m, m, mu0 + i, xr + 3 * i);
  if (warp == 0) tc::tmem_alloc(&taddr_s, kQCols);
  if (tid == 0) {
    tc::mbar_init(&mbar[0], 1);
    tc::mbar_init(&mbar[1], 1);
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tD = taddr_s, tA0 = taddr_s + kQAcol;
  const uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;
  // A producer / readout: frequency column t_l of the tile, half hh (nu 8hh.. / columns 32hh..)
  const int t_l = tid & (kQT - 1), hh = tid >> 7;
  const int tg = tc0 + t_l;
  const bool tv = t_l < ncol && tg < a.nl && (a.mask == nullptr || a.mask[tg]);
  // B producer: mu row bmu, nu pair (2 bq, 2 bq + 1) of the stage
  const int bmu = tid >> 3, bq = tid & 7;
  const bool cta_on = __syncthreads_or(tv || (lead && tid < a.tb && (a.mask == nullptr || a.mask[tid]))) != 0;
  double acc[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) acc[i] = 0.0;
  double2 lacc[2] = {make_double2(0.0, 0.0), make_double2(0.0, 0.0)};
  uint32_t stage = 0;
  for (int bi = sg.y; bi < (cta_on ? sg.z : sg.y); ++bi) {
    const int b = a.far_sorted[bi];
    const int rk = a.rank[b];
    if (rk == 0) continue;
    const int c = a.far_c[b];
    const double2* xh = a.xhat + (int64_t)c * a.nl * p;
    const double2 *zD, *zL;
    int zst;
    zrows(a.z, b, a.nl, a.tb, tc0, zD, zL, zst);
    tc::fence_before();
    __syncthreads();  // previous block read out; dtab / sig / xs free
    tc::fence_after();
    // (1) the block's (r, 1/(4 pi r)) table over this CTA's rows, r_min and r_max
    double rmn = 1e300, rmx = 0.0;
    for (int e = tid; e < kQRW * p; e += kQThreads) {
      const int i = e / p, nu = e - i * p;
      double2 v = make_double2(1.0, 0.0);
      if (i < nrow) {
        double cn[3];
        node(a.xi + (int64_t)c * 3 * m, m, nu, cn);
        const double dx = cn[0] - xr[3 * i], dy = cn[1] - xr[3 * i + 1], dz = cn[2] - xr[3 * i + 2];
        v = dist_pair(dx * dx + dy * dy + dz * dz);
        rmn = fmin(rmn, v.x);
        rmx = fmax(rmx, v.x);
      }
      dtab[e] = v;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      rmn = fmin(rmn, __shfl_xor_sync(0xffffffffu, rmn, o));
      rmx = fmax(rmx, __shfl_xor_sync(0xffffffffu, rmx, o));
    }
    if (lane == 0) { redmin[warp] = rmn; redmax[warp] = rmx; }
    __syncthreads();
    rmn = redmin[0]; rmx = redmax[0];
#pragma unroll
    for (int w = 1; w < kQThreads / 32; ++w) { rmn = fmin(rmn, redmin[w]); rmx = fmax(rmx, redmax[w]); }
    // (2) sigma_j = max |S_j| over the rows (the kernel's modulus is monotone or convex in r)
    for (int j = tid; j < rk; j += kQThreads) {
      const double sre = a.s[a.pivk[(int64_t)b * a.rcap + j]].x;
      const double sgm = fmax(kmag(rmn, sre, etab), kmag(rmx, sre, etab)) * (1.0 + 0x1p-30);
      sig[j] = sgm;
      isig[j] = sgm > 0.0 ? 0x1p46 / sgm : 0.0;
    }
    __syncthreads();
    // (3) per column t: A scale 2^(46 - e_t), readout scale 2^e_t
    if (tid < kQT) {
      double zm = 0.0;
      if (tv) {
        for (int j = 0; j < rk; ++j) {
          const double2 z = zD[(int64_t)j * zst + tg];
          zm = fmax(zm, sqrt(fma(z.x, z.x, z.y * z.y)) * sig[j]);
        }
      }
      const double bound = tv ? zm * a.xmax[(int64_t)c * a.nl + tg] : 0.0;
      int e = 0;
      if (bound > 0.0) frexp(bound, &e);
      ascl[tid] = bound > 0.0 ? ldexp(1.0, 46 - e) : 0.0;
      oscl[tid] = ldexp(1.0, e);
    }
    __syncthreads();
    const double as_t = ascl[t_l];
    const uint32_t first_stage = stage;
    // (4) stages: nu chunks (x^ chunk staged once), then the ACA terms
    for (int k0 = 0; k0 < p; k0 += kQKC) {
      if (k0 > 0) {
        tc::fence_before();
        __syncthreads();  // every thread done with the previous x^ chunk
        tc::fence_after();
      }
      for (int idx = tid; idx < kQXP * kQKC; idx += kQThreads) {
        const int tl = idx / kQKC, nu = idx - tl * kQKC;
        int tcol;
        bool ok;
        if (tl < kQT) { tcol = tc0 + tl; ok = tl < ncol && tcol < a.nl; }
        else { tcol = tl - kQT; ok = tcol < ntb; }
        xs[nu * kQXP + tl] = (ok && k0 + nu < p) ? xh[(int64_t)tcol * p + k0 + nu] : make_double2(0.0, 0.0);
      }
      __syncthreads();
      for (int j = 0; j < rk; ++j, ++stage) {
        const int buf = stage & 1;
        if (stage >= 2) tc::mbar_wait(&mbar[buf], ((stage >> 1) - 1) & 1);
        tc::fence_after();
        const double2 sv = a.s[a.pivk[(int64_t)b * a.rcap + j]];
        {  // ---- A: column t_l, nu 8hh .. 8hh + 7 -> TMEM lane t_l, columns 4hh .. 4hh + 3 per slice
          double2 z = tv ? zD[(int64_t)j * zst + tg] : make_double2(0.0, 0.0);
          const double f = sig[j] * as_t;
          z.x *= f;
          z.y *= f;
          uint64_t wr[8], wi[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const double2 x = xs[(8 * hh + u) * kQXP + t_l];
            wr[u] = biased(fma(z.x, x.x, -z.y * x.y));
            wi[u] = biased(fma(z.x, x.y, z.y * x.x));
          }
          const uint32_t ta = tA0 + (uint32_t)buf * 48 + lane_base + 4 * hh;
          uint32_t v[4];
#define FAR10_A(SI)                                                                                        \
  {                                                                                                        \
    _Pragma("unroll") for (int cc = 0; cc < 4; ++cc) v[cc] =                                               \
        pack4<SI>(wr[2 * cc], wi[2 * cc], wr[2 * cc + 1], wi[2 * cc + 1]);                                 \
    tc::tmem_st4(ta + SI * 8, v);                                                                          \
  }
          FAR10_A(0) FAR10_A(1) FAR10_A(2) FAR10_A(3) FAR10_A(4) FAR10_A(5)
#undef FAR10_A
        }
        {  // ---- B: slice entries (bmu, 2 bq + e), regenerated from the kernel (far8's DT path)
          uint64_t br[2], bi[2], bn[2];
          const double is = isig[j];
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int nl_ = 2 * bq + e, nu = k0 + nl_;
            double2 S = make_double2(0.0, 0.0);
            if (bmu < nrow && nu < p) S = kern_tab(dtab[bmu * p + nu], sv, etab, sctab);
            for (int tl = 0; tl < ntb; ++tl) {  // leftover columns on the FP64 pipe (lead CTA)
              const double2 zz = zL[(int64_t)j * zst + tl], xv = xs[nl_ * kQXP + kQT + tl];
              const double ax = zz.x * xv.x - zz.y * xv.y, ay = zz.x * xv.y + zz.y * xv.x;
              lacc[tl].x = fma(S.x, ax, fma(-S.y, ay, lacc[tl].x));
              lacc[tl].y = fma(S.x, ay, fma(S.y, ax, lacc[tl].y));
            }
            const long long vr = __double2ll_rn(S.x * is), vi = __double2ll_rn(S.y * is);
            br[e] = (uint64_t)vr + kQBias;
            bi[e] = (uint64_t)vi + kQBias;
            bn[e] = (uint64_t)(-vi) + kQBias;
          }
          uint8_t* sb = sB + buf * kQBStage;
          const uint32_t o0 = boff(2 * bmu, 4 * bq), o1 = boff(2 * bmu + 1, 4 * bq);
#define FAR10_B(SI)                                                                                        \
  {                                                                                                        \
    *(uint32_t*)(sb + SI * kQBSlice + o0) = pack4<SI>(br[0], bn[0], br[1], bn[1]);                         \
    *(uint32_t*)(sb + SI * kQBSlice + o1) = pack4<SI>(bi[0], br[0], bi[1], br[1]);                         \
  }
          FAR10_B(0) FAR10_B(1) FAR10_B(2) FAR10_B(3) FAR10_B(4) FAR10_B(5)
#undef FAR10_B
        }
        tc::wait_st();
        tc::fence_proxy_async();
        tc::fence_before();
        __syncthreads();
        tc::fence_after();
        if (tid == 0) {
          const bool first = stage == first_stage;
          const uint32_t ta = tA0 + (uint32_t)buf * 48;
          const uint32_t sbb = tc::smem_u32(sB + buf * kQBStage);
#pragma unroll
          for (int ia = 0; ia < kQSl; ++ia)
#pragma unroll
            for (int ib = 0; ib < kQSl - ia; ++ib)
              tc::mma_i8_ts(tD + (uint32_t)(ia + ib) * kQN, ta + ia * 8,
                            tc::smem_desc(sbb + ib * kQBSlice, 128, 256), kQIdesc, (first && ia == 0) ? 0u : 1u);
          tc::mma_commit(&mbar[buf]);
        }
        __syncwarp();
      }
    }
    // (5) read the six level accumulators out into the FP64 accumulators
    {
      const uint32_t last = stage - 1;
      tc::mbar_wait(&mbar[last & 1], (last >> 1) & 1);
      tc::fence_after();
      const double et = oscl[t_l];
      const double hs = et * 0x1p-28, ls = et * 0x1p-52;
#pragma unroll
      for (int g = 0; g < 4; ++g) {
        uint32_t d0[8], d1[8], d2[8], d3[8], d4[8], d5[8];
        const uint32_t col = tD + lane_base + 32 * hh + 8 * g;
        tc::tmem_ld8(col + 0 * kQN, d0);
        tc::tmem_ld8(col + 1 * kQN, d1);
        tc::tmem_ld8(col + 2 * kQN, d2);
        tc::tmem_ld8(col + 3 * kQN, d3);
        tc::tmem_ld8(col + 4 * kQN, d4);
        tc::tmem_ld8(col + 5 * kQN, d5);
        tc::wait_ld();
#pragma unroll
        for (int cc = 0; cc < 8; ++cc) {
          const long long H = ((long long)(int)d0[cc] << 16) + ((long long)(int)d1[cc] << 8) + (long long)(int)d2[cc];
          const long long Lo = ((long long)(int)d3[cc] << 16) + ((long long)(int)d4[cc] << 8) + (long long)(int)d5[cc];
          acc[8 * g + cc] = fma((double)H, hs, fma((double)Lo, ls, acc[8 * g + cc]));
        }
      }
    }
  }
  // (6) this segment's partial: columns 32 hh .. 32 hh + 31 = rows mu 16 hh .. 16 hh + 15 (Re, Im)
  double2* out = a.part + (int64_t)sg.w * a.nl * p;
  if (t_l < ncol && tg < a.nl) {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const int mu = 16 * hh + i;
      if (mu < nrow) {
        BEM_DASSERT((out - a.part) + (int64_t)tg * p + mu0 + mu < a.part_n);
        out[(int64_t)tg * p + mu0 + mu] = tv ? make_double2(acc[2 * i], acc[2 * i + 1]) : make_double2(0.0, 0.0);
      }
    }
  }
  for (int tl = 0; tl < ntb; ++tl) {
    double2 v = lacc[tl];
#pragma unroll
    for (int o = 1; o < 8; o <<= 1) {
      v.x += __shfl_xor_sync(0xffffffffu, v.x, o);
      v.y += __shfl_xor_sync(0xffffffffu, v.y, o);
    }
    if (bq == 0 && bmu < nrow) out[(int64_t)tl * p + mu0 + bmu] = v;
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(taddr_s, kQCols);
}

// max_nu |xhat_c(nu, t)| for every (cluster, frequency) row: one warp per row
__global__ void __launch_bounds__(256) xmax_kernel(const double2* __restrict__ xhat, int64_t rows, int p,
                                                   double* __restrict__ out) {
  const int64_t row = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= rows) return;
  double mx = 0.0;
  for (int nu = lane; nu < p; nu += 32) {
    const double2 v = xhat[row * p + nu];
    mx = fmax(mx, sqrt(fma(v.x, v.x, v.y * v.y)));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if (lane == 0) out[row] = mx * (1.0 + 0x1p-40);
}

}  // namespace

cudaError_t launch_far10(const Far10Args& a, int nseg, int ntile, cudaStream_t st) {
  const size_t need = 2 * (size_t)kQBStage + sizeof(double2) * ((size_t)kQKC * kQXP + (size_t)kQRW * a.p) +
                      sizeof(double) * 2 * (size_t)a.rcap + 64;
  const size_t smem = need > kQMinSmem ? need : kQMinSmem;
  cudaError_t e = cudaFuncSetAttribute(far10_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  far10_kernel<<<dim3((unsigned)(nseg * a.nch), (unsigned)ntile, 1u), kQThreads, smem, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_xmax(const double2* xhat, int64_t rows, int p, double* out, cudaStream_t st) {
  xmax_kernel<<<(unsigned)((rows + 7) / 8), 256, 0, st>>>(xhat, rows, p, out);
  return cudaGetLastError();
}

}  // namespace bem
