// K3 on the INT8 tensor cores ("far10"): the MACA coupling step (eq:maca
// P:1314-1320 inside the H^2 matvec P:938-944)
//   yhat_r[:, t] += sum_b sum_j S_b(s_{k_j}) (Z_b[j, t] xhat_c[:, t])
// as complex FP64 products emulated exactly on tcgen05.mma kind::i8 (DESIGN.md §7,
// "far10").  B200's FP64 path (DMMA / DFMA) peaks at 37 TFLOP/s while its INT8 tensor
// cores run 8192 MACs per clock per SM; every FP64 operand is written as a 48-bit
// fixed-point number of six bytes (A: two's complement bytes, the top one signed; B: balanced
// signed digits), and the 21 byte-slice products with i + j <= 5 (weights 2^{8(10-i-j)}) are
// accumulated exactly in int32 tensor-memory accumulators, one per level i + j
// (dropped levels and the roundings to 48 bits: ~4e-13 relative per block product,
// far below the 1e-10 parity bar).
//
// Scaling (exact powers of two, so the integer sums are exact):
//   B (kernel slice S_j, regenerated from the kernel -- far8's table exp / sincos): S_j / sigma_j with
//     sigma_j = max |S_j| over this CTA's rows = max(f(r_min), f(r_max)), f(r) =
//     |e^{-s r}| / (4 pi r) (f has no interior maximum for any Re s);
//   A (Z_b[j, t] sigma_j xhat_c[nu, t]): per frequency column t the power of two above
//     max_j |Z_b[j, t]| sigma_j * max_nu |xhat_c[nu, t]|.
// After every block (and every group of gmax ACA terms of a long block: level sums are
// bounded by 179584 per contracted byte, so gmax = floor((2^31 - 1) / (179584 K_term))) the
// six level accumulators are read out, recombined in int64 and added to FP64 accumulators.
//
// GEMM per stage (one ACA term j, 16 nu): D[t][n] (M = 128 frequency columns,
// N = 64 = 32 mu rows x (Re, Im)) += A[t][k] B[n][k], K = 32 bytes = 16 nu x (Re, Im):
//   B[2 mu][(nu, re)] = Re S, B[2 mu][(nu, im)] = -Im S,
//   B[2 mu + 1][(nu, re)] = Im S, B[2 mu + 1][(nu, im)] = Re S.
// A lives in tensor memory (written by the producing threads with tcgen05.st, no
// shared-memory read bandwidth spent on it), B in shared memory (canonical K-major
// layout).  Two stages in flight: the threads build stage s + 1 while the tensor
// cores run stage s (completion through an mbarrier per stage buffer).
//
// Persistent CTAs (default): one CTA per SM takes (segment x mu chunk, frequency tile) work
// items from a counter; the coupling warps synchronise with named barriers only, so that
// NEARW extra warps can run K1 (near field, a3) items from a second counter for as long as
// the CTA's coupling work lasts (near_common.cuh; the items they leave run in a tail kernel
// after the launch). K1 as a separate kernel never shares an SM with a far10 CTA (DESIGN.md
// §7); 9 + 3 warps x 168 registers fill the register file.
#include <algorithm>
#include <cstdlib>

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
constexpr int kQSl = 6;               // byte slices per operand
constexpr int kQBSlice = kQN * 32;    // bytes of one B slice tile [64][32]
constexpr int kQBStage = kQSl * kQBSlice;
constexpr uint32_t kQCols = 512;      // TMEM: six level accumulators [0, 384), A of stages 0, 1 [384, 480)
constexpr uint32_t kQAcol = 384;
// slice products: A's top slice (index 0) signed, its other slices unsigned; B balanced (signed)
__device__ __forceinline__ constexpr uint32_t qidesc(int ia, int ib) {
  return tc::idesc_i8s(kQT, kQN, ia == 0 ? 1 : 0, 1);
}
constexpr int kQNB = 2;               // pipeline stages, both A stages in TMEM (a third stage with A in shared
                                      // memory measured slower: 982 vs 930 ms at config 4)
constexpr size_t kQMinSmem = 116 * 1024;  // one CTA per SM (it owns all 512 TMEM columns)

// canonical K-major no-swizzle offset of (n, k) in a [64][32] int8 tile: 8-row x 16-byte
// core matrices, the two K halves 128 B apart (LBO), 8-row groups 256 B apart (SBO)
__device__ __forceinline__ uint32_t boff(int n, int k) {
  return (uint32_t)((n >> 3) * 256 + (k >> 4) * 128 + (n & 7) * 16 + (k & 15));
}

// Fixed-point conversion on the FP64 pipe: for |v| < 2^47, v + 1.5 2^52 rounds v to the
// nearest integer and leaves v mod 2^48 (two's complement) in the low 48 bits of the double
// (exponent fixed).  A operand (kQMagicA): v = d5 2^40 + sum_{i<5} d_i 2^{8i} with d5 = byte 5
// read as a signed byte, d_0..d_4 = bytes 0..4 read as unsigned bytes (no fix-up at all).
// B operand (kQMagicB = 1.5 2^52 + 0x808080808080): balanced digits byte_i(v + C) - 128 =
// byte_i ^ 0x80 read as signed bytes.  One zero-mean operand keeps the dropped slice levels
// (i + j >= 6) unbiased: with unsigned lower digits on both sides the truncation error adds
// up linearly (measured: config 4 rel. error 3.2e-10 instead of ~1e-12).
constexpr double kQMagicA = 6755399441055744.0;  // 1.5 * 2^52
constexpr double kQMagicB = 6896688841130112.0;  // 1.5 * 2^52 + 0x808080808080

// 4 x 4 byte transpose of the low words of four digit carriers: out[b] = byte b of (a, b, c, d)
// packed little-endian (slice 5 - b); hi words give slices 1, 0
__device__ __forceinline__ void tr_lo(uint32_t a, uint32_t b, uint32_t c, uint32_t d, uint32_t (&o)[4]) {
  const uint32_t t0 = __byte_perm(a, b, 0x5140), t1 = __byte_perm(c, d, 0x5140);
  const uint32_t t2 = __byte_perm(a, b, 0x7362), t3 = __byte_perm(c, d, 0x7362);
  o[0] = __byte_perm(t0, t1, 0x5410);
  o[1] = __byte_perm(t0, t1, 0x7632);
  o[2] = __byte_perm(t2, t3, 0x5410);
  o[3] = __byte_perm(t2, t3, 0x7632);
}
__device__ __forceinline__ void tr_hi(uint32_t a, uint32_t b, uint32_t c, uint32_t d, uint32_t (&o)[2]) {
  const uint32_t t0 = __byte_perm(a, b, 0x5140), t1 = __byte_perm(c, d, 0x5140);
  o[0] = __byte_perm(t0, t1, 0x5410);
  o[1] = __byte_perm(t0, t1, 0x7632);
}

// the slice entry's modulus and phase factors (kern_tab's intermediates): S = e (cs, -sn)
__device__ __forceinline__ void kern_parts(double2 rw, double2 s, const double* etab, const double2* sctab, double& e,
                                           double& sn, double& cs) {
  e = fast::exp_neg_tab(-s.x * rw.x, etab) * rw.y;
  fast::sincos_tab(s.y * rw.x, sctab, &sn, &cs);
}

__device__ __forceinline__ double kmag(double r, double sre, const double* etab) {  // |e^{-s r}| / (4 pi r)
  return (sre >= 0.0 ? fast::exp_neg_tab(-sre * r, etab) : exp(-sre * r)) * (0.079577471545947667884 / r);
}

template <int ID, int N>
__device__ __forceinline__ void named_sync() {
  asm volatile("bar.sync %0, %1;" ::"n"(ID), "n"(N) : "memory");
}
template <int ID, int N>
__device__ __forceinline__ bool named_or(bool v) {  // barrier over N threads, OR of v
  uint32_t r;
  asm volatile("{\n .reg .pred p, q;\n setp.ne.u32 p, %1, 0;\n barrier.red.or.pred q, %2, %3, p;\n selp.u32 %0, 1, 0, q;\n}"
               : "=r"(r) : "r"((uint32_t)v), "n"(ID), "n"(N) : "memory");
  return r != 0;
}
template <int NP>
__device__ __forceinline__ void prod_sync() {  // the producer warps only (named barrier 1)
  asm volatile("bar.sync 1, %0;" ::"n"(NP) : "memory");
}
__device__ __forceinline__ void cp_async16z(void* dst, const void* src, bool ok) {  // zero-fill when !ok
  const unsigned sa = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(src), "r"(ok ? 16 : 0) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

// PW producer warps (16: one B slice entry and 4 nu of A per thread per stage, 96 registers;
// 8: two B entries and 8 nu, 168 registers -- fewer warps, more independent work per thread)
// NEARW > 0: that many extra warps run K1 (near field) items from a.nctr while the coupling work
// of the CTA lasts (the SMs' FP64 pipes are ~20 % busy in far10; K1 cannot co-reside as a
// separate kernel)
template <int PW, int NEARW>
__global__ void __launch_bounds__(PW * 32 + 32 + NEARW * 32, 1) far10_kernel(const Far10Args a) {
  constexpr int kQProd = PW * 32;        // producer threads
  constexpr int kQThreads = kQProd + 32;  // + the MMA-issue warp
  constexpr int NQ = kQProd / kQT;        // nu groups per frequency column (4 / 2)
  constexpr int NUP = kQKC / NQ;          // nu of A per producer thread per stage (4 / 8)
  constexpr int NG = NUP / 2;             // A words per slice per thread (2 / 4)
  constexpr int NCOL = kQN / NQ;          // accumulator columns per thread (16 / 32)
  constexpr int EB = kQRW * kQKC / kQProd;  // B slice entries per thread per stage (1 / 2)
  static_assert(EB == 1 || EB == 2, "far10: 8 or 16 producer warps");
  extern __shared__ __align__(1024) uint8_t smq[];
  __shared__ uint32_t taddr_s;
  __shared__ int k3done, item_s;
  __shared__ __align__(8) uint64_t full[kQNB], empty[kQNB], drained;
  __shared__ double etab[64];
  __shared__ double2 sctab[64];
  __shared__ double xr[3 * kQRW];
  __shared__ double ascl[kQT], oscl[kQT];
  __shared__ double zred[kQProd / kQT][kQT];
  __shared__ double redmin[kQProd / 32], redmax[kQProd / 32];
  __shared__ int cmap[kQT];  // local frequency of the tile's column t_l (-1: padding)
  const int p = a.p, m = a.m;
  uint8_t* sB = smq;                                          // 2 x [6][64][32] int8
  double2* xsb = (double2*)(smq + kQNB * kQBStage);           // 2 x [16][kQXP]
  double2* svs = xsb + 2 * kQKC * kQXP;                       // [rcap] pivot frequencies s_{k_j}
  double* sig = (double*)(svs + a.rcap);                      // [rcap] sigma_j
  double* isig = sig + a.rcap;                                // [rcap] 2^46 / sigma_j
  double* accs = isig + a.rcap;                               // [64][128] FP64 accumulators (column-major in t)
  double2* lzs = (double2*)(accs + (size_t)kQN * kQT);        // [rcap][2] Z_b[j, leftover columns]
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nkc = (p + kQKC - 1) / kQKC;  // nu chunks per term
  for (int i = tid; i < 64; i += blockDim.x) {
    etab[i] = fast::kExp2Tab[i];
    sctab[i] = fast::kSinCosTab[i];
  }
  if (warp == 0) tc::tmem_alloc(&taddr_s, kQCols);
  if (tid == 0) {
    for (int i = 0; i < kQNB; ++i) {
      tc::mbar_init(&full[i], kQProd / 32);  // one arrival per producer warp
      tc::mbar_init(&empty[i], 1);
    }
    tc::mbar_init(&drained, kQProd / 32);
    k3done = 0;
  }
  // producer roles: A / readout (frequency column t_l, quarter q4: nu 4 q4 .. 4 q4 + 3 of a
  // stage, accumulator columns 16 q4 .. 16 q4 + 15 = rows mu 8 q4 .. 8 q4 + 7); B (slice entry
  // (bmu, bnu) of a stage)
  const int t_l = tid & (kQT - 1), q4 = (tid >> 7) & (NQ - 1);
  // B: EB = 1: entry (bmu, bnu); EB = 2: entries (bmu, bnu), (bmu, bnu + 1), bnu even
  const int bmu = EB == 1 ? (tid >> 4) & 31 : (tid >> 3) & 31;
  const int bnu = EB == 1 ? tid & 15 : 2 * (tid & 7);
  const uint32_t full_a = tc::smem_u32(&full[0]), empty_a = tc::smem_u32(&empty[0]), drained_a = tc::smem_u32(&drained);
  __syncthreads();  // tables, barriers, TMEM address
  tc::fence_after();
  const uint32_t tD = taddr_s, tA0 = taddr_s + kQAcol;

  if (warp > kQProd / 32) {
    // ================= fused K1 warps: (target, 4-class tile) items until the coupling work is done
    if constexpr (NEARW > 0) {
      if (a.nctr != nullptr) {
        for (;;) {
          if (*(volatile int*)&k3done) break;
          unsigned i = 0;
          if (lane == 0) i = atomicAdd(a.nctr, 1u);
          i = __shfl_sync(0xffffffffu, i, 0);
          if (i >= a.n_items) break;
          near_item<4, false>(a.na, (int64_t)(i % (unsigned)a.na.M), (int)(i / (unsigned)a.na.M) * 4, etab, sctab);
        }
      }
    }
  } else {
  // pipeline counters (mbarrier phases) run on across the work items of a persistent CTA
  uint32_t mstage = 0, mblk = 0, pstage = 0;
  // work items (segment x mu chunk, frequency tile): one per CTA (grid = all items), or
  // persistent CTAs (one per SM) taking items from a.ctr (named barriers: the coupling warps only)
  for (int it = 0;; ++it) {
  int w;
  if (a.ctr != nullptr) {
    if (tid == 0) item_s = atomicAdd(a.ctr, 1);
    named_sync<2, kQThreads>();  // also: every coupling warp is done with the previous item
    w = item_s;
  } else {
    if (it > 0) break;
    w = blockIdx.x + blockIdx.y * gridDim.x;
  }
  if (w >= a.nitems) break;
  const int bx = w % a.gx;
  const int4 sg = a.segs[bx / a.nch];
  const int r = sg.x;
  const int tile = w / a.gx + a.tile0;
  const int tc0 = a.tb + tile * kQT;
  const int ncol = min(kQT, a.tb + a.nd - tc0);
  const bool lead = tile == 0;
  const int ntb = lead ? a.tb : 0;  // leftover columns (FP64 path) handled by this CTA
  const int mu0 = (bx % a.nch) * kQRW;
  const int nrow = min(kQRW, p - mu0);
  for (int i = tid; i < nrow; i += kQThreads) node(a.xi + (int64_t)r * 3 * m, m, mu0 + i, xr + 3 * i);
  // the tile's columns: a.colmap orders the local frequencies by damping (Re s ascending), so
  // that whole tiles fall under the underflow mask; identity when the mask is off
  BEM_DASSERT(tile >= 0 && tile * kQT + t_l < a.ncm);
  const int tg = t_l < ncol ? a.colmap[tile * kQT + t_l] : -1;
  BEM_DASSERT(tg < a.nl);
  if (tid < kQT) cmap[tid] = tg;  // read after the named_or barrier below
  const int zt = a.z.tiled ? tc0 + t_l : tg;  // Z column: tile buffers hold the tile's columns in tile order
  const bool tv = tid < kQProd && tg >= 0 && (a.mask == nullptr || a.mask[tg]);
  const bool cta_on = named_or<3, kQThreads>(tv || (lead && tid < a.tb && (a.mask == nullptr || a.mask[tid])));
  const int bend = cta_on ? sg.z : sg.y;
  if (warp == kQProd / 32) {
    // ================= MMA-issue warp: every lane runs the loop (operands stay warp-uniform),
    // one elected lane issues -- a divergent single-thread issue loop measured ~4x slower
    // per MMA (tools/i8_rate.py: 117-156 vs 35 cycles at N = 64)
    uint32_t &stage = mstage, &blk = mblk;
    for (int bi = sg.y; bi < bend; ++bi) {
      const int b = a.far_sorted[bi];
      BEM_DASSERT(b >= 0 && (a.skip == nullptr || b < a.nfar));
      if (a.skip != nullptr && ((a.skip[b] >> tile) & 1u)) continue;  // underflow mask (same test in the producers)
      const int rk = a.rank[b];
      for (int g0 = 0; g0 < rk; g0 += a.gmax, ++blk) {  // term groups (int32 sums stay exact)
      if (blk > 0) tc::mbar_wait_a(drained_a, (blk - 1) & 1);  // previous group read out
      tc::fence_after();
      const int ns = (min(rk, g0 + a.gmax) - g0) * nkc;
      uint32_t buf = stage % kQNB, use = stage / kQNB;
      for (int s = 0; s < ns; ++s, ++stage) {
        tc::mbar_wait_a(full_a + 8 * buf, use & 1);
        tc::fence_after();
        const uint32_t sbb = tc::smem_u32(sB + buf * kQBStage);
        const uint32_t ta = tA0 + buf * 48;
#pragma unroll
        for (int ia = 0; ia < kQSl; ++ia)
#pragma unroll
          for (int ib = 0; ib < kQSl - ia; ++ib)
            tc::mma_i8_ts_warp(tD + (uint32_t)(ia + ib) * kQN, ta + ia * 8,
                               tc::smem_desc(sbb + ib * kQBSlice, 128, 256), qidesc(ia, ib), (s == 0 && ia == 0) ? 0u : 1u);
        tc::mma_commit_warp_a(empty_a + 8 * buf);
        if (++buf == kQNB) { buf = 0; ++use; }
      }
      }
    }
  } else {
    // ================= producer warps
    const uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;
    double* acc = accs + (NCOL * q4) * kQT + t_l;  // this thread's NCOL columns, stride kQT
#pragma unroll
    for (int i = 0; i < NCOL; ++i) acc[i * kQT] = 0.0;
    double2 lacc[2] = {make_double2(0.0, 0.0), make_double2(0.0, 0.0)};
    uint32_t& stage = pstage;
    int pending = 0;        // a block whose accumulators still have to be read out
    double et_prev = 1.0;   // its readout scale for column t_l
    auto readout = [&]() {
      const uint32_t last = stage - 1;
      tc::mbar_wait_a(empty_a + 8 * (last % kQNB), (last / kQNB) & 1);
      tc::fence_after();
      const double hs = et_prev * 0x1p-28, ls = et_prev * 0x1p-52;
#pragma unroll
      for (int g = 0; g < NCOL / 8; ++g) {
        uint32_t d0[8], d1[8], d2[8], d3[8], d4[8], d5[8];
        const uint32_t col = tD + lane_base + NCOL * q4 + 8 * g;
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
          acc[(8 * g + cc) * kQT] = fma((double)H, hs, fma((double)Lo, ls, acc[(8 * g + cc) * kQT]));
        }
      }
      tc::fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive_a(drained_a);
    };
    auto stage_x = [&](const double2* xh, int k0, double2* xs) {  // x^ chunk [16][kQXP] (cp.async, zero-filled)
      for (int idx = tid; idx < kQXP * kQKC; idx += kQProd) {
        const int tl = idx / kQKC, nu = idx - tl * kQKC;
        int tcol;
        bool ok;
        if (tl < kQT) { tcol = cmap[tl]; ok = tcol >= 0; }
        else { tcol = tl - kQT; ok = tcol < ntb; }
        ok = ok && k0 + nu < p;
        cp_async16z(xs + nu * kQXP + tl, ok ? (const void*)(xh + (int64_t)tcol * p + k0 + nu) : (const void*)xh, ok);
      }
      cp_async_commit();
    };
    for (int bi = sg.y; bi < bend; ++bi) {
      const int b = a.far_sorted[bi];
      const int rk = a.rank[b];
      if (rk == 0) continue;
      if (a.skip != nullptr && ((a.skip[b] >> tile) & 1u)) continue;
      const int c = a.far_c[b];
      const double2* xh = a.xhat + (int64_t)c * a.nl * p;
      const double2 *zD, *zL;
      int zst;
      zrows(a.z, b, a.nl, a.tb, tc0, zD, zL, zst);
      prod_sync<kQProd>();  // every producer done with the previous block's smem (sig, svs, x^)
      stage_x(xh, 0, xsb);  // chunk 0 in flight during the prologue
      // (1) r_min and r_max over this CTA's rows and the block's columns (the (r, 1/(4 pi r))
      // pair of a thread's own slice entry is recomputed per nu chunk, in a register)
      double rmn = 1e300, rmx = 0.0;
      for (int e = tid; e < nrow * p; e += kQProd) {
        const int i = e / p, nu = e - i * p;
        double cn[3];
        node(a.xi + (int64_t)c * 3 * m, m, nu, cn);
        const double dx = cn[0] - xr[3 * i], dy = cn[1] - xr[3 * i + 1], dz = cn[2] - xr[3 * i + 2];
        const double2 v = dist_pair(dx * dx + dy * dy + dz * dz);
        rmn = fmin(rmn, v.x);
        rmx = fmax(rmx, v.x);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        rmn = fmin(rmn, __shfl_xor_sync(0xffffffffu, rmn, o));
        rmx = fmax(rmx, __shfl_xor_sync(0xffffffffu, rmx, o));
      }
      if (lane == 0) { redmin[warp] = rmn; redmax[warp] = rmx; }
      prod_sync<kQProd>();
      rmn = redmin[0]; rmx = redmax[0];
#pragma unroll
      for (int w = 1; w < kQProd / 32; ++w) { rmn = fmin(rmn, redmin[w]); rmx = fmax(rmx, redmax[w]); }
      // (2) pivot frequencies and sigma_j = max |S_j| over the rows (the kernel's modulus
      // is monotone or convex in r)
      for (int j = tid; j < rk; j += kQProd) {
        const double2 sv = a.s[a.pivk[(int64_t)b * a.rcap + j]];
        const double sgm = fmax(kmag(rmn, sv.x, etab), kmag(rmx, sv.x, etab)) * (1.0 + 0x1p-30);
        svs[j] = sv;
        if (ntb > 0) lzs[2 * j] = zL[(int64_t)j * zst];
        if (ntb > 1) lzs[2 * j + 1] = zL[(int64_t)j * zst + 1];
        sig[j] = sgm;
        isig[j] = sgm > 0.0 ? 0x1p46 / sgm : 0.0;
      }
      prod_sync<kQProd>();
      // (3) per column t: A scale 2^(46 - e_t), readout scale 2^e_t (terms split over the quarters)
      {
        double zm = 0.0;
        if (tv)
          for (int j = q4; j < rk; j += kQProd / kQT) {
            const double2 z = zD[(int64_t)j * zst + zt];
            zm = fmax(zm, sqrt(fma(z.x, z.x, z.y * z.y)) * sig[j]);
          }
        zred[q4][t_l] = zm;
      }
      prod_sync<kQProd>();
      if (tid < kQT) {
        double zm = zred[0][tid];
#pragma unroll
        for (int q = 1; q < kQProd / kQT; ++q) zm = fmax(zm, zred[q][tid]);
        const double bound = tv ? zm * a.xmax[(int64_t)c * a.nl + tg] : 0.0;
        int e = 0;
        if (bound > 0.0) frexp(bound, &e);
        ascl[tid] = bound > 0.0 ? ldexp(1.0, 46 - e) : 0.0;
        oscl[tid] = ldexp(1.0, e);
      }
      // (4) the previous block's accumulators (its MMAs ran during this prologue)
      if (pending) readout();
      prod_sync<kQProd>();  // ascl / oscl written
      const double as_t = ascl[t_l];
      et_prev = oscl[t_l];
      pending = 1;
      // (5) term groups of <= gmax terms (readout between groups: every int32 level sum stays
      // below 2^31), per group the nu chunks (x^ chunk double-buffered), then its terms
      for (int g0 = 0; g0 < rk; g0 += a.gmax) {
      const int g1 = min(rk, g0 + a.gmax);
      if (g0 > 0) {
        readout();
        prod_sync<kQProd>();  // every producer past the previous group's x^ chunks
        stage_x(xh, 0, xsb);
      }
      double2 znext = tv ? zD[(int64_t)g0 * zst + zt] : make_double2(0.0, 0.0);
      double2 svn = svs[g0];
      double sgn = sig[g0], isn = isig[g0];
      for (int kc = 0; kc < nkc; ++kc) {
        const int k0 = kc * kQKC;
        double2* xs = xsb + (kc & 1) * kQKC * kQXP;
        cp_async_wait_all();
        prod_sync<kQProd>();  // chunk kc landed everywhere; chunk kc - 1's buffer is free
        if (kc + 1 < nkc) stage_x(xh, k0 + kQKC, xsb + ((kc + 1) & 1) * kQKC * kQXP);
        double2 rw[EB];  // (r, 1/(4 pi r)) of this thread's slice entries; off the slice (1, 0): S = 0
#pragma unroll
        for (int eb = 0; eb < EB; ++eb) {
          rw[eb] = make_double2(1.0, 0.0);
          if (bmu < nrow && k0 + bnu + eb < p) {
            double cn[3];
            node(a.xi + (int64_t)c * 3 * m, m, k0 + bnu + eb, cn);
            const double dx = cn[0] - xr[3 * bmu], dy = cn[1] - xr[3 * bmu + 1], dz = cn[2] - xr[3 * bmu + 2];
            rw[eb] = dist_pair(dx * dx + dy * dy + dz * dz);
          }
        }
        for (int j = g0; j < g1; ++j, ++stage) {
          const uint32_t buf = stage % kQNB;
          const double2 zc = znext;
          const int jn = j + 1 < g1 ? j + 1 : g0;
          znext = tv ? zD[(int64_t)jn * zst + zt] : make_double2(0.0, 0.0);
          const double2 sv = svn;
          const double sgj = sgn, isj = isn;
          svn = svs[jn];
          sgn = sig[jn];
          isn = isig[jn];
          // ---- compute (one basic block, no buffer access): A = Z x^ for column t_l and
          // nu NUP q4 ..; B = slice entries regenerated from the kernel (far8's table exp / sincos)
          const double f = sgj * as_t;
          const double zx = zc.x * f, zy = zc.y * f;
          double w[2 * NUP];  // (re, im) of the NUP nu, as digit carriers
#pragma unroll
          for (int u = 0; u < NUP; ++u) {
            const double2 x = xs[(NUP * q4 + u) * kQXP + t_l];
            w[2 * u] = fma(zx, x.x, fma(-zy, x.y, kQMagicA));
            w[2 * u + 1] = fma(zx, x.y, fma(zy, x.x, kQMagicA));
          }
          double e[EB], sn[EB], cs[EB], wr[EB], wi[EB], wn[EB];
#pragma unroll
          for (int eb = 0; eb < EB; ++eb) {
            kern_parts(rw[eb], sv, etab, sctab, e[eb], sn[eb], cs[eb]);
            const double es = e[eb] * isj;
            wr[eb] = fma(es, cs[eb], kQMagicB);
            wi[eb] = fma(-es, sn[eb], kQMagicB);
            wn[eb] = fma(es, sn[eb], kQMagicB);
          }
          uint32_t lo[NG][4], hi[NG][2];
#pragma unroll
          for (int g = 0; g < NG; ++g) {
            tr_lo(__double2loint(w[4 * g]), __double2loint(w[4 * g + 1]), __double2loint(w[4 * g + 2]),
                  __double2loint(w[4 * g + 3]), lo[g]);
            tr_hi(__double2hiint(w[4 * g]), __double2hiint(w[4 * g + 1]), __double2hiint(w[4 * g + 2]),
                  __double2hiint(w[4 * g + 3]), hi[g]);
          }
          // B rows 2 bmu: (Re S, -Im S) at k = 2 nu, 2 nu + 1; 2 bmu + 1: (Im S, Re S)
          uint32_t bw0[6], bw1[6];
          if constexpr (EB == 1) {
            const uint32_t rl = __double2loint(wr[0]), il = __double2loint(wi[0]), nlw = __double2loint(wn[0]);
            const uint32_t rh = __double2hiint(wr[0]), ih = __double2hiint(wi[0]), nh = __double2hiint(wn[0]);
#define FAR10_B(SI, X, Y, Z_, SEL)                                                                        \
  bw0[SI] = __byte_perm(X, Y, SEL) ^ 0x8080u;                                                            \
  bw1[SI] = __byte_perm(Z_, X, SEL) ^ 0x8080u;
            FAR10_B(0, rh, nh, ih, 0x51) FAR10_B(1, rh, nh, ih, 0x40)
            FAR10_B(2, rl, nlw, il, 0x73) FAR10_B(3, rl, nlw, il, 0x62)
            FAR10_B(4, rl, nlw, il, 0x51) FAR10_B(5, rl, nlw, il, 0x40)
#undef FAR10_B
          } else {  // two entries: whole 32-bit words (k = 2 bnu .. 2 bnu + 3) per row and slice
            uint32_t l0[4], h0[2], l1[4], h1[2];
            tr_lo(__double2loint(wr[0]), __double2loint(wn[0]), __double2loint(wr[1]), __double2loint(wn[1]), l0);
            tr_hi(__double2hiint(wr[0]), __double2hiint(wn[0]), __double2hiint(wr[1]), __double2hiint(wn[1]), h0);
            tr_lo(__double2loint(wi[0]), __double2loint(wr[0]), __double2loint(wi[1]), __double2loint(wr[1]), l1);
            tr_hi(__double2hiint(wi[0]), __double2hiint(wr[0]), __double2hiint(wi[1]), __double2hiint(wr[1]), h1);
            bw0[0] = h0[1]; bw0[1] = h0[0]; bw0[2] = l0[3]; bw0[3] = l0[2]; bw0[4] = l0[1]; bw0[5] = l0[0];
            bw1[0] = h1[1]; bw1[1] = h1[0]; bw1[2] = l1[3]; bw1[3] = l1[2]; bw1[4] = l1[1]; bw1[5] = l1[0];
#pragma unroll
            for (int si = 0; si < kQSl; ++si) { bw0[si] ^= 0x80808080u; bw1[si] ^= 0x80808080u; }  // balanced
          }
          // ---- the buffer is free once the MMAs of its previous use completed
          if (stage >= kQNB) tc::mbar_wait_a(empty_a + 8 * buf, ((stage / kQNB) - 1) & 1);
          tc::fence_after();
          {  // A: slice si = 5 - byte (bytes 5, 4 from the hi words, 3 .. 0 from the lo words)
            const uint32_t ta = tA0 + buf * 48 + lane_base + NG * q4;
#pragma unroll
            for (int si = 0; si < kQSl; ++si) {
              uint32_t v[NG];
#pragma unroll
              for (int g = 0; g < NG; ++g) v[g] = si < 2 ? hi[g][1 - si] : lo[g][5 - si];
              if constexpr (NG == 2) tc::tmem_st2(ta + si * 8, v[0], v[1]);
              else tc::tmem_st4(ta + si * 8, *reinterpret_cast<uint32_t(*)[4]>(v));
            }
          }
          {
            uint8_t* sb = sB + buf * kQBStage;
            const uint32_t o0 = boff(2 * bmu, 2 * bnu), o1 = boff(2 * bmu + 1, 2 * bnu);
#pragma unroll
            for (int si = 0; si < kQSl; ++si) {
              if constexpr (EB == 1) {
                *(uint16_t*)(sb + si * kQBSlice + o0) = (uint16_t)bw0[si];
                *(uint16_t*)(sb + si * kQBSlice + o1) = (uint16_t)bw1[si];
              } else {
                *(uint32_t*)(sb + si * kQBSlice + o0) = bw0[si];
                *(uint32_t*)(sb + si * kQBSlice + o1) = bw1[si];
              }
            }
          }
          tc::wait_st();
          tc::fence_proxy_async();
          tc::fence_before();
          __syncwarp();
          if (lane == 0) tc::mbar_arrive_a(full_a + 8 * buf);
          if (ntb > 0) {  // leftover columns on the FP64 pipe (lead CTA; no buffer access)
#pragma unroll
            for (int eb = 0; eb < EB; ++eb) {
              const double sx = e[eb] * cs[eb], sy = -e[eb] * sn[eb];
#pragma unroll
              for (int tl = 0; tl < 2; ++tl) {
                if (tl < ntb) {
                  const double2 zz = lzs[2 * j + tl], xv = xs[(bnu + eb) * kQXP + kQT + tl];
                  const double ax = zz.x * xv.x - zz.y * xv.y, ay = zz.x * xv.y + zz.y * xv.x;
                  lacc[tl].x = fma(sx, ax, fma(-sy, ay, lacc[tl].x));
                  lacc[tl].y = fma(sx, ay, fma(sy, ax, lacc[tl].y));
                }
              }
            }
          }
        }
      }
      }
    }
    if (pending) readout();
    // (6) this segment's partial: columns 16 q4 .. 16 q4 + 15 = rows mu 8 q4 .. 8 q4 + 7 (Re, Im)
    double2* out = a.part + (int64_t)sg.w * a.nl * p;
    if (tg >= 0) {
#pragma unroll
      for (int i = 0; i < NCOL / 2; ++i) {
        const int mu = (NCOL / 2) * q4 + i;
        if (mu < nrow) {
          BEM_DASSERT((out - a.part) + (int64_t)tg * p + mu0 + mu < a.part_n);
          out[(int64_t)tg * p + mu0 + mu] = tv ? make_double2(acc[2 * i * kQT], acc[(2 * i + 1) * kQT]) : make_double2(0.0, 0.0);
        }
      }
    }
#pragma unroll
    for (int tl = 0; tl < 2; ++tl) {
      if (tl >= ntb) break;
      double2 v = lacc[tl];
#pragma unroll
      for (int o = 1; o < (EB == 1 ? 16 : 8); o <<= 1) {  // the lanes holding the row's nu
        v.x += __shfl_xor_sync(0xffffffffu, v.x, o);
        v.y += __shfl_xor_sync(0xffffffffu, v.y, o);
      }
      if (bnu == 0 && bmu < nrow) out[(int64_t)tl * p + mu0 + bmu] = v;
    }
  }
  }  // work items
  if (tid == 0) *(volatile int*)&k3done = 1;
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(taddr_s, kQCols);
}

// (block, frequency tile) underflow mask of the coupling step ("K3 underflow mask").
// The compressed block of frequency t is sum_j S_b(s_{k_j}) Z_b[j, t] (eq:maca P:1314-1320); with
// r_lb = the distance of the two clusters' node boxes, |S_b(s)[mu, nu]| = e^{-Re s r} / (4 pi r)
// <= g_j := e^{-Re s_{k_j} r_lb} / (4 pi r_lb) (Re s >= 0), so every entry of the fibre is bounded
// by beta_t = sum_j g_j |Z_b[j, t]|.  At the strongly damped CQM frequencies (Re s_t r >> 1) the
// far field underflows against the O(1 / |s_t|) diagonal of V(s_t): a tile whose columns all have
// beta_t max(|s_t|, 1, 1 / (4 hmax)) < delta (2^-70; hmax = the mesh's largest node-to-centroid
// distance: the diagonal is O(1 / |s|) only while |s| h >> 1, O(h) below) is not computed.  The mask depends on the skeleton only
// (not on x): one pass at assembly (stored Z) or per regenerated tile (factors-only; the Z
// columns are bitwise the same, hence the same mask).
__global__ void __launch_bounds__(kQT) far10_skip_kernel(const Far10SkipArgs a) {
  __shared__ double gs[512];
  __shared__ double gap[3];
  const int tid = threadIdx.x;
  for (int b = blockIdx.x; b < a.nfar; b += gridDim.x) {
    const int rk = a.rank[b];
    __syncthreads();  // gs / gap of the previous block
    if (tid < 3) {
      const double* xr = a.xi + (int64_t)a.far_r[b] * 3 * a.m + tid * a.m;
      const double* xc = a.xi + (int64_t)a.far_c[b] * 3 * a.m + tid * a.m;
      double lr = xr[0], hr = xr[0], lc = xc[0], hc = xc[0];
      for (int i = 1; i < a.m; ++i) {
        lr = fmin(lr, xr[i]); hr = fmax(hr, xr[i]);
        lc = fmin(lc, xc[i]); hc = fmax(hc, xc[i]);
      }
      gap[tid] = fmax(0.0, fmax(lr - hc, lc - hr));
    }
    __syncthreads();
    const double rlb = sqrt(gap[0] * gap[0] + gap[1] * gap[1] + gap[2] * gap[2]) * (1.0 - 0x1p-40);
    for (int j = tid; j < rk; j += kQT) {
      const double sre = a.s[a.pivk[(int64_t)b * a.rcap + j]].x;
      gs[j] = (rlb > 0.0 && sre >= 0.0) ? exp(-sre * rlb) * (0.079577471545947667884 / rlb) * (1.0 + 0x1p-30)
                                         : __longlong_as_double(0x7ff0000000000000LL);
    }
    __syncthreads();
    uint32_t bits = a.skip[b];
    for (int tile = a.tile_lo; tile < a.tile_hi; ++tile) {
      const int tc0 = a.tb + tile * kQT;
      const int ncol = min(kQT, a.tb + a.nd - tc0);
      const double2 *zD, *zL;
      int zst;
      zrows(a.z, b, a.nl, a.tb, tc0, zD, zL, zst);
      bool keep = false;
      auto column = [&](const double2* zc, int t) {  // zc: the column's Z entries (stride zst), t: local frequency
        double beta = 0.0;
        for (int j = 0; j < rk; ++j) {
          const double2 z = zc[(int64_t)j * zst];
          beta = fma(sqrt(fma(z.x, z.x, z.y * z.y)), gs[j], beta);
        }
        const double2 st = a.s[a.local_l[t]];
        const double v = beta * (1.0 + 0x1p-20) * fmax(sqrt(fma(st.x, st.x, st.y * st.y)), a.sref);
        if (!(v < a.delta)) keep = true;  // NaN / inf keep the tile
      };
      const int t = tid < ncol ? a.colmap[tile * kQT + tid] : -1;
      if (t >= 0) column(zD + (a.z.tiled ? tc0 + tid : t), t);
      if (tile == 0 && tid < a.tb) column(zL + tid, tid);  // leftover columns ride with tile 0
      keep = __syncthreads_or(keep) || rk > 512;
      bits = keep ? bits & ~(1u << tile) : bits | (1u << tile);
    }
    if (tid == 0) a.skip[b] = bits;
  }
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

cudaError_t launch_far10(const Far10Args& a, int nseg, int ntile, cudaStream_t st, int nearw) {
  static const int pw = [] { const char* e = getenv("BEM_FAR10_PW"); return e ? atoi(e) : 8; }();  // r3d: 8 warps 912 ms, 16 warps 934 ms (config 4)
  const size_t need = kQNB * (size_t)kQBStage + sizeof(double2) * (2 * (size_t)kQKC * kQXP) +
                      sizeof(double) * (8 * (size_t)a.rcap + (size_t)kQN * kQT) + 64;
  const size_t smem = need > kQMinSmem ? need : kQMinSmem;
  const bool fused = a.nctr != nullptr && nearw > 0 && pw == 8;
  auto k = pw != 8 ? far10_kernel<16, 0>
           : !fused ? far10_kernel<8, 0>
           : nearw == 1 ? far10_kernel<8, 1> : nearw == 2 ? far10_kernel<8, 2> : far10_kernel<8, 3>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const unsigned nthr = (pw == 8 ? 8 : 16) * 32 + 32 + (fused ? std::min(nearw, 3) * 32 : 0);
  Far10Args b = a;
  b.gx = nseg * a.nch;
  b.nitems = b.gx * ntile;
  if (b.ctr != nullptr) {  // persistent: one CTA per SM, items from the counter (zeroed here, in stream order)
    int dev = 0, nsm = 0;
    if ((e = cudaGetDevice(&dev)) != cudaSuccess) return e;
    if ((e = cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess) return e;
    if ((e = cudaMemsetAsync(b.ctr, 0, sizeof(int), st)) != cudaSuccess) return e;
    k<<<(unsigned)std::max(1, std::min(b.nitems, nsm)), nthr, smem, st>>>(b);
  } else {
    k<<<dim3((unsigned)b.gx, (unsigned)ntile, 1u), nthr, smem, st>>>(b);
  }
  return cudaGetLastError();
}

cudaError_t launch_far10_skip(const Far10SkipArgs& a, cudaStream_t st) {
  if (a.nfar <= 0 || a.tile_hi <= a.tile_lo) return cudaSuccess;
  far10_skip_kernel<<<(unsigned)std::min(a.nfar, 148 * 16), kQT, 0, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_xmax(const double2* xhat, int64_t rows, int p, double* out, cudaStream_t st) {
  xmax_kernel<<<(unsigned)((rows + 7) / 8), 256, 0, st>>>(xhat, rows, p, out);
  return cudaGetLastError();
}

}  // namespace bem
