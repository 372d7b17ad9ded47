// K3: far-field coupling.
//
// For each admissible block b = (r,c) (eq:qadm P:905-912) the coupling tensor
// S_b[mu,nu,l] = k(|xi_{c,nu} - xi_{r,mu}|; s_l) is represented
// by its MACA skeleton (eq:maca P:1314-1320, Alg. 2):
//   S_b(s_l) ~= sum_{j<r_b} Z_b[j,l] S_b(s_{k_j}),
// so the coupling step of the H^2 matvec is
//   yhat_r[:,t] += sum_b sum_j S_b(s_{k_j}) (Z_b[j,t] xhat_c[:,t]).
// Only the pivot slices S_b(s_{k_j}) are evaluated ("only pivot frequencies
// are evaluated", north_star); they are regenerated on the fly from the
// kernel (no slice storage: 223 GB at config 4).  The
// coefficients Z_b come either from the stored pool or, in the factors-only
// skeleton (BEM_SKEL_FACTORS), from the blocks' r_b x r_b LU factors: the
// coupling then runs one frequency tile at a time, and before each tile
// zgen_tile_kernel regenerates every block's Z columns of the tile (pivot
// fibres + two pinned triangular solves, zgen.cuh) into a tile buffer
// (sum_b r_b x 130 complex: 7 GB at config 4 instead of 28 GB of stored Z),
// which the unchanged coupling kernel reads.  (A first version regenerated the
// tile in each CTA's block prologue; that serialised the substitutions inside
// the GEMM kernel and cost it 20-40 %: profiles/r02_factors.md.)
//
// Kernels (all deterministic: one CTA owns each output tile of a segment's
// partial sum; segments of a row are reduced in fixed order, no atomics):
//   far8_kernel / far7_kernel (default, p > 32 / p <= 32): the per-term slice
//     product on the FP64 tensor cores (mma.sync m8n8k4 f64), slices
//     regenerated in shared memory -- DESIGN.md §7;
//   h2o_kernel: BEM_MODE_H2ONLY, couplings evaluated per frequency on the fly
//     (the paper's plain-H^2 comparison);
//   far_generic_kernel: fallback for shapes the tiled kernels cannot hold
//     (stored Z only).
// Variants measured slower in round 1 (far6, DSMEM-shared slices, 16- and
// 6-warp CTAs, 3M complex products, split remainder rows) were removed; they
// are in git history and profiles/r01_sweeps.md.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <type_traits>
#include <vector>

#include "common.cuh"
#include "fastmath.cuh"
#include "zgen.cuh"
#include "far_common.cuh"

namespace bem {
namespace {

__device__ __forceinline__ void cmac(double2& acc, double2 a, double2 b) {
  acc.x = fma(a.x, b.x, acc.x);
  acc.x = fma(-a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y);
  acc.y = fma(a.y, b.x, acc.y);
}

__device__ __forceinline__ double2 kern(double r, double2 s) {
  const double e = fast::exp_neg(-s.x * r) / (12.566370614359172954 * r);
  double sn, cs;
  fast::sincos_(s.y * r, &sn, &cs);
  return make_double2(e * cs, -e * sn);
}

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// slice entry k(r; s) with rsqrt (no IEEE division / sqrt) and the table exp / sincos
__device__ __forceinline__ double2 kern_rs(double d2, double2 s, const double* etab, const double2* sctab) {
  const double ir = rsqrt(d2);
  const double r = d2 * ir;
  const double e = fast::exp_neg_tab(-s.x * r, etab) * (ir * 0.079577471545947667884);  // 1/(4 pi)
  double sn, cs;
  fast::sincos_tab(s.y * r, sctab, &sn, &cs);
  return make_double2(e * cs, -e * sn);
}

// Factors-only skeleton: the Z columns of one frequency tile for every far block
// (zgen.cuh; the same function as the stored-Z regeneration, hence bit-identical).
// CTA per block (grid-stride); columns in batches of nb in shared memory: the pivot
// fibres over all threads, then one column per thread for the two substitutions, then
// a coalesced copy to the tile buffer.
__global__ void __launch_bounds__(256) zgen_tile_kernel(zgen::Src g, int nfar, const int32_t* __restrict__ rank,
                                                        const int64_t* __restrict__ ztoff,
                                                        const int32_t* __restrict__ local_l,
                                                        const int32_t* __restrict__ mask, int nl, int tb, int tc0,
                                                        int ncol, int lead, int ZW, int cap, double2* __restrict__ Zt,
                                                        int64_t zt_n, const int32_t* __restrict__ cmap) {
  extern __shared__ double2 work[];
  const int ncp = tb + ncol;
  for (int b = blockIdx.x; b < nfar; b += gridDim.x) {
    double2* out = Zt + ztoff[b];
    BEM_DASSERT(ztoff[b] + (int64_t)rank[b] * ZW <= zt_n);
    zgen::block_columns(
        g, b, rank[b], lead ? 0 : tb, ncp,
        [&](int c) {
          // cmap (far10): the tile's columns in its damping order; else the natural order
          const int t = c < tb ? c : cmap != nullptr ? cmap[c - tb] : tc0 + (c - tb);
          return (t >= 0 && t < nl && (mask == nullptr || mask[t])) ? local_l[t] : -1;
        },
        work, cap, [&](int j, int c, double2 v) { out[(int64_t)j * ZW + c] = v; });
  }
}

// ------------------------------------------------ far7: p <= 32, whole p staged
// out[t, mu] += sum_j sum_nu (Z_b[j,t] xhat_c[nu,t]) S_b(s_{k_j})[mu,nu]
// as an (M = t) x (N = mu) x (K = nu) FP64 tensor-core product per term j:
//   A[t,nu] = Z_b[j,t] xhat_c[nu,t]  (formed in registers from the shared-memory
//             xhat tile and the thread's Z values: one complex multiply per
//             fragment, reused for the mu tiles),
//   B[nu,mu] = S_b(s_{k_j})[mu,nu]   (the regenerated slice rows in shared memory,
//             double-buffered: one barrier per term, warps may run a term apart).
// NJ DMMA mu tiles per 32-row chunk; REM further rows (p = 27: rows 24..26) on
// DFMA from the same A fragments instead of a 5/8-empty fourth DMMA tile.  Up to
// two leftover columns (n_l mod 8, e.g. the real l = 0 when L = 2^k + 1) are
// accumulated by all 256 threads of the lead CTA; more are zero-padded DMMA columns.
struct Far7Args {
  int nl, m, p, p4, rcap, SST, TT, XTP, tb, nd;  // DMMA columns [tb, tb+nd) (padded past nl)
  int64_t part_n = 0;                            // elements of part (bounds checks)
  int tile0 = 0;                                 // first frequency tile of this launch (grid y offset)
  const int4* segs;
  const int32_t* far_sorted;
  const int32_t* far_c;
  const double* xi;
  const double2* s;
  const int32_t* rank;
  const int32_t* pivk;
  ZSrc z;
  const double2* xhat;
  double2* part;
  const int32_t* mask;  // nullable: per local frequency, 0 = skip (output 0)
};

template <int MT, int NJ, int REM>
__global__ void __launch_bounds__(256, 2) far7_kernel(Far7Args a) {
  extern __shared__ double2 sm[];
  const int p = a.p, m = a.m, SST = a.SST, XTP = a.XTP, p4 = a.p4, tb = a.tb;
  const int4 sg = a.segs[blockIdx.x];
  const int r = sg.x;
  const int tile = blockIdx.y + a.tile0;
  const int tc0 = a.tb + tile * a.TT;
  const int ncol = min(a.TT, a.tb + a.nd - tc0);
  const bool lead = tile == 0;
  const int mu0 = blockIdx.z * 32;
  const int nrow = min(32, p - mu0);
  const int nS = nrow * p;
  double2* S0 = sm;                                   // 2 x (32 x SST): double-buffered slice rows
  double2* xs = S0 + 2 * 32 * SST;                    // p4 x XTP
  double2* sctab = xs + (size_t)p4 * XTP;             // 64 (cos, sin)(k pi/32)
  double* etab = (double*)(sctab + 64);               // 64
  double* xr = etab + 64;                             // 96
  double* xcn = xr + 96;                              // 3p
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, q = lane & 3;
  for (int i = tid; i < 2 * 32 * SST + p4 * XTP; i += blockDim.x) sm[i] = make_double2(0.0, 0.0);
  for (int i = tid; i < 64; i += blockDim.x) {
    etab[i] = fast::kExp2Tab[i];
    sctab[i] = fast::kSinCosTab[i];
  }
  for (int i = tid; i < nrow; i += blockDim.x) node(a.xi + (int64_t)r * 3 * m, m, mu0 + i, xr + 3 * i);
  const int ntile = ncol / 8;
  bool ton[MT];  // 8-column frequency tile has at least one unmasked column (GMRES mask)
  bool cta_on = false;
#pragma unroll
  for (int i = 0; i < MT; ++i) {
    const int tt = warp + 8 * i;
    const int t = tc0 + tt * 8 + g;
    const bool v = tt < ntile && t < a.nl && (a.mask == nullptr || a.mask[t]);
    ton[i] = __any_sync(0xffffffffu, v);
  }
  {
    int lo = 0;
    for (int t = tid; t < ncol; t += blockDim.x) lo |= (tc0 + t < a.nl) && (a.mask == nullptr || a.mask[tc0 + t]);
    if (lead) for (int t = tid; t < tb; t += blockDim.x) lo |= a.mask == nullptr || a.mask[t];
    cta_on = __syncthreads_or(lo) != 0;
  }
  double acc[MT][NJ > 0 ? NJ : 1][2][2];
  double2 racc[MT][REM > 0 ? REM : 1];
#pragma unroll
  for (int i = 0; i < MT; ++i) {
#pragma unroll
    for (int j = 0; j < NJ; ++j) acc[i][j][0][0] = acc[i][j][0][1] = acc[i][j][1][0] = acc[i][j][1][1] = 0.0;
#pragma unroll
    for (int j = 0; j < (REM > 0 ? REM : 1); ++j) racc[i][j] = make_double2(0.0, 0.0);
  }
  // leftover columns: thread -> (row lrow, nu residue lpart)
  const int lrow = tid >> 3, lpart = tid & 7;
  const bool lown = lead && tb > 0 && lrow < nrow;
  // leftover-column accumulators in shared memory (registers would be live through the
  // whole kernel and spill)
  double2* lacc = (double2*)(((uintptr_t)(xcn + 3 * p) + 15) & ~(uintptr_t)15) + 2 * tid;
  lacc[0] = lacc[1] = make_double2(0.0, 0.0);
  const int ncp = tb + ncol;
  for (int bi = sg.y; bi < (cta_on ? sg.z : sg.y); ++bi) {
    const int b = a.far_sorted[bi];
    const int c = a.far_c[b];
    const int rk = a.rank[b];
    __syncthreads();
    const double2 *zD, *zL;
    int zst;
    zrows(a.z, b, a.nl, tb, tc0, zD, zL, zst);
    for (int i = tid; i < p; i += blockDim.x) node(a.xi + (int64_t)c * 3 * m, m, i, xcn + 3 * i);
    const double2* xh = a.xhat + (int64_t)c * a.nl * p;
    for (int idx = tid; idx < ncp * p; idx += blockDim.x) {
      const int tl = idx / p, nu = idx - tl * p;
      const int tg = tl < tb ? tl : tc0 + (tl - tb);
      BEM_DASSERT(nu < p4 && tl < XTP);
      if (tl >= tb || lead) xs[nu * XTP + tl] = tg < a.nl ? xh[(int64_t)tg * p + nu] : make_double2(0.0, 0.0);
    }
    __syncthreads();
    for (int l = 0; l < rk; ++l) {
      double2* S = S0 + (l & 1) * 32 * SST;
      const double2 sv = a.s[a.pivk[(int64_t)b * a.rcap + l]];
      const bool real_slice = sv.y == 0.0;
      const double2* Zl = zD + (int64_t)l * zst;
      double2 zt[MT];
#pragma unroll
      for (int i = 0; i < MT; ++i) {
        const int tt = warp + 8 * i;
        const int t = tc0 + tt * 8 + g;
        BEM_DASSERT(!(tt < ntile && t < a.nl) || (Zl + t >= a.z.Z && Zl + t < a.z.Z + a.z.zn));
        zt[i] = (tt < ntile && t < a.nl) ? Zl[t] : make_double2(0.0, 0.0);
      }
      for (int e = tid; e < nS; e += blockDim.x) {
        const int i = e / p, nu = e - i * p;
        const double dx = xcn[3 * nu] - xr[3 * i], dy = xcn[3 * nu + 1] - xr[3 * i + 1],
                     dz = xcn[3 * nu + 2] - xr[3 * i + 2];
        S[i * SST + nu] = kern_rs(dx * dx + dy * dy + dz * dz, sv, etab, sctab);
      }
      __syncthreads();
      // the real pivot slice (s_0) needs two DMMAs per complex MAC: the branch is hoisted out
      // of the k loop (one loop body per case)
      auto gemm = [&](auto realc) {
        constexpr bool RS = decltype(realc)::value;
      for (int k0 = 0; k0 < p4; k0 += 4) {
        double2 bf[NJ > 0 ? NJ : 1], rf[REM > 0 ? REM : 1];
#pragma unroll
        for (int j = 0; j < NJ; ++j) bf[j] = S[(j * 8 + g) * SST + k0 + q];
#pragma unroll
        for (int j = 0; j < REM; ++j) rf[j] = S[(NJ * 8 + j) * SST + k0 + q];
#pragma unroll
        for (int i = 0; i < MT; ++i) {
          const int tt = warp + 8 * i;
          if (tt < ntile && ton[i]) {
            const double2 xv = xs[(k0 + q) * XTP + tb + tt * 8 + g];
            const double ar = zt[i].x * xv.x - zt[i].y * xv.y;
            const double ai = zt[i].x * xv.y + zt[i].y * xv.x;
            const double nai = -ai;
            if constexpr (RS) {  // pivot frequency s_0 is real: Im S = 0, two DMMAs per complex MAC
#pragma unroll
              for (int j = 0; j < NJ; ++j) {
                dmma(acc[i][j][0][0], acc[i][j][0][1], ar, bf[j].x);
                dmma(acc[i][j][1][0], acc[i][j][1][1], ai, bf[j].x);
              }
            } else {
              // two passes: dependent DMMAs on one accumulator are 2*NJ instructions apart
#pragma unroll
              for (int j = 0; j < NJ; ++j) {
                dmma(acc[i][j][0][0], acc[i][j][0][1], ar, bf[j].x);
                dmma(acc[i][j][1][0], acc[i][j][1][1], ar, bf[j].y);
              }
#pragma unroll
              for (int j = 0; j < NJ; ++j) {
                dmma(acc[i][j][0][0], acc[i][j][0][1], nai, bf[j].y);
                dmma(acc[i][j][1][0], acc[i][j][1][1], ai, bf[j].x);
              }
            }
#pragma unroll
            for (int j = 0; j < REM; ++j) {  // partial over this lane's k = k0 + q; reduced over q at the end
              racc[i][j].x = fma(ar, rf[j].x, fma(nai, rf[j].y, racc[i][j].x));
              racc[i][j].y = fma(ar, rf[j].y, fma(ai, rf[j].x, racc[i][j].y));
            }
          }
        }
      }
      };
      if (real_slice) gemm(std::true_type{});
      else gemm(std::false_type{});
      if (lown) {
#pragma unroll
        for (int tl = 0; tl < 2; ++tl) {
          if (tl >= tb) break;
          double2 sacc = make_double2(0.0, 0.0);
          for (int nu = lpart; nu < p; nu += 8) {
            const double2 sv2 = S[lrow * SST + nu], xv = xs[nu * XTP + tl];
            sacc.x = fma(sv2.x, xv.x, sacc.x);
            sacc.x = fma(-sv2.y, xv.y, sacc.x);
            sacc.y = fma(sv2.x, xv.y, sacc.y);
            sacc.y = fma(sv2.y, xv.x, sacc.y);
          }
          const double2 zz = zL[(int64_t)l * zst + tl];
          lacc[tl].x = fma(zz.x, sacc.x, fma(-zz.y, sacc.y, lacc[tl].x));
          lacc[tl].y = fma(zz.x, sacc.y, fma(zz.y, sacc.x, lacc[tl].y));
        }
      }
    }
  }
  double2* out = a.part + (int64_t)sg.w * a.nl * p;
#pragma unroll
  for (int i = 0; i < MT; ++i) {
    const int tt = warp + 8 * i;
    if (tt >= ntile) continue;
    const int t = tc0 + tt * 8 + g;
    if (t >= a.nl) continue;
#pragma unroll
    for (int j = 0; j < NJ; ++j)
#pragma unroll
      for (int v = 0; v < 2; ++v) {
        const int row = j * 8 + 2 * q + v;
        if (row < nrow) {
          BEM_DASSERT((out - a.part) + (int64_t)t * p + mu0 + row < a.part_n);
          out[(int64_t)t * p + mu0 + row] = make_double2(acc[i][j][0][v], acc[i][j][1][v]);
        }
      }
  }
  if (REM > 0) {
#pragma unroll
    for (int i = 0; i < MT; ++i) {
      const int tt = warp + 8 * i;  // warp-uniform
      if (tt >= ntile) continue;
      const int t = tc0 + tt * 8 + g;
#pragma unroll
      for (int j = 0; j < (REM > 0 ? REM : 1); ++j) {
        double2 v = racc[i][j];
        v.x += __shfl_xor_sync(0xffffffffu, v.x, 1);
        v.y += __shfl_xor_sync(0xffffffffu, v.y, 1);
        v.x += __shfl_xor_sync(0xffffffffu, v.x, 2);
        v.y += __shfl_xor_sync(0xffffffffu, v.y, 2);
        if (q == 0 && t < a.nl && NJ * 8 + j < nrow) out[(int64_t)t * p + mu0 + NJ * 8 + j] = v;
      }
    }
  }
  if (lead && tb > 0) {  // uniform per warp: reduce the 8 nu residues of each row
#pragma unroll
    for (int tl = 0; tl < 2; ++tl) {
      if (tl >= tb) break;
      double2 v = lacc[tl];
#pragma unroll
      for (int off = 1; off < 8; off <<= 1) {
        v.x += __shfl_xor_sync(0xffffffffu, v.x, off);
        v.y += __shfl_xor_sync(0xffffffffu, v.y, off);
      }
      if (lpart == 0 && lrow < nrow) out[(int64_t)tl * p + mu0 + lrow] = v;
    }
  }
}

struct Far7Cfg {
  int p4 = 0, SST = 0, TT = 0, XTP = 0, tb = 0, nd = 0, ntiles = 0, nchunks = 0, mt = 0;
  size_t smem = 0;
};

Far7Cfg choose7(int p, int nl, size_t cap) {
  int tb = nl % 8;
  if (tb > 2 || tb == nl) tb = 0;  // pad instead (zero columns past nl)
  const int nD = (nl - tb + 7) / 8 * 8;
  const int p4 = (p + 3) / 4 * 4;
  int SST = p4;
  while (SST % 8 != 4) ++SST;
  for (int TTmax : {256, 128, 64, 32, 16, 8}) {
    Far7Cfg c;
    const int ntiles = (nD + TTmax - 1) / TTmax;
    const int TT = ((nD / 8 + ntiles - 1) / ntiles) * 8;
    int XTP = tb + TT;
    while (XTP % 8 != 2) ++XTP;
    const size_t smem = sizeof(double2) * (2 * 32 * (size_t)SST + (size_t)p4 * XTP + 64 + 2 * 256) + 16 +
                        sizeof(double) * (64 + 96 + 3 * p);
    if (smem > cap) continue;
    c.p4 = p4; c.SST = SST; c.TT = TT; c.XTP = XTP; c.tb = tb; c.nd = nD; c.ntiles = ntiles;
    c.nchunks = (p + 31) / 32; c.mt = (TT / 8 + 7) / 8; c.smem = smem;
    if (c.mt > 2) continue;  // MT >= 3 spills at 128 registers
    return c;
  }
  return Far7Cfg{};
}

template <int MT, int NJ, int REM>
cudaError_t launch7(const Far7Cfg& c, int nseg, const Far7Args& a, int ntile, cudaStream_t st) {
  auto k = far7_kernel<MT, NJ, REM>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)c.smem);
  if (e != cudaSuccess) return e;
  k<<<dim3((unsigned)nseg, (unsigned)ntile, (unsigned)c.nchunks), 256, c.smem, st>>>(a);
  return cudaGetLastError();
}

template <int NJ, int REM>
cudaError_t dispatch7_(const Far7Cfg& c, int nseg, const Far7Args& a, int ntile, cudaStream_t st) {
  return c.mt == 1 ? launch7<1, NJ, REM>(c, nseg, a, ntile, st) : launch7<2, NJ, REM>(c, nseg, a, ntile, st);
}

// mu tiling: p = 27 -> 3 DMMA tiles + 3 DFMA rows; p <= 8 -> 1 tile; otherwise 4 tiles per 32-row chunk
// ntile frequency tiles from a.tile0 (grid y)
cudaError_t dispatch7(const Far7Cfg& c, int p, int nseg, const Far7Args& a, int ntile, cudaStream_t st) {
  if (p <= 8) return dispatch7_<1, 0>(c, nseg, a, ntile, st);
  if (p == 27) return dispatch7_<3, 3>(c, nseg, a, ntile, st);
  return dispatch7_<4, 0>(c, nseg, a, ntile, st);
}

// ------------------------------------------------ far8: far7 with K (nu) chunks
// The contraction index nu is processed in chunks of KC (a multiple of 4): per
// block, for each nu chunk the x^ tile [KC][TT] is staged once, and for each
// ACA term j the slice columns S_j[mu-chunk][nu-chunk] are regenerated and
// contracted.  Regeneration per (b, j) is unchanged (every slice entry is
// evaluated once per CTA), but shared memory no longer grows with p, so the
// frequency tile stays at TT = 128 with two CTAs per SM for p = 64 and 125.
struct Far8Args {
  int nl, m, p, rcap, SST, TT, XTP, tb, nd, KC;
  int64_t part_n = 0;  // elements of part (bounds checks)
  int tile0 = 0;  // first frequency tile of this launch (grid y offset)
  int nch = 1;  // mu chunks (grid x = segment * nch + chunk)
  const int4* segs;
  const int32_t* far_sorted;
  const int32_t* far_c;
  const double* xi;
  const double2* s;
  const int32_t* rank;
  const int32_t* pivk;
  ZSrc z;
  const double2* xhat;
  double2* part;
  const int32_t* mask;  // nullable: per local frequency, 0 = skip (output 0)
};

// M3: three real DMMA products per complex one (P1 = Ar Br, P2 = Ai Bi, P3 = (Ar + Ai)(Br + Bi);
// Re = P1 - P2, Im = P3 - P1 - P2): 25 % fewer DMMAs for a third accumulator, which fits
// at NJ = 2 (16-row mu chunks); the real slice S_b(s_0) takes P1 and P3 only.
// DT: the block's (r, 1/(4 pi r)) table [RW][p] in shared memory, computed once per block,
// so the per-term slice regeneration skips the distance (rsqrt) work.
template <int MT, int NJ, int REM, bool M3 = false, bool DT = false>
__global__ void __launch_bounds__(256, 2) far8_kernel(Far8Args a) {
  constexpr int RW = NJ * 8 + REM;  // mu rows per CTA
  constexpr int NA = M3 ? 3 : 2;    // accumulators per (tile, mu tile)
  extern __shared__ double2 sm[];
  const int p = a.p, m = a.m, SST = a.SST, XTP = a.XTP, tb = a.tb, KC = a.KC;
  // the mu chunks of one (segment, tile) are adjacent CTAs: the second chunk re-reads the
  // x^ and Z tiles from L2 instead of DRAM
  const int4 sg = a.segs[blockIdx.x / a.nch];
  const int r = sg.x;
  const int tile = blockIdx.y + a.tile0;
  const int tc0 = a.tb + tile * a.TT;
  const int ncol = min(a.TT, a.tb + a.nd - tc0);
  const bool lead = tile == 0;
  const int mu0 = (blockIdx.x % a.nch) * RW;
  const int nrow = min(RW, p - mu0);
  double2* S0 = sm;                                   // 2 x (RW x SST), SST >= KC: double-buffered slice
  double2* xs = S0 + 2 * RW * SST;                    // KC x XTP
  double2* sctab = xs + (size_t)KC * XTP;             // 64 (cos, sin)(k pi/32)
  double* etab = (double*)(sctab + 64);               // 64
  double* xr = etab + 64;                             // 96
  double* xcn = xr + 96;                              // 3p
  double2* dtab = (double2*)(((uintptr_t)(xcn + 3 * p) + 15) & ~(uintptr_t)15);  // DT: [RW][p]
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, q = lane & 3;
  for (int i = tid; i < 2 * RW * SST + KC * XTP; i += blockDim.x) sm[i] = make_double2(0.0, 0.0);
  int sbuf = 0;
  for (int i = tid; i < 64; i += blockDim.x) {
    etab[i] = fast::kExp2Tab[i];
    sctab[i] = fast::kSinCosTab[i];
  }
  for (int i = tid; i < nrow; i += blockDim.x) node(a.xi + (int64_t)r * 3 * m, m, mu0 + i, xr + 3 * i);
  const int ntile = ncol / 8;
  bool ton[MT];  // 8-column frequency tile has at least one unmasked column (GMRES mask)
  bool cta_on = false;
#pragma unroll
  for (int i = 0; i < MT; ++i) {
    const int tt = warp + 8 * i;
    const int t = tc0 + tt * 8 + g;
    const bool v = tt < ntile && t < a.nl && (a.mask == nullptr || a.mask[t]);
    ton[i] = __any_sync(0xffffffffu, v);
  }
  {
    int lo = 0;
    for (int t = tid; t < ncol; t += blockDim.x) lo |= (tc0 + t < a.nl) && (a.mask == nullptr || a.mask[tc0 + t]);
    if (lead) for (int t = tid; t < tb; t += blockDim.x) lo |= a.mask == nullptr || a.mask[t];
    cta_on = __syncthreads_or(lo) != 0;
  }
  double acc[MT][NJ][NA][2];
  double2 racc[MT][REM > 0 ? REM : 1];
#pragma unroll
  for (int i = 0; i < MT; ++i) {
#pragma unroll
    for (int j = 0; j < NJ; ++j)
#pragma unroll
      for (int u = 0; u < NA; ++u) acc[i][j][u][0] = acc[i][j][u][1] = 0.0;
#pragma unroll
    for (int j = 0; j < (REM > 0 ? REM : 1); ++j) racc[i][j] = make_double2(0.0, 0.0);
  }
  const int lrow = tid >> 3, lpart = tid & 7;
  const bool lown = lead && tb > 0 && lrow < nrow;
  double2 lacc[2] = {make_double2(0.0, 0.0), make_double2(0.0, 0.0)};
  const int ncp = tb + ncol;
  for (int bi = sg.y; bi < (cta_on ? sg.z : sg.y); ++bi) {
    const int b = a.far_sorted[bi];
    const int c = a.far_c[b];
    const double2* xh = a.xhat + (int64_t)c * a.nl * p;
    const int rk = a.rank[b];
    __syncthreads();
    const double2 *zD, *zL;
    int zst;
    zrows(a.z, b, a.nl, tb, tc0, zD, zL, zst);
    if constexpr (DT) {
      for (int e = tid; e < nrow * p; e += blockDim.x) {
        const int i = e / p, nu = e - i * p;
        double cn[3];
        node(a.xi + (int64_t)c * 3 * m, m, nu, cn);
        const double dx = cn[0] - xr[3 * i], dy = cn[1] - xr[3 * i + 1], dz = cn[2] - xr[3 * i + 2];
        dtab[e] = dist_pair(dx * dx + dy * dy + dz * dz);
      }
    } else {
      for (int i = tid; i < p; i += blockDim.x) node(a.xi + (int64_t)c * 3 * m, m, i, xcn + 3 * i);
    }
    for (int k0c = 0; k0c < p; k0c += KC) {
      const int kw = min(KC, p - k0c);          // real nu in this chunk
      const int kw4 = (kw + 3) & ~3;            // k-steps cover kw4 (padding rows/cols are zero)
      if (k0c > 0) __syncthreads();             // previous chunk's GEMM done with xs
      for (int idx = tid; idx < ncp * KC; idx += blockDim.x) {
        const int tl = idx / KC, nu = idx - tl * KC;
        const int tg = tl < tb ? tl : tc0 + (tl - tb);
        BEM_DASSERT(nu < KC && tl < XTP);
        if (tl >= tb || lead)
          xs[nu * XTP + tl] = (nu < kw && tg < a.nl) ? xh[(int64_t)tg * p + k0c + nu] : make_double2(0.0, 0.0);
      }
      for (int l = 0; l < rk; ++l) {
        const double2 sv = a.s[a.pivk[(int64_t)b * a.rcap + l]];
        const bool real_slice = sv.y == 0.0;
        // S alternates between two buffers: one barrier per term, and warps may
        // run one term apart (regeneration overlaps other warps' DMMA work)
        double2* S = S0 + sbuf * RW * SST;
        sbuf ^= 1;
        if (l == 0) __syncthreads();  // xs / node coordinates / Z tile staged
        const double2* Zl = zD + (int64_t)l * zst;
        double2 zt[MT];
#pragma unroll
        for (int i = 0; i < MT; ++i) {
          const int tt = warp + 8 * i;
          const int t = tc0 + tt * 8 + g;
          BEM_DASSERT(!(tt < ntile && t < a.nl) || (Zl + t >= a.z.Z && Zl + t < a.z.Z + a.z.zn));
          zt[i] = (tt < ntile && t < a.nl) ? Zl[t] : make_double2(0.0, 0.0);
        }
        for (int e = tid; e < nrow * KC; e += blockDim.x) {
          const int i = e / KC, nu = e - i * KC;
          double2 v = make_double2(0.0, 0.0);
          if (nu < kw) {
            const int nn = k0c + nu;
            if constexpr (DT) {
              v = kern_tab(dtab[i * p + nn], sv, etab, sctab);
            } else {
              const double dx = xcn[3 * nn] - xr[3 * i], dy = xcn[3 * nn + 1] - xr[3 * i + 1],
                           dz = xcn[3 * nn + 2] - xr[3 * i + 2];
              v = kern_rs(dx * dx + dy * dy + dz * dz, sv, etab, sctab);
            }
          }
          BEM_DASSERT(i < RW && nu < SST);
          S[i * SST + nu] = v;
        }
        __syncthreads();
        auto gemm = [&](auto realc) {  // real pivot slice: two DMMAs per complex MAC (hoisted branch)
          constexpr bool RS = decltype(realc)::value;
        for (int k0 = 0; k0 < kw4; k0 += 4) {
          double2 bf[NJ], rf[REM > 0 ? REM : 1];
#pragma unroll
          for (int j = 0; j < NJ; ++j) bf[j] = S[(j * 8 + g) * SST + k0 + q];
#pragma unroll
          for (int j = 0; j < REM; ++j) rf[j] = S[(NJ * 8 + j) * SST + k0 + q];
#pragma unroll
          for (int i = 0; i < MT; ++i) {
            const int tt = warp + 8 * i;
            if (tt < ntile && ton[i]) {
              const double2 xv = xs[(k0 + q) * XTP + tb + tt * 8 + g];
              const double ar = zt[i].x * xv.x - zt[i].y * xv.y;
              const double ai = zt[i].x * xv.y + zt[i].y * xv.x;
              const double nai = -ai;
              if constexpr (M3) {
                const double as = ar + ai;
                if constexpr (RS) {
#pragma unroll
                  for (int j = 0; j < NJ; ++j) {
                    dmma(acc[i][j][0][0], acc[i][j][0][1], ar, bf[j].x);
                    dmma(acc[i][j][NA - 1][0], acc[i][j][NA - 1][1], as, bf[j].x);
                  }
                } else {
#pragma unroll
                  for (int j = 0; j < NJ; ++j) {
                    dmma(acc[i][j][0][0], acc[i][j][0][1], ar, bf[j].x);
                    dmma(acc[i][j][1][0], acc[i][j][1][1], ai, bf[j].y);
                    dmma(acc[i][j][NA - 1][0], acc[i][j][NA - 1][1], as, bf[j].x + bf[j].y);
                  }
                }
              } else if constexpr (RS) {  // pivot frequency s_0 is real: Im S = 0, two DMMAs per complex MAC
#pragma unroll
                for (int j = 0; j < NJ; ++j) {
                  dmma(acc[i][j][0][0], acc[i][j][0][1], ar, bf[j].x);
                  dmma(acc[i][j][1][0], acc[i][j][1][1], ai, bf[j].x);
                }
              } else {
                // two passes: dependent DMMAs on one accumulator are 2*NJ instructions apart
#pragma unroll
                for (int j = 0; j < NJ; ++j) {
                  dmma(acc[i][j][0][0], acc[i][j][0][1], ar, bf[j].x);
                  dmma(acc[i][j][1][0], acc[i][j][1][1], ar, bf[j].y);
                }
#pragma unroll
                for (int j = 0; j < NJ; ++j) {
                  dmma(acc[i][j][0][0], acc[i][j][0][1], nai, bf[j].y);
                  dmma(acc[i][j][1][0], acc[i][j][1][1], ai, bf[j].x);
                }
              }
#pragma unroll
              for (int j = 0; j < REM; ++j) {
                racc[i][j].x = fma(ar, rf[j].x, fma(nai, rf[j].y, racc[i][j].x));
                racc[i][j].y = fma(ar, rf[j].y, fma(ai, rf[j].x, racc[i][j].y));
              }
            }
          }
        }
        };
        if (real_slice) gemm(std::true_type{});
        else gemm(std::false_type{});
        if (lown) {
#pragma unroll
          for (int tl = 0; tl < 2; ++tl) {
            if (tl >= tb) break;
            double2 sacc = make_double2(0.0, 0.0);
            for (int nu = lpart; nu < kw; nu += 8) {
              const double2 sv2 = S[lrow * SST + nu], xv = xs[nu * XTP + tl];
              sacc.x = fma(sv2.x, xv.x, sacc.x);
              sacc.x = fma(-sv2.y, xv.y, sacc.x);
              sacc.y = fma(sv2.x, xv.y, sacc.y);
              sacc.y = fma(sv2.y, xv.x, sacc.y);
            }
            const double2 zz = zL[(int64_t)l * zst + tl];
            lacc[tl].x = fma(zz.x, sacc.x, fma(-zz.y, sacc.y, lacc[tl].x));
            lacc[tl].y = fma(zz.x, sacc.y, fma(zz.y, sacc.x, lacc[tl].y));
          }
        }
      }
    }
  }
  double2* out = a.part + (int64_t)sg.w * a.nl * p;
#pragma unroll
  for (int i = 0; i < MT; ++i) {
    const int tt = warp + 8 * i;
    if (tt >= ntile) continue;
    const int t = tc0 + tt * 8 + g;
    if (t >= a.nl) continue;
#pragma unroll
    for (int j = 0; j < NJ; ++j)
#pragma unroll
      for (int v = 0; v < 2; ++v) {
        const int row = j * 8 + 2 * q + v;
        if (row < nrow) {
          BEM_DASSERT((out - a.part) + (int64_t)t * p + mu0 + row < a.part_n);
          if constexpr (M3)
            out[(int64_t)t * p + mu0 + row] = make_double2(acc[i][j][0][v] - acc[i][j][1][v],
                                                           acc[i][j][NA - 1][v] - acc[i][j][0][v] - acc[i][j][1][v]);
          else
            out[(int64_t)t * p + mu0 + row] = make_double2(acc[i][j][0][v], acc[i][j][1][v]);
        }
      }
  }
  if (REM > 0) {
#pragma unroll
    for (int i = 0; i < MT; ++i) {
      const int tt = warp + 8 * i;
      if (tt >= ntile) continue;
      const int t = tc0 + tt * 8 + g;
#pragma unroll
      for (int j = 0; j < (REM > 0 ? REM : 1); ++j) {
        double2 v = racc[i][j];
        v.x += __shfl_xor_sync(0xffffffffu, v.x, 1);
        v.y += __shfl_xor_sync(0xffffffffu, v.y, 1);
        v.x += __shfl_xor_sync(0xffffffffu, v.x, 2);
        v.y += __shfl_xor_sync(0xffffffffu, v.y, 2);
        if (q == 0 && t < a.nl && NJ * 8 + j < nrow) out[(int64_t)t * p + mu0 + NJ * 8 + j] = v;
      }
    }
  }
  if (lead && tb > 0) {
#pragma unroll
    for (int tl = 0; tl < 2; ++tl) {
      if (tl >= tb) break;
      double2 v = lacc[tl];
#pragma unroll
      for (int off = 1; off < 8; off <<= 1) {
        v.x += __shfl_xor_sync(0xffffffffu, v.x, off);
        v.y += __shfl_xor_sync(0xffffffffu, v.y, off);
      }
      if (lpart == 0 && lrow < nrow) out[(int64_t)tl * p + mu0 + lrow] = v;
    }
  }
}

struct Far8Cfg {
  int SST = 0, TT = 0, XTP = 0, tb = 0, nd = 0, ntiles = 0, nchunks = 0, mt = 0, KC = 0;
  size_t smem = 0;
};

// KC: nu chunk width (kc_req > 0 forces it; otherwise the whole p if a
// 128-column frequency tile fits, else 32); TT up to 128 (MT <= 2).
Far8Cfg choose8(int p, int nl, size_t cap, int kc_req) {
  int tb = nl % 8;
  if (tb > 2 || tb == nl) tb = 0;
  const int nD = (nl - tb + 7) / 8 * 8;
  const int p4 = (p + 3) / 4 * 4;
  auto make = [&](int KC, int TTmax) {
    Far8Cfg c;
    int SST = KC;
    while (SST % 8 != 4) ++SST;
    const int ntiles = (nD + TTmax - 1) / TTmax;
    const int TT = ((nD / 8 + ntiles - 1) / ntiles) * 8;
    int XTP = tb + TT;
    while (XTP % 8 != 2) ++XTP;
    const size_t smem =
        sizeof(double2) * (2 * 32 * (size_t)SST + (size_t)KC * XTP + 64) + sizeof(double) * (64 + 96 + 3 * p);
    if (smem > cap) return c;
    c.SST = SST; c.TT = TT; c.XTP = XTP; c.tb = tb; c.nd = nD; c.ntiles = ntiles;
    c.nchunks = (p + 31) / 32; c.mt = (TT / 8 + 7) / 8; c.smem = smem; c.KC = KC;
    return c;
  };
  std::vector<int> kcs;
  if (kc_req > 0) kcs = {std::min(p4, (kc_req + 3) / 4 * 4)};
  else kcs = {p4, std::min(p4, 32)};
  for (int TTmax : {128, 64, 32, 16, 8})
    for (int KC : kcs) {
      Far8Cfg c = make(KC, TTmax);
      if (c.mt > 0 && c.mt <= 2) return c;
    }
  return Far8Cfg{};
}

template <int MT, int NJ, int REM, bool M3 = false, bool DT = false>
cudaError_t launch8(const Far8Cfg& c, int nseg, const Far8Args& a, int ntile, cudaStream_t st) {
  auto k = far8_kernel<MT, NJ, REM, M3, DT>;
  // choose8 sizes the slice buffers for 32 rows; this instantiation uses RW = NJ * 8 + REM
  constexpr int RW = NJ * 8 + REM;
  static_assert(RW <= 32, "far8: at most 32 mu rows per CTA");
  const size_t smem = c.smem - sizeof(double2) * 2 * (32 - RW) * (size_t)c.SST +
                      (DT ? sizeof(double2) * ((size_t)RW * a.p + 1) : 0);
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  Far8Args a2 = a;
  a2.nch = (a.p + NJ * 8 + REM - 1) / (NJ * 8 + REM);  // mu chunks of NJ * 8 + REM rows
  k<<<dim3((unsigned)(nseg * a2.nch), (unsigned)ntile, 1u), 256, smem, st>>>(a2);
  return cudaGetLastError();
}

cudaError_t dispatch8(const Far8Cfg& c, int p, int nseg, const Far8Args& a, int ntile, cudaStream_t st,
                      bool m3 = false, bool dt_on = true) {
  if (m3 && p > 8 && p != 27) {
    // the (r, 1/(4 pi r)) table when two CTAs per SM still fit (p = 64: +16 KB; not p = 125)
    const bool dt = c.smem - sizeof(double2) * 2 * 16 * (size_t)c.SST + sizeof(double2) * (16 * (size_t)p + 1) <=
                        113 * 1024 && dt_on;
    if (dt)
      return c.mt == 1 ? launch8<1, 2, 0, true, true>(c, nseg, a, ntile, st)
                       : launch8<2, 2, 0, true, true>(c, nseg, a, ntile, st);
    return c.mt == 1 ? launch8<1, 2, 0, true>(c, nseg, a, ntile, st) : launch8<2, 2, 0, true>(c, nseg, a, ntile, st);
  }
  if (p <= 8) return c.mt == 1 ? launch8<1, 1, 0>(c, nseg, a, ntile, st) : launch8<2, 1, 0>(c, nseg, a, ntile, st);
  if (p == 27) return c.mt == 1 ? launch8<1, 3, 3>(c, nseg, a, ntile, st) : launch8<2, 3, 3>(c, nseg, a, ntile, st);
  return c.mt == 1 ? launch8<1, 4, 0>(c, nseg, a, ntile, st) : launch8<2, 4, 0>(c, nseg, a, ntile, st);
}

// ------------------------------- h2o: plain-H^2 coupling evaluated on the fly
// BEM_MODE_H2ONLY (the paper's "plain H^2-matrix"
// comparison): no ACA, the coupling matrix of every far block is
// evaluated per frequency from the kernel,
//   yhat_r(l) += S_b(s_l) xhat_c(l),   S_b(s_l)[mu,nu] = k(|xi_{c,nu} - xi_{r,mu}|; s_l),
// with one exp/sincos shared by the conjugate pair (l, L-l):
// S_b(conj s) = conj S_b(s).  CTA = (segment of a row's far blocks, tile of
// FC frequency classes); warp w takes blocks w, w+8, ... of the segment;
// lane owns rows mu = lane + 32 u; per (mu, nu) the distance and 1/(4 pi r)
// are computed once for all FC classes.  Warps' partial yhat are summed in a
// fixed order through shared memory (deterministic, no atomics).
struct H2oArgs {
  int nl, m, p, n_class, FCs;
  const int4* segs;
  const int32_t* far_sorted;
  const int32_t* far_c;
  const double* xi;
  const double2* s;
  const int32_t* local_l;
  const int32_t* class_t1;
  const int32_t* class_t2;
  const double2* xhat;
  double2* part;
  const int32_t* mask;
  // underflow cutoff: a block whose node boxes are r_lb apart is left out for a
  // class tile with min Re s * r_lb > tau (every entry is below e^{-tau} / (4 pi r_lb)); 0: off
  double tau = 0.0;
};

constexpr int kH2oWarps = 4;

template <int U, int FC>
__global__ void __launch_bounds__(kH2oWarps * 32, 3) h2o_kernel(H2oArgs a) {
  extern __shared__ double2 sm[];
  const int p = a.p, m = a.m;
  const int4 sg = a.segs[blockIdx.x];
  const int r = sg.x;
  const int c0 = blockIdx.y * FC;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  double2* sctab = sm;                                  // 64
  double* etab = (double*)(sctab + 64);                 // 64
  double2* xw = (double2*)(etab + 64) + (size_t)warp * 2 * FC * p;  // per warp: [2 FC][p] xhat of its block
  double* cw = (double*)((double2*)(etab + 64) + (size_t)kH2oWarps * 2 * FC * p) + (size_t)warp * 3 * p;  // per warp nodes
  double2* red = (double2*)((double*)((double2*)(etab + 64) + (size_t)kH2oWarps * 2 * FC * p) + (size_t)kH2oWarps * 3 * p);
  for (int i = tid; i < 64; i += blockDim.x) {
    etab[i] = fast::kExp2Tab[i];
    sctab[i] = fast::kSinCosTab[i];
  }
  int t1[FC], t2[FC];
  double sre[FC], sim[FC];
#pragma unroll
  for (int f = 0; f < FC; ++f) {
    const int c = c0 + f;
    t1[f] = c < a.n_class ? a.class_t1[c] : -1;
    t2[f] = c < a.n_class ? a.class_t2[c] : -1;
    if (t1[f] >= 0 && a.mask != nullptr && !a.mask[t1[f]] && (t2[f] < 0 || !a.mask[t2[f]])) t1[f] = t2[f] = -1;
    const double2 sv = t1[f] >= 0 ? a.s[a.local_l[t1[f]]] : make_double2(0.0, 0.0);
    sre[f] = sv.x;
    sim[f] = sv.y;
  }
  double xr[U][3];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const int mu = lane + 32 * u;
    node(a.xi + (int64_t)r * 3 * m, m, mu < p ? mu : 0, xr[u]);
  }
  double2 y1[FC][U], y2[FC][U];
#pragma unroll
  for (int f = 0; f < FC; ++f)
#pragma unroll
    for (int u = 0; u < U; ++u) y1[f][u] = y2[f][u] = make_double2(0.0, 0.0);
  bool any = false;
#pragma unroll
  for (int f = 0; f < FC; ++f) any |= t1[f] >= 0;
  // underflow cutoff: the row cluster's node box (shared memory) and the smallest Re s of the
  // tile's classes
  __shared__ double rbox[6];
  double smin = 1e300;
#pragma unroll
  for (int f = 0; f < FC; ++f)
    if (t1[f] >= 0) smin = fmin(smin, sre[f]);
  if (tid < 3) {
    const double* x = a.xi + (int64_t)r * 3 * m + tid * m;
    double lo = x[0], hi = x[0];
    for (int i = 1; i < m; ++i) { lo = fmin(lo, x[i]); hi = fmax(hi, x[i]); }
    rbox[tid] = lo;
    rbox[3 + tid] = hi;
  }
  __syncthreads();
  for (int bi = sg.y + warp; bi < (any ? sg.z : sg.y); bi += kH2oWarps) {
    const int b = a.far_sorted[bi];
    const int c = a.far_c[b];
    if (a.tau > 0.0 && smin > 0.0) {  // warp-uniform: every lane computes the same distance
      double g2 = 0.0;
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        const double* x = a.xi + (int64_t)c * 3 * m + d * m;
        double lo = x[0], hi = x[0];
        for (int i = 1; i < m; ++i) { lo = fmin(lo, x[i]); hi = fmax(hi, x[i]); }
        const double gp = fmax(0.0, fmax(rbox[d] - hi, lo - rbox[3 + d]));
        g2 = fma(gp, gp, g2);
      }
      if (smin * (sqrt(g2) * (1.0 - 0x1p-40)) > a.tau) continue;
    }
    const double2* xh = a.xhat + (int64_t)c * a.nl * p;
    __syncwarp();
    for (int i = lane; i < p; i += 32) node(a.xi + (int64_t)c * 3 * m, m, i, cw + 3 * i);
    for (int i = lane; i < FC * p; i += 32) {
      const int f = i / p, nu = i - f * p;
      xw[(2 * f) * p + nu] = t1[f] >= 0 ? xh[(int64_t)t1[f] * p + nu] : make_double2(0.0, 0.0);
      xw[(2 * f + 1) * p + nu] = t2[f] >= 0 ? xh[(int64_t)t2[f] * p + nu] : make_double2(0.0, 0.0);
    }
    __syncwarp();
    for (int nu = 0; nu < p; ++nu) {
      const double cx = cw[3 * nu], cy = cw[3 * nu + 1], cz = cw[3 * nu + 2];
      double2 x1[FC], x2[FC];  // U > 1: loaded once for all u; U == 1: at their use (fewer live registers)
      if (U > 1) {
#pragma unroll
        for (int f = 0; f < FC; ++f) {
          x1[f] = xw[(2 * f) * p + nu];
          x2[f] = xw[(2 * f + 1) * p + nu];
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const double dx = cx - xr[u][0], dy = cy - xr[u][1], dz = cz - xr[u][2];
        const double d2 = dx * dx + dy * dy + dz * dz;
        const double ir = rsqrt(d2);
        const double rr = d2 * ir;
        const double w = ir * 0.079577471545947667884;  // 1/(4 pi r)
#pragma unroll
        for (int f = 0; f < FC; ++f) {
          const double e = fast::exp_neg_tab(-sre[f] * rr, etab) * w;
          double sn, cs;
          fast::sincos_tab(sim[f] * rr, sctab, &sn, &cs);
          const double kr = e * cs, ki = -e * sn;  // S(s) = kr + i ki; S(conj s) = kr - i ki
          if (U == 1) {
            x1[f] = xw[(2 * f) * p + nu];
            x2[f] = xw[(2 * f + 1) * p + nu];
          }
          y1[f][u].x = fma(kr, x1[f].x, fma(-ki, x1[f].y, y1[f][u].x));
          y1[f][u].y = fma(kr, x1[f].y, fma(ki, x1[f].x, y1[f][u].y));
          y2[f][u].x = fma(kr, x2[f].x, fma(ki, x2[f].y, y2[f][u].x));
          y2[f][u].y = fma(kr, x2[f].y, fma(-ki, x2[f].x, y2[f][u].y));
        }
      }
    }
  }
  // fixed-order reduction over the warps: red[w][2 FC][U*32]
  const int R = 2 * FC * U * 32;
#pragma unroll
  for (int f = 0; f < FC; ++f)
#pragma unroll
    for (int u = 0; u < U; ++u) {
      red[(size_t)warp * R + ((2 * f) * U + u) * 32 + lane] = y1[f][u];
      red[(size_t)warp * R + ((2 * f + 1) * U + u) * 32 + lane] = y2[f][u];
    }
  __syncthreads();
  double2* out = a.part + (int64_t)sg.w * a.nl * p;
  for (int i = tid; i < R; i += blockDim.x) {
    double2 v = red[i];
    for (int w2 = 1; w2 < kH2oWarps; ++w2) {
      const double2 q2 = red[(size_t)w2 * R + i];
      v.x += q2.x;
      v.y += q2.y;
    }
    const int lane2 = i & 31, rest = i >> 5;
    const int u = rest % U, fh = rest / U;
    const int f = fh >> 1, half = fh & 1;
    const int mu = lane2 + 32 * u;
    const int t = half ? t2[f] : t1[f];
    const int c = c0 + f;
    if (mu < p && c < a.n_class) {
      const int tt = half ? a.class_t2[c] : a.class_t1[c];  // masked classes still write (zeros)
      if (tt >= 0) out[(int64_t)tt * p + mu] = t >= 0 ? v : make_double2(0.0, 0.0);
    }
  }
}

template <int U, int FC>
cudaError_t launch_h2o(const H2oArgs& a, int nseg, int ntile, cudaStream_t st) {
  const size_t smem = sizeof(double2) * 64 + sizeof(double) * 64 + sizeof(double2) * kH2oWarps * 2 * FC * (size_t)a.p +
                      sizeof(double) * kH2oWarps * 3 * (size_t)a.p + sizeof(double2) * kH2oWarps * 2 * FC * U * 32;
  auto k = h2o_kernel<U, FC>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  k<<<dim3((unsigned)nseg, (unsigned)ntile), kH2oWarps * 32, smem, st>>>(a);
  return cudaGetLastError();
}

// yhat[r] = sum over the row's segments (fixed order)
__global__ void seg_reduce_kernel(const int32_t* __restrict__ rows, const int32_t* __restrict__ seg_ptr,
                                  const double2* __restrict__ part, double2* __restrict__ yhat, int64_t tile) {
  const int r = rows[blockIdx.x];
  const int s0 = seg_ptr[blockIdx.x], s1 = seg_ptr[blockIdx.x + 1];
  for (int64_t i = threadIdx.x; i < tile; i += blockDim.x) {
    double2 acc = part[(int64_t)s0 * tile + i];
    for (int sgi = s0 + 1; sgi < s1; ++sgi) {
      const double2 v = part[(int64_t)sgi * tile + i];
      acc.x += v.x;
      acc.y += v.y;
    }
    yhat[(int64_t)r * tile + i] = acc;
  }
}

// ---------------------------------------------------------------- generic
struct FarArgs {
  int nl, m, p, mode, rcap;
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

constexpr int kGenT = 32;

__global__ void __launch_bounds__(256) far_generic_kernel(FarArgs a) {
  extern __shared__ double2 sm[];
  const int p = a.p, m = a.m;
  const int r = blockIdx.x;
  const int t0 = blockIdx.y * kGenT;
  const int nt = min(kGenT, a.nl - t0);
  double* xr = (double*)sm;
  double* xcn = xr + 3 * p;
  double2* acc = (double2*)(xcn + 3 * p);  // p x kGenT
  double2* Bm = acc + p * kGenT;           // p x kGenT
  double2* S = Bm + p * kGenT;             // rb x p
  const int rb = max(1, min(p, 2048 / p));
  for (int i = threadIdx.x; i < p * kGenT; i += blockDim.x) acc[i] = make_double2(0.0, 0.0);
  for (int i = threadIdx.x; i < p; i += blockDim.x) node(a.xi + (int64_t)r * 3 * m, m, i, xr + 3 * i);
  __syncthreads();
  for (int bi = a.far_ptr[r]; bi < a.far_ptr[r + 1]; ++bi) {
    const int b = a.far_sorted[bi];
    const int c = a.far_c[b];
    for (int i = threadIdx.x; i < p; i += blockDim.x) node(a.xi + (int64_t)c * 3 * m, m, i, xcn + 3 * i);
    __syncthreads();
    const double2* xh = a.xhat + ((int64_t)c * a.nl + t0) * p;
    if (a.mode == BEM_MODE_H2ONLY) {
      for (int idx = threadIdx.x; idx < p * nt; idx += blockDim.x) {
        const int t = idx / p, mu = idx % p;
        const double2 sv = a.s[a.local_l[t0 + t]];
        double2 v = acc[mu * kGenT + t];
        for (int nu = 0; nu < p; ++nu) {
          const double dx = xcn[3 * nu] - xr[3 * mu], dy = xcn[3 * nu + 1] - xr[3 * mu + 1],
                       dz = xcn[3 * nu + 2] - xr[3 * mu + 2];
          cmac(v, kern(sqrt(dx * dx + dy * dy + dz * dz), sv), xh[(int64_t)t * p + nu]);
        }
        acc[mu * kGenT + t] = v;
      }
      __syncthreads();
      continue;
    }
    const int rk = a.rank[b];
    const double2* Zb = a.Z + a.zoff[b];
    for (int l = 0; l < rk; ++l) {
      const double2 sv = a.s[a.pivk[(int64_t)b * a.rcap + l]];
      for (int idx = threadIdx.x; idx < p * kGenT; idx += blockDim.x) {
        const int nu = idx / kGenT, t = idx % kGenT;
        double2 v = make_double2(0.0, 0.0);
        if (t < nt) {
          const double2 z = Zb[(int64_t)l * a.nl + t0 + t], xv = xh[(int64_t)t * p + nu];
          v = make_double2(z.x * xv.x - z.y * xv.y, z.x * xv.y + z.y * xv.x);
        }
        Bm[idx] = v;
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
        for (int idx = threadIdx.x; idx < nr * kGenT; idx += blockDim.x) {
          const int mu = mu0 + idx / kGenT, t = idx % kGenT;
          double2 v = acc[mu * kGenT + t];
          const double2* Sr = S + (mu - mu0) * p;
          for (int nu = 0; nu < p; ++nu) cmac(v, Sr[nu], Bm[nu * kGenT + t]);
          acc[mu * kGenT + t] = v;
        }
      }
      __syncthreads();
    }
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < p * nt; idx += blockDim.x) {
    const int t = idx / p, mu = idx % p;
    a.yhat[((int64_t)r * a.nl + t0 + t) * p + mu] = acc[mu * kGenT + t];
  }
}

}  // namespace

// K3 launch geometry of an ACA op: kernel (7/8), CTA grid and Z-tile row width.
struct FarGeom {
  int fk = 0;
  Far7Cfg f7;
  Far8Cfg f8;
  int ntiles = 0, tb = 0, TT = 0, ZW = 0, nd = 0;
};

static FarGeom far_geom(const Op& op) {
  const Tree& t = *op.tree;
  const int p = t.p, nl = op.n_local;
  FarGeom g;
  // default: far10 (INT8 tensor cores) wherever it applies; far8 / far7 (FP64 tensor cores)
  // otherwise -- r01: far8 wins at p = 64, far7 at p = 27
  g.fk = op.far_kernel != 0 ? op.far_kernel : 10;
  if (op.force_generic || op.n_segs == 0) { g.fk = 0; return g; }
  if (g.fk == 10) {
    // far10 (farq.cu): 128-column frequency tiles, <= 2 leftover columns on the FP64 pipe
    // (the per-term tables in shared memory bound the rank capacity)
    int tb = nl % kFar10Tile;
    if (tb > 2 || tb == nl) tb = 0;
    if (p <= 128 && op.rcap <= 512 && nl > tb) {
      g.tb = tb; g.nd = nl - tb; g.TT = kFar10Tile; g.ntiles = (g.nd + kFar10Tile - 1) / kFar10Tile;
      g.ZW = g.tb + g.TT;
      return g;
    }
    g.fk = p > 32 ? 8 : 7;
  }
  if (g.fk == 8) {
    g.f8 = choose8(p, nl, op.far4_smem_cap, op.far8_kc);
    if (g.f8.mt > 0) { g.ntiles = g.f8.ntiles; g.tb = g.f8.tb; g.TT = g.f8.TT; g.ZW = g.tb + g.TT; g.nd = g.f8.nd; return g; }
  } else if (g.fk == 7) {
    g.f7 = choose7(p, nl, op.far4_smem_cap);
    if (g.f7.mt > 0) { g.ntiles = g.f7.ntiles; g.tb = g.f7.tb; g.TT = g.f7.TT; g.ZW = g.tb + g.TT; g.nd = g.f7.nd; return g; }
  }
  g.fk = 0;
  return g;
}

int far_kernel_selected(const Op& op) { return far_geom(op).fk; }

bool far_fuses_near(const Op& op) {
  if (!op.k1_fuse || op.mode != BEM_MODE_H2ACA || op.d_nctr.p == nullptr) return false;
  const int c = op.n_class;  // near_args's class tile must be 4 (the fused warps' F)
  const double w4 = double((c + 3) / 4 * 4 - c) / c, w5 = double((c + 4) / 5 * 5 - c) / c;
  return !(w4 > 0.03 && w5 < w4) && far_geom(op).fk == 10;
}

static Far10SkipArgs far10_skip_args(Op& op, int tb, int nd, int tile_lo, int tile_hi, const ZSrc& z) {
  Tree& t = *op.tree;
  Far10SkipArgs a;
  a.nfar = (int)t.far_r.size(); a.nl = op.n_local; a.m = t.m; a.rcap = op.rcap; a.tb = tb; a.nd = nd;
  a.tile_lo = tile_lo; a.tile_hi = tile_hi; a.delta = op.far_delta;
  a.sref = std::max(1.0, t.hmax > 0.0 ? 0.25 / t.hmax : 1.0);
  a.far_r = t.d_far_r.p; a.far_c = t.d_far_c.p; a.xi = t.d_xi.p; a.s = (const double2*)op.d_s.p;
  a.local_l = op.d_local_l.p; a.rank = op.d_rank.p; a.pivk = op.d_pivk.p; a.z = z; a.skip = op.d_skip.p;
  a.colmap = op.d_colmap.p;
  return a;
}

// executed / total (rank x frequency column) products of the far10 coupling step under the
// underflow mask (bench accounting); without a mask both are the total
void far10_work(Op& op, int64_t* run, int64_t* total) {
  const FarGeom g = far_geom(op);
  int64_t tot = 0, r = 0;
  std::vector<unsigned> h;
  if (g.fk == 10 && op.d_skip.p != nullptr) {
    h.resize(op.d_skip.n);
    if (cudaMemcpy(h.data(), op.d_skip.p, sizeof(unsigned) * h.size(), cudaMemcpyDeviceToHost) != cudaSuccess) h.clear();
  }
  for (size_t b = 0; b < op.ranks.size(); ++b) {
    tot += (int64_t)op.ranks[b] * op.n_local;
    if (h.empty()) { r += (int64_t)op.ranks[b] * op.n_local; continue; }
    for (int tile = 0; tile < g.ntiles; ++tile) {
      if ((h[b] >> tile) & 1u) continue;
      const int tc0 = g.tb + tile * g.TT;
      r += (int64_t)op.ranks[b] * (std::min(g.TT, g.tb + g.nd - tc0) + (tile == 0 ? g.tb : 0));  // nd columns over the tiles
    }
  }
  *run = r; *total = tot;
}

constexpr int kZgenSmem = 64 * 1024;  // zgen_tile_kernel batch buffer (4096 complex)

// Factors-only skeleton: the tile buffer (sum_b r_b x ZW complex) and its per-block
// offsets, allocated at assembly so that an apply never allocates (graph capture).
bem_status far_prepare(Op& op) {
  if (op.ranks.empty()) return BEM_OK;
  op.rmax = *std::max_element(op.ranks.begin(), op.ranks.end());
  const FarGeom g = far_geom(op);
  if (g.fk == 10) {
    BEM_CK(op.d_xmax.alloc((size_t)op.tree->C * op.n_local));
    BEM_CK(op.d_nctr.alloc(1));
    BEM_CK(op.d_f10ctr.alloc(1));
    op.d_skip.release();
    const bool masked = op.far_delta > 0.0 && g.ntiles <= 32 && op.mode == BEM_MODE_H2ACA;
    {
      // tile columns: the local frequencies [tb, nl) by damping (Re s ascending, stable), so that
      // the strongly damped ones share tiles (tile 0, which carries the leftover columns, holds
      // the least damped); the natural order without the mask
      std::vector<int32_t> ord((size_t)g.nd);
      for (int i = 0; i < g.nd; ++i) ord[i] = g.tb + i;
      if (masked) {
        std::vector<double> sh(2 * (size_t)op.L);
        BEM_CK(cudaMemcpy(sh.data(), op.d_s.p, sizeof(double) * sh.size(), cudaMemcpyDeviceToHost));
        std::stable_sort(ord.begin(), ord.end(), [&](int32_t x, int32_t y) {
          return sh[2 * (size_t)op.local_l[x]] < sh[2 * (size_t)op.local_l[y]];
        });
      }
      op.colmap.assign((size_t)g.ntiles * kFar10Tile, -1);
      for (int i = 0; i < g.nd; ++i) op.colmap[i] = ord[i];
      BEM_CK(op.d_colmap.upload(op.colmap));
    }
    if (masked) {
      BEM_CK(op.d_skip.alloc(op.ranks.size()));
      BEM_CK(cudaMemset(op.d_skip.p, 0, sizeof(unsigned) * op.ranks.size()));
      if (op.z_stored) {  // the mask depends on the skeleton only: one pass over every tile
        BEM_CK(cudaDeviceSynchronize());
        ZSrc z{};
        z.zoff = op.d_zoff.p; z.Z = (const double2*)op.d_Z.p; z.tiled = 0; z.ZW = g.ZW; z.zn = (int64_t)op.d_Z.n / 2;
        BEM_CK(launch_far10_skip(far10_skip_args(op, g.tb, g.nd, 0, g.ntiles, z), nullptr));
        BEM_CK(cudaDeviceSynchronize());
      }
    }
  }
  if (op.z_stored) return BEM_OK;
  if (g.fk == 0) {
    set_error("bem_assemble_h2_aca: factors-only skeleton needs the tiled coupling kernels (p <= 128)");
    return BEM_EINVAL;
  }
  std::vector<int64_t> off(op.ranks.size());
  int64_t acc = 0;
  for (size_t b = 0; b < off.size(); ++b) { off[b] = acc; acc += (int64_t)op.ranks[b] * g.ZW; }
  op.rmax = *std::max_element(op.ranks.begin(), op.ranks.end());
  BEM_CK(op.d_ztoff.upload(off));
  BEM_CK(op.d_zs.alloc((size_t)std::max<int64_t>(acc, 1) * 2));
  BEM_CK(cudaFuncSetAttribute(zgen_tile_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kZgenSmem));
  return BEM_OK;
}

bem_status launch_far(Op& op, const double2* xhat, double2* yhat, cudaStream_t st, const NearArgs* fna) {
  Tree& t = *op.tree;
  const int nl = op.n_local, p = t.p;
  const bool aca = op.mode == BEM_MODE_H2ACA || op.mode == BEM_MODE_COMBINED;  // far blocks via the MACA skeleton
  if (op.mode == BEM_MODE_H2ONLY && !op.force_generic && op.n_segs > 0 && p <= 128) {
    BEM_CK(cudaMemsetAsync(yhat, 0, sizeof(double2) * (size_t)t.C * nl * p, st));
    H2oArgs a;
    a.nl = nl; a.m = t.m; a.p = p; a.n_class = op.n_class;
    a.segs = (const int4*)op.d_segs.p; a.far_sorted = t.d_far_sorted.p; a.far_c = t.d_far_c.p;
    a.xi = t.d_xi.p; a.s = (const double2*)op.d_s.p; a.local_l = op.d_local_l.p;
    a.class_t1 = op.d_class_t1.p; a.class_t2 = op.d_class_t2.p; a.xhat = xhat; a.part = (double2*)op.d_part.p;
    a.mask = op.d_mask;
    a.tau = op.near_tau > 0.0 ? op.near_tau + 8.0 : 0.0;  // far blocks: e^{-50} of 1 / (4 pi r_lb)
    const int U = (p + 31) / 32;
    int FC = p <= 32 ? 6 : 2;  // r01 sweep: p = 27 FC 2/4/6 = 2.45/2.48/2.39 ms; p = 64 FC 2/3/4 = 356/369/383 ms
    if (op.h2o_fc > 0) FC = op.h2o_fc;
    a.FCs = FC;
    const int ntile = (op.n_class + FC - 1) / FC;
    cudaError_t e;
    if (U == 1) e = FC == 2 ? launch_h2o<1, 2>(a, op.n_segs, ntile, st) : FC == 6 ? launch_h2o<1, 6>(a, op.n_segs, ntile, st)
                                                                              : launch_h2o<1, 4>(a, op.n_segs, ntile, st);
    else if (U == 2) e = FC == 3 ? launch_h2o<2, 3>(a, op.n_segs, ntile, st) : FC == 4 ? launch_h2o<2, 4>(a, op.n_segs, ntile, st)
                                                                                 : launch_h2o<2, 2>(a, op.n_segs, ntile, st);
    else if (U == 3) e = launch_h2o<3, 2>(a, op.n_segs, ntile, st);
    else e = launch_h2o<4, 2>(a, op.n_segs, ntile, st);
    BEM_CK(e);
    seg_reduce_kernel<<<op.n_seg_rows, 256, 0, st>>>(op.d_seg_rows.p, op.d_seg_ptr.p, (const double2*)op.d_part.p,
                                                     yhat, (int64_t)nl * p);
    BEM_CK(cudaGetLastError());
    return BEM_OK;
  }
  const FarGeom g = aca ? far_geom(op) : FarGeom{};
  const bool fac = aca && !op.z_stored;
  if (fac && (g.fk == 0 || op.d_zs.p == nullptr)) {
    set_error("launch_far: factors-only skeleton without its tile buffer");
    return BEM_ESTATE;
  }
  if (aca && g.fk != 0) {
    BEM_CK(cudaMemsetAsync(yhat, 0, sizeof(double2) * (size_t)t.C * nl * p, st));
    ZSrc z{};
    z.zoff = fac ? op.d_ztoff.p : op.d_zoff.p;
    z.Z = fac ? (const double2*)op.d_zs.p : (const double2*)op.d_Z.p;
    z.tiled = fac ? 1 : 0;
    z.ZW = g.ZW;
    z.zn = (int64_t)(fac ? op.d_zs.n : op.d_Z.n) / 2;
    zgen::Src zsrc{};
    zsrc.m = t.m; zsrc.p = p; zsrc.L = op.L; zsrc.far_r = t.d_far_r.p; zsrc.far_c = t.d_far_c.p; zsrc.xi = t.d_xi.p;
    zsrc.s = (const double2*)op.d_s.p; zsrc.pivk = op.d_pivk.p; zsrc.pivq = op.d_pivq.p; zsrc.foff = op.d_foff.p;
    zsrc.F = (const double2*)op.d_F.p; zsrc.rcap = op.rcap;
    const int nfar = (int)t.far_r.size();
    // stored Z: all tiles in one launch; factors-only: per tile, regenerate its Z columns first
    for (int tile = 0; tile < (fac ? g.ntiles : 1); ++tile) {
      const int ntile = fac ? 1 : g.ntiles;
      if (fac) {
        const int tc0 = g.tb + tile * g.TT;
        const int nd = g.nd;
        const int ncol = std::min(g.TT, g.tb + nd - tc0);
        zgen_tile_kernel<<<std::min(nfar, 148 * 8), 256, kZgenSmem, st>>>(
            zsrc, nfar, op.d_rank.p, op.d_ztoff.p, op.d_local_l.p, op.d_mask, nl, g.tb, tc0, ncol, tile == 0 ? 1 : 0,
            g.ZW, kZgenSmem / (int)sizeof(double2), (double2*)op.d_zs.p, (int64_t)op.d_zs.n / 2,
            g.fk == 10 ? op.d_colmap.p + (size_t)tile * kFar10Tile : nullptr);
        BEM_CK(cudaGetLastError());
        if (g.fk == 10 && op.d_skip.p != nullptr) BEM_CK(launch_far10_skip(far10_skip_args(op, g.tb, g.nd, tile, tile + 1, z), st));
      }
      if (g.fk == 10) {
        if (tile == 0) BEM_CK(launch_xmax(xhat, (int64_t)t.C * nl, p, op.d_xmax.p, st));
        Far10Args a;
        a.nl = nl; a.m = t.m; a.p = p; a.rcap = op.rcap; a.tb = g.tb; a.nd = g.nd; a.tile0 = fac ? tile : 0;
        a.nch = (p + 31) / 32;
        // level l sums <= 5 u8 x s8 + 1 s8 x s8 slice products per k byte: <= 179584 per k,
        // K = 32 bytes per nu chunk and term
        a.gmax = std::max(1, (int)(2147483647LL / (179584LL * 32 * ((p + 15) / 16))));
        if (const char* ge = getenv("BEM_FAR10_GMAX"))  // tests: force term groups
          if (atoi(ge) > 0) a.gmax = std::min(a.gmax, atoi(ge));
        a.segs = (const int4*)op.d_segs.p; a.far_sorted = t.d_far_sorted.p; a.far_c = t.d_far_c.p;
        a.xi = t.d_xi.p; a.s = (const double2*)op.d_s.p; a.rank = op.d_rank.p; a.pivk = op.d_pivk.p;
        a.z = z; a.xhat = xhat; a.xmax = op.d_xmax.p; a.part = (double2*)op.d_part.p; a.mask = op.d_mask;
        a.part_n = (int64_t)op.d_part.n / 2;
        a.skip = op.d_skip.p;
        a.colmap = op.d_colmap.p;
        a.nfar = (int)op.d_skip.n; a.ncm = (int)op.d_colmap.n;
        if (fna != nullptr) {
          if (tile == 0) BEM_CK(cudaMemsetAsync(op.d_nctr.p, 0, sizeof(unsigned), st));
          a.na = *fna;
          a.nctr = op.d_nctr.p;
          a.n_items = (unsigned)(fna->M * (int64_t)((fna->n_class + 3) / 4));
        }
        a.ctr = op.far10_persist ? op.d_f10ctr.p : nullptr;
        BEM_CK(launch_far10(a, op.n_segs, ntile, st, fna != nullptr ? op.k1_warps : 0));
      } else if (g.fk == 8) {
        const Far8Cfg& f8 = g.f8;
        Far8Args a;
        a.nl = nl; a.m = t.m; a.p = p; a.rcap = op.rcap; a.SST = f8.SST; a.TT = f8.TT; a.XTP = f8.XTP;
        a.tb = f8.tb; a.nd = f8.nd; a.KC = f8.KC; a.tile0 = fac ? tile : 0;
        a.segs = (const int4*)op.d_segs.p; a.far_sorted = t.d_far_sorted.p; a.far_c = t.d_far_c.p;
        a.xi = t.d_xi.p; a.s = (const double2*)op.d_s.p; a.rank = op.d_rank.p; a.pivk = op.d_pivk.p;
        a.z = z; a.xhat = xhat; a.part = (double2*)op.d_part.p; a.mask = op.d_mask;
        a.part_n = (int64_t)op.d_part.n / 2;
        BEM_CK(dispatch8(f8, p, op.n_segs, a, ntile, st, op.far8_m3, op.far8_dt));
      } else {
        const Far7Cfg& f7 = g.f7;
        Far7Args a;
        a.nl = nl; a.m = t.m; a.p = p; a.p4 = f7.p4; a.rcap = op.rcap; a.SST = f7.SST; a.TT = f7.TT;
        a.XTP = f7.XTP; a.tb = f7.tb; a.nd = f7.nd; a.tile0 = fac ? tile : 0;
        a.segs = (const int4*)op.d_segs.p; a.far_sorted = t.d_far_sorted.p; a.far_c = t.d_far_c.p;
        a.xi = t.d_xi.p; a.s = (const double2*)op.d_s.p; a.rank = op.d_rank.p; a.pivk = op.d_pivk.p;
        a.z = z; a.xhat = xhat; a.part = (double2*)op.d_part.p; a.mask = op.d_mask;
        a.part_n = (int64_t)op.d_part.n / 2;
        BEM_CK(dispatch7(f7, p, op.n_segs, a, ntile, st));
      }
    }
    seg_reduce_kernel<<<op.n_seg_rows, 256, 0, st>>>(op.d_seg_rows.p, op.d_seg_ptr.p, (const double2*)op.d_part.p,
                                                     yhat, (int64_t)nl * p);
    BEM_CK(cudaGetLastError());
    if (fna != nullptr) {
      if (g.fk != 10) {
        set_error("launch_far: K1 fusion needs far10");
        return BEM_ESTATE;
      }
      bem_status rs = launch_near_tail(*fna, 4, op.d_nctr.p, st);  // the K1 items the fused warps left
      if (rs != BEM_OK) return rs;
    }
    return BEM_OK;
  }
  if (fac) {
    set_error("launch_far: factors-only skeleton needs far7/far8");
    return BEM_ESTATE;
  }
  FarArgs a;
  a.nl = nl; a.m = t.m; a.p = p; a.mode = aca ? BEM_MODE_H2ACA : op.mode; a.rcap = op.rcap;
  a.far_ptr = t.d_far_ptr.p; a.far_sorted = t.d_far_sorted.p; a.far_c = t.d_far_c.p; a.xi = t.d_xi.p;
  a.s = (const double2*)op.d_s.p; a.local_l = op.d_local_l.p; a.rank = op.d_rank.p; a.pivk = op.d_pivk.p;
  a.zoff = op.d_zoff.p; a.Z = (const double2*)op.d_Z.p; a.xhat = xhat; a.yhat = yhat;
  const int rb = std::max(1, std::min(p, 2048 / p));
  const size_t smem = sizeof(double) * 6 * p + sizeof(double2) * (2 * (size_t)p * kGenT + (size_t)rb * p);
  BEM_CK(cudaFuncSetAttribute(far_generic_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  far_generic_kernel<<<dim3((unsigned)t.C, (unsigned)((nl + kGenT - 1) / kGenT)), 256, smem, st>>>(a);
  BEM_CK(cudaGetLastError());
  return BEM_OK;
}

}  // namespace bem
