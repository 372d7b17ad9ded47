// K1m: near field of the combined mode (BEM_MODE_COMBINED).
//
// Alg. 3 compresses the near blocks b in P- across frequency too:
//   V_l[b] ~= sum_{t < r_b} Z_b[t,l] V_{k_t}[b]      (eq:lrfinal P:1404-1410, eq:maca),
// with the pivot slices V_{k_t}[b] (n_r x n_c complex, the tensor C_b) stored by the
// near-field ACA (aca.cu).  The near-field product is then a dense contraction,
//   yc[t, i] = sum_b sum_j sum_nu V_{k_j}[b][i,nu] (Z_b[j,t] xc[t, c0 + nu]),
// run on the FP64 tensor cores (mma.sync m8n8k4 f64) like K3's far6 product:
//   A[t,nu] = Z_b[j,t] xc[t, c0+nu]  formed in registers (one complex multiply
//             per fragment, reused for the four 8-row tiles),
//   B[nu,i] = V_{k_j}[b][i,nu]       slice rows staged in shared memory with
//             cp.async, double-buffered so term j+1 loads while term j multiplies.
// One CTA owns (row leaf, 8*8-column frequency tile, 32-row chunk) and walks all
// near blocks of its row leaf, so the output is written once (no partial sums,
// deterministic).  Leftover columns (n_local mod 8) use DFMA on lanes 0..3.
#include <algorithm>

#include "common.cuh"

namespace bem {
namespace {

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

struct NearmArgs {
  int64_t M;
  int nl, tb, TT, XTP, SST, p4max;
  const int32_t* leaves;
  const int32_t* nb_ptr;
  const int32_t* nb_sorted;
  const int32_t* near_c;
  const int32_t* cbegin;
  const int32_t* cend;
  const int32_t* rank;
  const int64_t* soff;
  const int64_t* zoff;
  const double2* S;
  const double2* Z;
  const double2* xc;
  double2* yc;
  const int32_t* mask;
};

constexpr int kNmThreads = 256;

__global__ void __launch_bounds__(kNmThreads, 2) nearm_kernel(NearmArgs a) {
  extern __shared__ double2 sm[];
  const int SST = a.SST, XTP = a.XTP, tb = a.tb;
  const int r = a.leaves[blockIdx.x];
  const int rb0 = a.cbegin[r], nr = a.cend[r] - rb0;
  const int mu0 = blockIdx.z * 32;
  const int nrow = min(32, nr - mu0);
  if (nrow <= 0) return;
  const int tc0 = tb + blockIdx.y * a.TT;
  const int ncol = max(0, min(a.TT, a.nl - tc0));
  const bool lead = blockIdx.y == 0;
  double2* Sb[2] = {sm, sm + 32 * SST};
  double2* xs = sm + 64 * SST;  // p4max x XTP: [nu][0..tb) leftover, [tb..) DMMA columns
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, q = lane & 3;
  const int ntile = ncol / 8;
  const bool wt = warp < ntile;  // this warp's 8-column tile exists
  const int njt = (nrow + 7) / 8;
  double acc[4][2][2];
#pragma unroll
  for (int j = 0; j < 4; ++j) acc[j][0][0] = acc[j][0][1] = acc[j][1][0] = acc[j][1][1] = 0.0;
  double2 lacc[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) lacc[i] = make_double2(0.0, 0.0);
  const int lrow = 4 * warp + lane;
  const bool lown = lead && lane < 4 && lrow < nrow && tb > 0;
  const int ncp = tb + ncol;
  for (int bi = a.nb_ptr[blockIdx.x]; bi < a.nb_ptr[blockIdx.x + 1]; ++bi) {
    const int b = a.nb_sorted[bi];
    const int c = a.near_c[b];
    const int cb0 = a.cbegin[c], nc = a.cend[c] - cb0;
    const int p4 = (nc + 3) & ~3;
    const int rk = a.rank[b];
    const double2* Sg = a.S + a.soff[b] + (int64_t)mu0 * nc;
    const double2* Zb = a.Z + a.zoff[b];
    const int64_t slice = (int64_t)nr * nc;
    __syncthreads();  // previous block's xs / S reads are done
    // stage xc[t, c0 + nu] (zero rows nu in [nc, p4)) and zero the padded S columns
    for (int idx = tid; idx < ncp * p4; idx += kNmThreads) {
      const int tl = idx / p4, nu = idx - tl * p4;
      const int tg = tl < tb ? tl : tc0 + (tl - tb);
      if (tl >= tb || lead)
        xs[nu * XTP + tl] = nu < nc ? a.xc[(int64_t)tg * a.M + cb0 + nu] : make_double2(0.0, 0.0);
    }
    for (int idx = tid; idx < 2 * 32 * (p4 - nc); idx += kNmThreads) {
      const int w = idx / (32 * (p4 - nc)), e = idx - w * 32 * (p4 - nc);
      const int i = e / (p4 - nc), nu = nc + (e - i * (p4 - nc));
      Sb[w][i * SST + nu] = make_double2(0.0, 0.0);
    }
    auto load = [&](int j, double2* dst) {
      const double2* src = Sg + (int64_t)j * slice;
      for (int idx = tid; idx < nrow * nc; idx += kNmThreads) {
        const int i = idx / nc, nu = idx - i * nc;
        cp_async16(dst + i * SST + nu, src + idx);
      }
      cp_commit();
    };
    if (rk > 0) load(0, Sb[0]);
    for (int j = 0; j < rk; ++j) {
      const double2 zt = wt ? Zb[(int64_t)j * a.nl + tc0 + warp * 8 + g] : make_double2(0.0, 0.0);
      if (j + 1 < rk) {
        load(j + 1, Sb[(j + 1) & 1]);
        cp_wait<1>();
      } else {
        cp_wait<0>();
      }
      __syncthreads();
      const double2* S = Sb[j & 1];
      if (wt) {
        for (int k0 = 0; k0 < p4; k0 += 4) {
          const double2 xv = xs[(k0 + q) * XTP + tb + warp * 8 + g];
          const double ar = zt.x * xv.x - zt.y * xv.y;
          const double ai = zt.x * xv.y + zt.y * xv.x;
          const double nai = -ai;
          double2 bf[4];
#pragma unroll
          for (int jt = 0; jt < 4; ++jt) bf[jt] = S[(jt * 8 + g) * SST + k0 + q];
#pragma unroll
          for (int jt = 0; jt < 4; ++jt)
            if (jt < njt) {
              dmma(acc[jt][0][0], acc[jt][0][1], ar, bf[jt].x);
              dmma(acc[jt][1][0], acc[jt][1][1], ar, bf[jt].y);
            }
#pragma unroll
          for (int jt = 0; jt < 4; ++jt)
            if (jt < njt) {
              dmma(acc[jt][0][0], acc[jt][0][1], nai, bf[jt].y);
              dmma(acc[jt][1][0], acc[jt][1][1], ai, bf[jt].x);
            }
        }
      }
      if (lown) {
        for (int tl = 0; tl < tb; ++tl) {
          const double2 z = Zb[(int64_t)j * a.nl + tl];
          double2 sacc = make_double2(0.0, 0.0);
          for (int nu = 0; nu < nc; ++nu) {
            const double2 sv = S[lrow * SST + nu], xv = xs[nu * XTP + tl];
            sacc.x += sv.x * xv.x - sv.y * xv.y;
            sacc.y += sv.x * xv.y + sv.y * xv.x;
          }
          lacc[tl].x += z.x * sacc.x - z.y * sacc.y;
          lacc[tl].y += z.x * sacc.y + z.y * sacc.x;
        }
      }
      __syncthreads();  // buffer j&1 is refilled by the load of term j+2
    }
  }
  if (wt) {
    const int t = tc0 + warp * 8 + g;
    const bool on = a.mask == nullptr || a.mask[t] != 0;
#pragma unroll
    for (int jt = 0; jt < 4; ++jt)
#pragma unroll
      for (int v = 0; v < 2; ++v) {
        const int row = jt * 8 + 2 * q + v;
        if (row < nrow)
          a.yc[(int64_t)t * a.M + rb0 + mu0 + row] =
              on ? make_double2(acc[jt][0][v], acc[jt][1][v]) : make_double2(0.0, 0.0);
      }
  }
  if (lown)
    for (int tl = 0; tl < tb; ++tl) {
      const bool on = a.mask == nullptr || a.mask[tl] != 0;
      a.yc[(int64_t)tl * a.M + rb0 + mu0 + lrow] = on ? lacc[tl] : make_double2(0.0, 0.0);
    }
}

}  // namespace

bem_status launch_near_maca(Op& op, const double2* xc, double2* yc, cudaStream_t st) {
  Tree& t = *op.tree;
  const int nl = op.n_local;
  if (t.near_r.empty()) {
    BEM_CK(cudaMemsetAsync(yc, 0, sizeof(double2) * (size_t)nl * t.M, st));
    return BEM_OK;
  }
  NearmArgs a;
  a.M = t.M; a.nl = nl;
  a.tb = nl % 8;
  const int nD = nl - a.tb;
  const int ntiles = std::max(1, (nD + 63) / 64);
  a.TT = nD == 0 ? 0 : ((nD / 8 + ntiles - 1) / ntiles) * 8;
  a.p4max = (t.max_leaf + 3) & ~3;
  int SST = a.p4max;
  while (SST % 8 != 4) ++SST;  // B fragment rows 8 apart: stride 4 (mod 8) complex -> conflict-free
  a.SST = SST;
  int XTP = a.tb + a.TT;
  while (XTP % 8 != 2) ++XTP;
  a.XTP = XTP;
  a.leaves = t.d_leaves.p; a.nb_ptr = t.d_nb_ptr.p; a.nb_sorted = t.d_nb_sorted.p; a.near_c = t.d_near_c.p;
  a.cbegin = t.d_begin.p; a.cend = t.d_end.p;
  a.rank = op.d_nrank.p; a.soff = op.d_nsoff.p; a.zoff = op.d_nzoff.p;
  a.S = (const double2*)op.d_nS.p; a.Z = (const double2*)op.d_nZ.p; a.xc = xc; a.yc = yc; a.mask = op.d_mask;
  const size_t smem = sizeof(double2) * (64 * (size_t)SST + (size_t)a.p4max * XTP);
  BEM_CK(cudaFuncSetAttribute(nearm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const unsigned nchunks = (unsigned)((t.max_leaf + 31) / 32);
  nearm_kernel<<<dim3((unsigned)t.n_leaves, (unsigned)ntiles, nchunks), kNmThreads, smem, st>>>(a);
  BEM_CK(cudaGetLastError());
  return BEM_OK;
}

}  // namespace bem
