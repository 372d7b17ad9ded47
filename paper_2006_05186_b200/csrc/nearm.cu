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
// One CTA owns (row leaf, nw*8-column frequency tile, 32-row chunk) and walks all
// near blocks of its row leaf, so the output is written once (no partial sums,
// deterministic).  The last frequency tile is zero-padded to 8 columns.
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
  int nl, nw, XTP, SST, p4max;  // nw warps per CTA = 8-column frequency tiles per CTA
  const int32_t* leaves;
  const int32_t* order;  // leaf indices, descending sum_b r_b n_c (LPT)
  int* counter;          // work-item counter (zeroed before each launch)
  int nitems, ntiles, nchunks;
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

// Columns past n_local (the last tile's padding, e.g. 129 -> 144) carry zero Z and x:
// a zero-padded DMMA column is cheaper than a DFMA side path (r01: far7 / K1m v1).
// Slices are triple-buffered (one barrier per term: the barrier that publishes
// term j also retires term j-1's buffer, which term j+2's cp.async then refills);
// the real and imaginary partial products go to separate accumulators so that
// dependent DMMAs are 2 * njt instructions apart in each pass (r01 ncu: v2 was
// "stall wait" bound at 6 apart).
constexpr int kNmMaxWarps = 6;

__device__ __forceinline__ void nearm_item(const NearmArgs& a, int item) {
  extern __shared__ double2 sm[];
  const int SST = a.SST, XTP = a.XTP, nth = blockDim.x;
  const int tile = item % a.ntiles, rest = item / a.ntiles;
  const int chunk = rest % a.nchunks;
  const int li = a.order[rest / a.nchunks];
  const int r = a.leaves[li];
  const int rb0 = a.cbegin[r], nr = a.cend[r] - rb0;
  const int mu0 = chunk * 32;
  const int nrow = min(32, nr - mu0);
  if (nrow <= 0) return;
  const int ncp = a.nw * 8;                    // staged columns of this CTA
  const int tc0 = tile * ncp;
  double2* Sb[3] = {sm, sm + 32 * SST, sm + 64 * SST};
  double2* xs = sm + 96 * SST;  // p4max x XTP: [nu][column]
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, q = lane & 3;
  const int tcol = tc0 + warp * 8 + g;         // this lane's A-fragment column
  const bool live = tcol < a.nl;
  const bool wlive = tc0 + warp * 8 < a.nl;    // the warp's tile holds a real column
  const int njt = (nrow + 7) / 8;
  double acc[4][2][2], bcc[4][2][2];
#pragma unroll
  for (int j = 0; j < 4; ++j)
#pragma unroll
    for (int u = 0; u < 2; ++u) acc[j][u][0] = acc[j][u][1] = bcc[j][u][0] = bcc[j][u][1] = 0.0;
  for (int bi = a.nb_ptr[li]; bi < a.nb_ptr[li + 1]; ++bi) {
    const int b = a.nb_sorted[bi];
    const int c = a.near_c[b];
    const int cb0 = a.cbegin[c], nc = a.cend[c] - cb0;
    const int p4 = (nc + 3) & ~3;
    const int rk = a.rank[b];
    const double2* Sg = a.S + a.soff[b] + (int64_t)mu0 * nc;
    const double2* Zb = a.Z + a.zoff[b];
    const int64_t slice = (int64_t)nr * nc;
    __syncthreads();  // previous block's xs / S reads are done
    // stage xc[t, c0 + nu] (zero for nu in [nc, p4) and t >= n_local), zero the padded S columns
    for (int idx = tid; idx < ncp * p4; idx += nth) {
      const int tl = idx / p4, nu = idx - tl * p4;
      const int tg = tc0 + tl;
      xs[nu * XTP + tl] = (nu < nc && tg < a.nl) ? a.xc[(int64_t)tg * a.M + cb0 + nu] : make_double2(0.0, 0.0);
    }
    for (int idx = tid; idx < 3 * 32 * (p4 - nc); idx += nth) {
      const int w = idx / (32 * (p4 - nc)), e = idx - w * 32 * (p4 - nc);
      const int i = e / (p4 - nc), nu = nc + (e - i * (p4 - nc));
      Sb[w][i * SST + nu] = make_double2(0.0, 0.0);
    }
    auto load = [&](int j) {
      if (j < rk) {
        const double2* src = Sg + (int64_t)j * slice;
        double2* dst = Sb[j % 3];
        for (int idx = tid; idx < nrow * nc; idx += nth) {
          const int i = idx / nc, nu = idx - i * nc;
          cp_async16(dst + i * SST + nu, src + idx);
        }
      }
      cp_commit();  // empty groups keep the wait_group count uniform
    };
    load(0);
    load(1);
    for (int j = 0; j < rk; ++j) {
      const double2 zt = live ? Zb[(int64_t)j * a.nl + tcol] : make_double2(0.0, 0.0);
      cp_wait<1>();      // this thread's copies of term j have landed
      __syncthreads();   // ... everyone's; and term j-1's buffer is free
      load(j + 2);
      const double2* S = Sb[j % 3];
      for (int k0 = 0; k0 < (wlive ? p4 : 0); k0 += 4) {
        const double2 xv = xs[(k0 + q) * XTP + warp * 8 + g];
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
            dmma(bcc[jt][0][0], bcc[jt][0][1], nai, bf[jt].y);
            dmma(bcc[jt][1][0], bcc[jt][1][1], ai, bf[jt].x);
          }
      }
    }
    cp_wait<0>();
  }
  // accumulator element (row 2q+v of tile jt, column g of the warp's tile)
  const int t = tc0 + warp * 8 + g;
  if (t < a.nl) {
    const bool on = a.mask == nullptr || a.mask[t] != 0;
#pragma unroll
    for (int jt = 0; jt < 4; ++jt)
#pragma unroll
      for (int v = 0; v < 2; ++v) {
        const int row = jt * 8 + 2 * q + v;
        if (row < nrow)
          a.yc[(int64_t)t * a.M + rb0 + mu0 + row] =
              on ? make_double2(acc[jt][0][v] + bcc[jt][0][v], acc[jt][1][v] + bcc[jt][1][v])
                 : make_double2(0.0, 0.0);
      }
  }
}

// Persistent CTAs take work items (row leaf, 32-row chunk, column tile) from a
// counter in LPT order (leaves by descending sum_b r_b n_c): every item's output
// is written by exactly one CTA, so the result does not depend on the schedule.
__global__ void __launch_bounds__(kNmMaxWarps * 32, 2) nearm_kernel(NearmArgs a) {
  __shared__ int s_item;
  for (;;) {
    __syncthreads();
    if (threadIdx.x == 0) s_item = atomicAdd(a.counter, 1);
    __syncthreads();
    const int item = s_item;
    if (item >= a.nitems) return;
    nearm_item(a, item);
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
  // 8-column tiles; CTAs of nw in [4, 8] warps, nw chosen to minimise padded tiles
  // (129 frequencies: 17 tiles -> 3 x 6; 257: 33 -> 7 x 5 ... ties: more warps)
  const int ntl = (nl + 7) / 8;
  int nw = kNmMaxWarps, best = 1 << 30;
  for (int w = kNmMaxWarps; w >= 4; --w) {
    const int waste = ((ntl + w - 1) / w) * w - ntl;
    if (waste < best) { best = waste; nw = w; }
  }
  if (ntl < 4) nw = ntl;
  const int ntiles = (ntl + nw - 1) / nw;
  a.nw = nw;
  a.p4max = (t.max_leaf + 3) & ~3;
  int SST = a.p4max;
  while (SST % 8 != 4) ++SST;  // B fragment rows 8 apart: stride 4 (mod 8) complex -> conflict-free
  a.SST = SST;
  int XTP = nw * 8;
  while (XTP % 8 != 2) ++XTP;
  a.XTP = XTP;
  a.order = op.d_nm_order.p;
  a.leaves = t.d_leaves.p; a.nb_ptr = t.d_nb_ptr.p; a.nb_sorted = t.d_nb_sorted.p; a.near_c = t.d_near_c.p;
  a.cbegin = t.d_begin.p; a.cend = t.d_end.p;
  a.rank = op.d_nrank.p; a.soff = op.d_nsoff.p; a.zoff = op.d_nzoff.p;
  a.S = (const double2*)op.d_nS.p; a.Z = (const double2*)op.d_nZ.p; a.xc = xc; a.yc = yc; a.mask = op.d_mask;
  const size_t smem = sizeof(double2) * (96 * (size_t)SST + (size_t)a.p4max * XTP);
  BEM_CK(cudaFuncSetAttribute(nearm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  a.nchunks = (t.max_leaf + 31) / 32;
  a.ntiles = ntiles;
  a.nitems = t.n_leaves * a.nchunks * ntiles;
  if (op.d_nm_counter.n == 0) BEM_CK(op.d_nm_counter.alloc(1));
  a.counter = op.d_nm_counter.p;
  BEM_CK(cudaMemsetAsync(a.counter, 0, sizeof(int), st));
  int nsm = 148, per_sm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, t.device);
  BEM_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, nearm_kernel, nw * 32, smem));
  const int grid = std::max(1, std::min(a.nitems, nsm * std::max(1, per_sm)));
  nearm_kernel<<<grid, nw * 32, smem, st>>>(a);
  BEM_CK(cudaGetLastError());
  return BEM_OK;
}

}  // namespace bem
