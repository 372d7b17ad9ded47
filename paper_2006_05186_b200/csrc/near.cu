// K1: near field evaluated on the fly.
//
// For every target panel i (cluster order) and every source panel j in the
// near-field leaves of i's leaf (inadmissible leaf x leaf blocks, eq:qadm
// P:905-912), the collocation entry of the single layer V(s) (P:537-540,
// kernel eq:fundsol P:479-482) with the 7-point rule is
//   V[i,j](s) = sum_q (w_q |T_j| / 4 pi) e^{-s r_q} / r_q,  r_q = |c_i - y_{j,q}|,
// and for the self panel (analytic 1/r integral + rule on (e^{-sr}-1)/r)
//   V[i,i](s) = J(T_i)/4pi + sum_q (w_q |T_i|/4pi) phi(s, r_q),  phi(s,0) = -s.
// y_l[i] = sum_j V[i,j](s_l) x_l[j] for all local frequencies; a conjugate
// pair (l, L-l) shares one exp/sincos: V(conj s) = conj V(s).
//
// Mapping: one warp per (target, tile of F frequency classes); lanes stride
// over the source panels (coalesced loads of panel geometry and x); the node
// loop is kept rolled so the code body stays small (I-cache), F classes are
// unrolled for ILP; warp butterfly reduction, no atomics.
#include <cstdlib>

#include "near_common.cuh"

namespace bem {
namespace {

constexpr int kNearWarps = 4;

template <int F, bool DL, bool CUT>
__device__ __forceinline__ void near_body(const NearArgs& a) {
  __shared__ double etab[64];
  __shared__ double2 sctab[64];
  for (int i = threadIdx.x; i < 64; i += blockDim.x) {
    etab[i] = fast::kExp2Tab[i];
    sctab[i] = fast::kSinCosTab[i];
  }
  __syncthreads();
  near_item<F, DL, CUT>(a, (int64_t)blockIdx.x * kNearWarps + (threadIdx.x >> 5), blockIdx.y * F, etab, sctab);
}

// the items K3's fused near-field warps left: (target k, class tile) = (i mod M, i div M), one
// warp per item, items from the counter the far10 launch shares
template <int F>
__global__ void __launch_bounds__(kNearWarps * 32) near_tail_kernel(NearArgs a, unsigned* ctr, unsigned n_items) {
  __shared__ double etab[64];
  __shared__ double2 sctab[64];
  for (int i = threadIdx.x; i < 64; i += blockDim.x) {
    etab[i] = fast::kExp2Tab[i];
    sctab[i] = fast::kSinCosTab[i];
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  for (;;) {
    unsigned i = 0;
    if (lane == 0) i = atomicAdd(ctr, 1u);
    i = __shfl_sync(0xffffffffu, i, 0);
    if (i >= n_items) break;
    near_item<F, false>(a, (int64_t)(i % (unsigned)a.M), (int)(i / (unsigned)a.M) * F, etab, sctab);
  }
}

template <int F, bool CUT>
__global__ void __launch_bounds__(kNearWarps * 32) near_kernel(NearArgs a) {
  near_body<F, false, CUT>(a);
}
// double-layer near field (NEXT-1)
__global__ void __launch_bounds__(kNearWarps * 32) near_kernel_dl(NearArgs a) { near_body<4, true, false>(a); }

template <int F>
cudaError_t launch(const NearArgs& na, cudaStream_t st) {
  dim3 g((unsigned)((na.M + kNearWarps - 1) / kNearWarps), (unsigned)((na.n_class + F - 1) / F));
  if (na.tau > 0.0) near_kernel<F, true><<<g, kNearWarps * 32, 0, st>>>(na);
  else near_kernel<F, false><<<g, kNearWarps * 32, 0, st>>>(na);
  return cudaGetLastError();
}

}  // namespace

void near_args(Op& op, const double2* xc, double2* yc, NearArgs& na, int& F) {
  Tree& t = *op.tree;
  na.M = t.M; na.n_class = op.n_class; na.leaf_of = t.d_leaf_of.p;
  const bool dense = op.mode == BEM_MODE_DENSE;
  na.near_jb = dense ? op.d_dn_jb.p : t.d_near_jb.p;
  na.near_je = dense ? op.d_dn_je.p : t.d_near_je.p;
  na.near_j = dense ? op.d_dn_j.p : t.d_near_j.p;
  na.cen = t.d_cen.p; na.qn = t.d_qn.p; na.qw = t.d_qw.p; na.nrm = t.d_nrm.p; na.selfJ = t.d_selfJ.p;
  na.s = (const double2*)op.d_s.p; na.local_l = op.d_local_l.p;
  na.class_t1 = op.d_class_t1.p; na.class_t2 = op.d_class_t2.p; na.mask = op.d_mask; na.xc = xc; na.yc = yc;
  na.tau = op.near_tau;
  na.near_gb = dense ? nullptr : t.d_near_gb.p;
  na.gsuf = dense ? nullptr : t.d_near_gsuf.p;
  na.gsuf_n = (int64_t)t.d_near_gsuf.n;
  na.hmax = t.hmax;
  na.evals = op.profile ? op.d_near_evals.p : nullptr;
  // F = 4 classes per warp unless that pads the last class tile by more than 3 % and F = 5
  // pads less (config 2: 65 classes -> F = 5, 5.71 -> 5.64 ms; configs 3/4 keep F = 4)
  const int c = op.n_class;
  const double w4 = double((c + 3) / 4 * 4 - c) / c, w5 = double((c + 4) / 5 * 5 - c) / c;
  F = (w4 > 0.03 && w5 < w4) ? 5 : 4;
}

bem_status launch_near_tail(const NearArgs& na, int F, unsigned* ctr, cudaStream_t st) {
  static int nsm = [] {
    int dev = 0, n = 148;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n;
  }();
  const unsigned n_items = (unsigned)(na.M * (int64_t)((na.n_class + F - 1) / F));
  const unsigned grid = (unsigned)nsm * 4;  // 16 warps per SM (the standalone K1 residency)
  if (F == 5) near_tail_kernel<5><<<grid, kNearWarps * 32, 0, st>>>(na, ctr, n_items);
  else near_tail_kernel<4><<<grid, kNearWarps * 32, 0, st>>>(na, ctr, n_items);
  BEM_CK(cudaGetLastError());
  return BEM_OK;
}

bem_status launch_near(Op& op, const double2* xc, double2* yc, cudaStream_t st, bool dl) {
  if (!dl && op.mode == BEM_MODE_COMBINED) return launch_near_maca(op, xc, yc, st);  // NEXT-4 (nearm.cu)
  NearArgs na;
  int F = 4;
  near_args(op, xc, yc, na, F);
  cudaError_t e;
  if (dl) {
    dim3 g((unsigned)((na.M + kNearWarps - 1) / kNearWarps), (unsigned)((na.n_class + 3) / 4));
    near_kernel_dl<<<g, kNearWarps * 32, 0, st>>>(na);
    e = cudaGetLastError();
  } else {
    e = F == 5 ? launch<5>(na, st) : launch<4>(na, st);
  }
  BEM_CK(e);
  return BEM_OK;
}

}  // namespace bem
