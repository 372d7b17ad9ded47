// Internal definitions shared by the library's translation units.
// (Nothing here is shared with oracle/: the oracle is independent test infra.)
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <functional>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "../../include/bem.h"

namespace bem {

// Device-side bounds checks, compiled in only for the checked build
// (`python -m paper_2006_05186_b200.build --checked` -> libbem_checked.so): the
// memory-safety evidence on this pool, where compute-sanitizer is not available.
#ifdef BEM_CHECKS
#include <cstdio>
#define BEM_DASSERT(c)                                                                                 \
  do {                                                                                                 \
    if (!(c)) {                                                                                        \
      printf("BEM_DASSERT failed %s:%d: %s (block %d, thread %d)\n", __FILE__, __LINE__, #c, blockIdx.x, \
             threadIdx.x);                                                                             \
      __trap();                                                                                        \
    }                                                                                                  \
  } while (0)
#else
#define BEM_DASSERT(c) \
  do {                 \
  } while (0)
#endif

// Asynchronous 16-byte global -> shared copies (LDGSTS) for the software-pipelined
// kernels (K4 Stockham, K2 leaf products): the next tile streams in while the current
// one is computed.
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;\n" ::: "memory"); }

// NVTX range over a host scope (stage markers for ncu --nvtx / profilers: the paper's
// stage timings P:1808-1828 -- tree, ACA, gather, K1, K2, K3, K4, GMRES).  Header-only
// NVTX v3: a no-op unless a profiler injects itself.
struct Nvtx {
  explicit Nvtx(const char* name) { nvtxRangePushA(name); }
  ~Nvtx() { nvtxRangePop(); }
  Nvtx(const Nvtx&) = delete;
  Nvtx& operator=(const Nvtx&) = delete;
};

void set_error(const char* fmt, ...);

#define BEM_CK(call)                                                                        \
  do {                                                                                      \
    cudaError_t e_ = (call);                                                                \
    if (e_ != cudaSuccess) {                                                                \
      bem::set_error("CUDA error %s at %s:%d: %s", cudaGetErrorName(e_), __FILE__, __LINE__, \
                     cudaGetErrorString(e_));                                               \
      return e_ == cudaErrorMemoryAllocation ? BEM_ENOMEM : BEM_ECUDA;                      \
    }                                                                                       \
  } while (0)

#define BEM_REQ(cond, ...)        \
  do {                            \
    if (!(cond)) {                \
      bem::set_error(__VA_ARGS__); \
      return BEM_EINVAL;          \
    }                             \
  } while (0)

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    if (dev < 0) return;  // host-only handle
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    if (prev < 0) return;
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

template <class T>
struct DBuf {  // owning device buffer
  T* p = nullptr;
  size_t n = 0;
  DBuf() = default;
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  DBuf(DBuf&& o) noexcept : p(o.p), n(o.n) { o.p = nullptr; o.n = 0; }
  DBuf& operator=(DBuf&& o) noexcept {
    if (this != &o) { release(); p = o.p; n = o.n; o.p = nullptr; o.n = 0; }
    return *this;
  }
  ~DBuf() { release(); }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
  cudaError_t alloc(size_t count) {
    release();
    if (count == 0) return cudaSuccess;
    cudaError_t e = cudaMalloc((void**)&p, count * sizeof(T));
    if (e == cudaSuccess) n = count;
    return e;
  }
  cudaError_t upload(const std::vector<T>& h) {
    cudaError_t e = alloc(h.size());
    if (e != cudaSuccess || h.empty()) return e;
    return cudaMemcpy(p, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice);
  }
};

struct Tree {
  int device = 0;
  int64_t M = 0;
  int C = 0, n_leaves = 0, depth = 0, m = 1, p = 1, nmin = 2;
  double eta = 1.0;
  int refcount = 0;
  // host
  std::vector<int32_t> perm, begin, end, son0, son1, level, parent;
  std::vector<double> box, xi;  // box C*6, xi C*3*m
  std::vector<int32_t> near_r, near_c, far_r, far_c;
  std::vector<int32_t> leaves;                   // leaf cluster ids in DFS order
  std::vector<std::vector<int32_t>> level_nonleaf;  // non-leaf clusters per level
  int64_t nnz_near = 0;
  double hmax = 0.0;  // largest quadrature-node-to-centroid distance (K1's underflow cutoff)
  // device, cluster order
  DBuf<int32_t> d_perm, d_begin, d_end, d_son0, d_son1, d_parent, d_leaf_of;
  DBuf<double> d_cen;    // M*3
  DBuf<double> d_qn;     // M*21 quadrature nodes
  DBuf<double> d_qw;     // M*7  w_q * |T_j| / (4 pi)
  DBuf<double> d_selfJ;  // M    J(T)/(4 pi)
  DBuf<double> d_area;   // M
  DBuf<double> d_U, d_W; // M*p
  DBuf<double> d_WK;     // M*p double-layer column basis (NEXT-1)
  DBuf<double> d_nrm;    // M*3 unit normals (cluster order)
  DBuf<double> d_E;      // C*p*p (E of cluster c w.r.t. its parent)
  DBuf<double> d_E1;     // C*3*m*m: E = E_z (x) E_y (x) E_x, E_a[lam_a][mu_a] = parent's 1-D Lagrange mu_a at son node lam_a
  DBuf<double> d_ET, d_UT;  // transposed E (C*p*p) and U (p*M) for the downward pass
  DBuf<double> d_xi;     // C*3*m
  DBuf<int32_t> d_leaves;
  // near field per leaf index: [jb, je) into the flat list of near source panels
  DBuf<int32_t> d_near_jb, d_near_je, d_near_j;
  DBuf<int32_t> d_near_gb;   // per leaf: first entry of its warp steps in d_near_gsuf
  DBuf<unsigned> d_near_gsuf;  // per warp step of 32 sources: float bits of the min squared distance of the leaf box to any later source centroid (rounded down)
  // near blocks (combined mode, NEXT-4): block list, per-row-leaf CSR, raw J(T) (cluster order)
  DBuf<int32_t> d_near_r, d_near_c, d_nb_ptr, d_nb_sorted;
  DBuf<double> d_J;
  int max_leaf = 0;
  std::vector<int32_t> nb_ptr, nb_sorted;  // host copies of d_nb_ptr / d_nb_sorted
  // far CSR by row cluster
  std::vector<int32_t> far_ptr, far_sorted;  // far_sorted: block ids grouped by row cluster
  DBuf<int32_t> d_far_ptr, d_far_sorted, d_far_r, d_far_c;
  std::vector<DBuf<int32_t>> d_level_nonleaf;
};

// bem_time_step's device buffers and captured graph (step.cu)
struct StepGraph {
  DBuf<double> tx, xf, yf, ty;  // [L][M] complex each
  cudaStream_t own = nullptr;
  cudaEvent_t e0 = nullptr, e1 = nullptr, e2 = nullptr;  // e2: end of the last call's D2H
  bool used = false;
  cudaGraphExec_t exec = nullptr;
  double R = 0.0;
  StepGraph() = default;
  StepGraph(const StepGraph&) = delete;
  StepGraph& operator=(const StepGraph&) = delete;
  ~StepGraph();
};

struct Op {
  Tree* tree = nullptr;
  int L = 0, n_local = 0, mode = 0;
  double eps = 0.0;
  std::vector<int32_t> local_l;
  DBuf<double> d_s;        // L complex (interleaved)
  DBuf<int32_t> d_local_l; // n_local
  // frequency classes for the near field: (t1, t2) local indices, t2 = -1 if unpaired
  int n_class = 0;
  DBuf<int32_t> d_class_t1, d_class_t2;
  // BEM_MODE_DENSE: every leaf's near list is the whole index range [0, M)
  DBuf<int32_t> d_dn_jb, d_dn_je, d_dn_j;
  // ACA skeleton
  int rcap = 0;
  std::vector<int32_t> ranks;  // host copy
  DBuf<int32_t> d_rank, d_pivk, d_pivq;  // pivk/pivq: nfar * rcap
  DBuf<int64_t> d_zoff;                  // nfar
  DBuf<double> d_Z;                      // pool: sum r_b * n_local complex (if z_stored)
  DBuf<int64_t> d_foff;                  // nfar: offsets of F_b in d_F
  DBuf<double> d_F;                      // pool: sum r_b^2 complex, F_b = C^_b (lower) + U_b (strict upper)
  bool z_stored = true;                  // false: K3 regenerates Z tiles from F_b (factors-only)
  int rmax = 0;                          // largest far rank
  DBuf<double> d_zs;                     // factors-only: Z tile buffer, per block [r_b][ZW] at d_ztoff[b]
  DBuf<int64_t> d_ztoff;
  // row clusters owning far blocks, sorted by descending coupling work (K3 order)
  int n_far_rows = 0;
  DBuf<int32_t> d_far_rows;
  // K3 work segments: (row, bi0, bi1, slot) in launch (cost-descending) order;
  // seg_rows/seg_ptr: per row with far blocks, its contiguous slot range
  int n_segs = 0, n_seg_rows = 0;
  DBuf<int32_t> d_segs, d_seg_rows, d_seg_ptr;
  DBuf<double> d_part;  // n_segs * n_local * p complex
  // near-field MACA (BEM_MODE_COMBINED, Alg. 3 NEAR branch): per near block rank, pivots,
  // Z (r x n_local) and the pivot slices V_{k_t}[b] (r x n_r x n_c, row-major) in pools
  int nrcap = 0;
  std::vector<int32_t> nranks;
  DBuf<int32_t> d_nrank, d_npivk, d_npivq;
  DBuf<int64_t> d_nzoff, d_nsoff;
  DBuf<double> d_nZ, d_nS;
  DBuf<int32_t> d_nm_order, d_nm_counter;
  // time-domain path (NEXT-2, mot.cu): dhat rows of the far / near skeletons (same offsets as
  // d_Z / d_nZ, row length L), stored far pivot slices S_b(s_{k_t}) [r_b][p][p] at fsoff[b]
  bool mot_ready = false;
  double mot_R = 0.0;
  DBuf<double> d_Df, d_Dn, d_fS;
  DBuf<int64_t> d_fsoff;
  DBuf<double> d_g0f, d_g0n;  // Re V^_0 blocks (far p x p, near n_r x n_c at d_g0noff)
  DBuf<int64_t> d_g0noff;
  DBuf<double> d_conv_part;  // per-block partial sums of the time-domain convolution  // K1m CTA order: leaf indices by descending sum_b r_b n_c (LPT)
  // workspaces
  DBuf<double> d_xc, d_yc, d_xhat, d_yhat;
  DBuf<double> d_xmax;  // far10: [C][nl] max_nu |xhat|
  // kernel selection (env BEM_FAR_KERNEL / BEM_FAR8_KC / BEM_FAR_GENERIC, read at assembly: tests)
  bool force_generic = false;
  int far_kernel = 0;                 // 0: auto (far10 where it applies, else far8 for p > 32 / far7); 10, 8, 7
  size_t far4_smem_cap = 113 * 1024;  // 2 CTAs per SM
  int far8_kc = 0;                    // far8 nu-chunk width (0: automatic)
  bool far8_m3 = true;                // far8: 3M complex products at 16-row mu chunks (env BEM_FAR8_M3=0: 4M, 32 rows)
  bool far8_dt = true;                // far8 3M: per-block (r, 1/4 pi r) table in shared memory (env BEM_FAR8_DT=0: off)
  int aca_ctas_per_sm = 5;            // persistent ACA CTAs per SM = register-limited residency (r01: 4 -> 5 cut config-4 setup 2.96 -> 2.64 s)
  int h2o_fc = 0;                     // K3' classes per CTA tile (0: 6 for p <= 32, else 2)
  // optional per-local-frequency mask (1 = compute); set only by the GMRES driver so that
  // converged frequencies skip K1 / K3 work (their outputs are then zero)
  const int32_t* d_mask = nullptr;
  bool use_solve_mask = true;  // env BEM_SOLVE_MASK=0 disables
  StepGraph step;  // bem_time_step
  // K1 || far-branch overlap (apply.cu): side stream and fork/join events, created lazily
  bool overlap = true;
  bool k1_fuse = true;           // K1 fused into far10 where it runs (BEM_K1_FUSE=0: separate kernel)
  DBuf<unsigned> d_nctr;         // its item counter
  int k1_warps = 3;              // near-field warps per far10 CTA (1..3; 9 + 3 warps x 168 registers fill an SM)
  bool far10_persist = true;     // far10 as persistent CTAs (one per SM) taking items from d_f10ctr
  DBuf<int32_t> d_f10ctr;
  // underflow cutoffs: K1 skips a class over a warp step of sources when
  // Re s r_min > near_tau (env BEM_NEAR_TAU, 0: off); far10 skips a (block, frequency tile) whose
  // compressed fibres are bounded by far_delta / max(|s_t|, 1) (env BEM_FAR_SKIP_LOG2, 0: off)
  double near_tau = 42.0;
  double far_delta = 0x1p-70;
  DBuf<unsigned> d_skip;                 // far10: bit `tile` of d_skip[b]
  DBuf<int32_t> d_colmap;                // far10: [tiles][128] local frequency of a tile column (-1: padding)
  std::vector<int32_t> colmap;
  DBuf<unsigned long long> d_near_evals;  // profiling: kernel evaluations K1 ran in the last apply
  cudaStream_t side = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  // profiling
  bool profile = false;
  cudaEvent_t ev[6] = {};
  double timings[5] = {0, 0, 0, 0, 0};
};

// launchers (apply.cu, near.cu, far.cu)
bem_status apply_launch(Op& op, const double* x, double* y, cudaStream_t st, bool dl = false, double alpha = 0.0);
bem_status launch_near(Op& op, const double2* xc, double2* yc, cudaStream_t st, bool dl = false);
struct NearArgs;
// fna != nullptr (only when far_fuses_near(op)): K1 runs inside the far10 launch (near-field warps)
// and in a tail kernel after it, both taking items from op.d_nctr
bem_status launch_far(Op& op, const double2* xhat, double2* yhat, cudaStream_t st, const NearArgs* fna = nullptr);
bool far_fuses_near(const Op& op);
bem_status far_prepare(Op& op);  // K3 scratch of the factors-only skeleton (far.cu)
void far10_work(Op& op, int64_t* run, int64_t* total);  // (rank x column) products run / in total (far.cu)
int far_kernel_selected(const Op& op);  // the K3 kernel an apply launches (10, 8, 7; 0: generic)
bem_status launch_near_maca(Op& op, const double2* xc, double2* yc, cudaStream_t st);  // nearm.cu
bem_status h2_gather(Op& op, const double2* x, double2* xc, int ncols, cudaStream_t st);
bem_status h2_up(Op& op, const double2* xc, double2* xhat, int ncols, cudaStream_t st);
bem_status h2_down_scatter(Op& op, double2* yhat, const double2* ycn, double2* y, int ncols, cudaStream_t st);
// solve.cu: batched GMRES on an arbitrary operator ([nl][M] complex columns), stats;
// the workspace is reused across calls of the same shape (the MoT solves one system per step)
struct GmresWs {
  DBuf<double> r, w, V, h, H, g, cs, sn, y, beta, bnorm, hn;
  DBuf<int> active, cyc, jt, iters, cnt;
  int64_t n = -1;
  int nl = -1, restart = -1;
};
bem_status gmres_fn(int64_t M, int nl, const std::function<bem_status(const double*, double*)>& apply,
                    const double2* B, double2* X, double tol, int restart, int max_iter, cudaStream_t st,
                    std::vector<int>& hit, std::vector<double>& hrel, GmresWs& ws);
bem_status solve_stats(const std::vector<int>& hit, const std::vector<double>& hrel, double tol, int max_iter,
                       double imag_rel, bem_solve_stats* stats);
// fft.cu; tab (mode 1: input rows, 2: output rows) = host row-pointer table, copied into the launch
bem_status fft_transform_rows(const double* in, double* out, int64_t M, int N, double R, bool inverse,
                              cudaStream_t st, const double2* const* tab, int mode);
// comm.cu: NCCL frequency sharding
bool shard_frequencies(int L, int G, std::vector<int>& owner, std::vector<int>& slot,
                       std::vector<std::vector<int>>* lists);
bem_status shard_forward(Op& op, bem_comm c, const double* x_time, double R, double2** xf, cudaStream_t st);
bem_status shard_inverse(Op& op, bem_comm c, const double2* yf, double R, double* y_time, cudaStream_t st);
bem_status shard_yf(Op& op, bem_comm c, double2** yf);
bem_status comm_allreduce(bem_comm c, double* dev, int nmax, int nsum, cudaStream_t st);
bem_status comm_check(bem_comm c, const Op& op, int64_t M_loc);
double* comm_scratch(bem_comm c);
void shard_ws_release(const Op* op);
bem_status fft_transform(const double* in, double* out, int64_t M, int N, double R, bool inverse,
                         cudaStream_t st);

}  // namespace bem

struct bem_tree_s {
  bem::Tree t;
};
struct bem_op_s {
  bem::Op o;
};
