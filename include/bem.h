/* bem.h -- C-ABI of the B200 (sm_100a) multi-frequency H^2 + ACA single-layer
 * library (paper_2006_05186_b200/csrc, built as libbem.so).
 *
 * Paper: D. Seibel, "Boundary Element Methods for the Wave Equation based on
 * Hierarchical Matrices and Adaptive Cross Approximation", arXiv 2006.05186.
 * "P:<a-b>" below cites /root/reference/PAPER.md lines; "S:<a-b>" SPEC.md;
 * readings (AM<k>, D<k>) are listed in DESIGN.md.
 *
 * Conventions (all entry points):
 *  - Every call returns bem_status: 0 = OK, < 0 = error; bem_last_error()
 *    returns a thread-local message valid until the next bem_* call on the
 *    same thread.  On error outputs are unspecified and handles stay valid.
 *  - Host pointers are borrowed for the duration of the call and copied.
 *  - Device pointers are caller-owned (e.g. torch tensors), contiguous,
 *    16-byte aligned, on the handle's device, and must stay alive until the
 *    work enqueued on `cuda_stream` has finished.  Handles own their device
 *    memory and free it in *_destroy.
 *  - `cuda_stream` is a cudaStream_t (NULL = legacy default stream).  apply,
 *    cqm_forward and cqm_inverse are asynchronous; build, assemble and solve
 *    synchronise before returning.
 *  - Complex data are interleaved (re, im) doubles: the layout of
 *    std::complex<double>, cuDoubleComplex and torch.complex128.
 *  - Frequency-domain arrays are [l][panel] row-major with the panel index in
 *    INPUT order (the tree permutation is internal); time-domain arrays are
 *    [n][panel].
 *  - Results are bitwise reproducible for identical inputs and device.
 *  - Distinct handles may be used concurrently from different threads; a
 *    single handle may not.
 */
#ifndef BEM_H_
#define BEM_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef int32_t bem_status;
enum {
  BEM_OK = 0,
  BEM_EINVAL = -1,  /* invalid argument (ranges listed per call) */
  BEM_ENOMEM = -2,  /* device or host allocation failed */
  BEM_ECUDA = -3,   /* CUDA runtime error (launch or asynchronous fault) */
  BEM_ENCCL = -4,   /* NCCL missing or failed (sharded multi-GPU calls) */
  BEM_ENOCONV = -5, /* cqm_solve: some frequency hit max_iter (outputs written) */
  BEM_ESTATE = -6   /* handle misuse (wrong device, tree destroyed before its ops) */
};

/* BEM_MODE_COMBINED: Alg. 3 in full (eq:lrfinal P:1404-1410 for both
 * b in P+ and b in P-): the near blocks are MACA-compressed across frequency too
 * (SURVEY §8(f) NEXT-4), instead of evaluated on the fly per apply. */
enum { BEM_MODE_H2ACA = 0, BEM_MODE_H2ONLY = 1, BEM_MODE_DENSE = 2, BEM_MODE_COMBINED = 3 };
/* Skeleton storage flags, OR-ed into `mode` of bem_assemble_h2_aca (ACA modes).
 * The MACA of block b is kept as pivots (k_l, q_l) plus the r_b x r_b LU factors of
 * A_b[Q,K] (SURVEY C10 skeleton form, AM17; 16 r_b^2 bytes).  The coefficients
 * Z_b = U_b^{-1} C^_b^{-1} A_b[Q,:] (eq:maca P:1314-1320) of the local frequencies are
 *   BEM_SKEL_Z:       regenerated once at assembly and stored (16 r_b n_local bytes);
 *   BEM_SKEL_FACTORS: regenerated per apply in the coupling kernel's prologue, per
 *                     (block, frequency tile) -- nothing per frequency is stored;
 *   neither:          stored when that takes at most a third of the free device memory.
 * Both give bit-identical results (the same pinned substitutions as the ACA). */
enum { BEM_SKEL_Z = 0x100, BEM_SKEL_FACTORS = 0x200 };

typedef struct { double re, im; } bem_c128;
typedef struct bem_tree_s* bem_tree; /* panels, cluster tree, P+/P-, U, W, E, boxes; one device */
typedef struct bem_op_s* bem_op;     /* tree ref + s_l + ACA skeletons for a local frequency set */
typedef struct bem_comm_s* bem_comm; /* NCCL communicator of a frequency-sharded multi-GPU run */

typedef struct {
  int64_t M, clusters, leaves, near_blocks, far_blocks, nnz_near;
  int32_t depth, p;
} bem_tree_stats;

typedef struct {
  int32_t iters_max, iters_sum, n_unconverged, pad_;
  double resid_max, imag_rel_max;
} bem_solve_stats;

const char* bem_last_error(void);

/* CQM frequencies, eq:cqm_freq P:443-447 with the north_star sign (AM2):
 *   s_l = delta(R e^{-2 pi i l/L}) / dt,  dt = T/N,  L = N+1 (AM1),
 *   delta(z) = 1 - z (method 1, BDF1) or 3/2 - 2z + z^2/2 (method 2, BDF2);
 *   s_{L-l} := conj(s_l) exactly, Im s_0 = 0 exactly.
 * s_out: host, L = N+1 entries.  EINVAL: N < 1, T <= 0, R not in (0,1),
 * method not in {1,2}, s_out NULL. */
bem_status cqm_frequencies(int32_t N, double T, double R, int32_t method, bem_c128* s_out);

/* Geometry + cluster tree + admissible partition + cluster bases (P:738-1070,
 * Alg. 1; clustering P:832-835; partition eq:qadm P:905-912 with near <=>
 * inadmissible leaf x leaf (AM9); Chebyshev bases P:957-978).
 *   vertices  host [nv][3] doubles;  triangles host [nt][3] int32, 0-based;
 *   leaf_size n_min > 1 (leaves hold <= n_min panels, AM6); eta > 0;
 *   cheb_order 1 <= m <= 5 (p = m^3 interpolation points per box);
 *   device: CUDA ordinal.  Synchronous.  *out receives a new handle.
 * EINVAL: nv < 3, nt < 1, an index out of range, a degenerate triangle
 * (area <= 0), leaf_size <= 1, eta <= 0, m < 1 or m > 5, out NULL. */
bem_status bem_build_tree(const double* vertices, int64_t nv, const int32_t* triangles, int64_t nt,
                          int32_t leaf_size, double eta, int32_t cheb_order, int32_t device, bem_tree* out);
bem_status bem_tree_get_stats(bem_tree t, bem_tree_stats* out);
/* Host outputs, caller-sized from the stats (any may be NULL):
 *   perm [M] (perm[k] = input index of the k-th panel in cluster order),
 *   clusters [C][5] = (begin, end, son0, son1, level) in DFS pre-order,
 *   boxes [C][6] = (lo_x, lo_y, lo_z, hi_x, hi_y, hi_z),
 *   near_pairs [near][2], far_pairs [far][2] = (row cluster, col cluster). */
bem_status bem_tree_export(bem_tree t, int32_t* perm, int32_t* clusters, double* boxes, int32_t* near_pairs,
                           int32_t* far_pairs);
/* NULL-safe.  Returns BEM_ESTATE (and keeps the tree) while ops built on it live. */
bem_status bem_tree_destroy(bem_tree t);

/* Multi-frequency operator (Alg. 3, FAR branch; eq:lrfinal P:1404-1410).
 *   s: host [L] frequencies (normally from cqm_frequencies); must be exactly
 *      conjugation-symmetric, s[L-l] == conj(s[l]) for 0 < l < L (EINVAL otherwise):
 *      l > L/2 is evaluated as the conjugate of L - l (SURVEY C2, C10 reading 5);
 *   local_l: host [n_local] distinct frequency indices this handle applies
 *            (NULL = all L, n_local ignored);
 *   aca_eps > 0: MACA tolerance (Alg. 2, stop rule P:1288);
 *   mode: BEM_MODE_H2ACA (the product), BEM_MODE_H2ONLY (couplings evaluated
 *         per frequency, no ACA; plain-H^2 comparison path), BEM_MODE_DENSE
 *         (every leaf pair is evaluated as near field), BEM_MODE_COMBINED (H2ACA
 *         plus MACA of every near block: Alg. 3 NEAR branch P:1426-1431, entries
 *         V[b][i,j](s) of the NEAR procedure P:1444-1450 in the collocation reading,
 *         evaluated in pinned arithmetic; stores the pivot slices V_{k_t}[b], i.e.
 *         16 * sum_b r_b n_r n_c bytes -- the tensor C_b of eq:lrfinal).
 *         The double-layer apply of a COMBINED op keeps its near field exact.
 *         COMBINED requires leaves of at most 64 panels (EINVAL otherwise).
 * The ACA runs over ALL L frequencies on the device with pinned arithmetic
 * (bit-reproducible pivots) and keeps Z columns for local_l only.
 *   mode may carry one BEM_SKEL_* flag (ACA modes; COMBINED always stores Z).
 * Synchronous on return.  EINVAL: L < 1, s NULL or not conjugation-symmetric, local
 * index out of range or duplicated, aca_eps <= 0, unknown mode or flags.
 * ENOMEM: BEM_SKEL_Z (or COMBINED) and the stored Z does not fit. */
bem_status bem_assemble_h2_aca(bem_tree t, const bem_c128* s, int32_t L, const int32_t* local_l, int32_t n_local,
                               double aca_eps, int32_t mode, void* cuda_stream, bem_op* out);
/* ranks: host [far_blocks]; pivots: host [sum ranks][2] = (k_l, q_l) in block
 * order (q = mu*p + nu, mode-3 unfolding P:1322-1334).  Either may be NULL.
 * *total_rank (may be NULL) receives sum ranks.  ESTATE for non-ACA modes. */
bem_status bem_aca_export(bem_op op, int32_t* ranks, int32_t* pivots, int64_t* total_rank);
/* Near-block skeletons of a BEM_MODE_COMBINED op: ranks host [near_blocks];
 * pivots host [sum ranks][2] = (k_l, q_l), q = i_loc * n_c + j_loc with i_loc /
 * j_loc the row / column panel offsets inside the block's clusters (cluster
 * order), blocks in bem_tree_export's near_pairs order.  ESTATE otherwise. */
bem_status bem_aca_export_near(bem_op op, int32_t* ranks, int32_t* pivots, int64_t* total_rank);
bem_status bem_op_destroy(bem_op op); /* NULL-safe */
/* What an op holds (host struct):  skeleton = 0 (no ACA: H2ONLY / DENSE), 1 (stored Z),
 * 2 (factors only, BEM_SKEL_FACTORS); z_bytes / f_bytes = the stored Z and factor pools;
 * device_bytes = every device allocation the op owns (its per-GPU footprint besides
 * the tree and the caller's x / y); far_kernel = the K3 coupling kernel an apply launches:
 * 10 (far10: FP64 products emulated on the INT8 tensor cores), 8 / 7 (FP64 tensor cores,
 * mma.sync f64), 0 (generic / plain-H^2 / dense paths). */
typedef struct {
  int32_t mode, skeleton, n_local, rmax;
  int64_t total_rank, z_bytes, f_bytes, device_bytes;
  int32_t far_kernel, reserved_;
} bem_op_info;
bem_status bem_op_get_info(bem_op op, bem_op_info* out);

/* y_t = V(s_{local_l[t]}) x_t for t < n_local (P:529-540 operators V_l).
 * x, y: device [n_local][M] complex, input panel order; y is overwritten;
 * x and y must not overlap.  Asynchronous on cuda_stream. */
bem_status bem_apply_multifreq(bem_op op, const bem_c128* x, bem_c128* y, void* cuda_stream);

/* Double-layer operator (eq:wavebio P:301-303, the
 * gamma_{1,y}-derivative of the fundamental solution eq:fundsol P:479-482):
 *   y_t = (alpha I + K(s_{local_l[t]})) x_t,
 *   K[i,j](s) = |T_j| sum_q w_q d/dn_y [e^{-s r}/(4 pi r)] at (c_i, y_{j,q}),
 *             = |T_j| sum_q w_q (-(1 + s r) e^{-s r} (y - c_i).n_j / (4 pi r^3)),
 *   K[i,i] = 0 (flat panels), n_j = (b-a)x(c-a)/|.| in the triangle's vertex order.
 * Far field: the op's coupling tensors / ACA skeleton (unchanged: the kernel
 * is interpolated in y and then differentiated) with the column basis
 * |T_j| sum_q w_q n_j . grad L_{c,nu}(y_{j,q}).  alpha = -1/2 gives the right-hand
 * side (-1/2 I + K) g of the direct Dirichlet formulation eq:cqmdir P:1801-1806.
 * x, y: device [n_local][M] complex, input panel order, no overlap.  Asynchronous. */
bem_status bem_apply_double_layer(bem_op op, const bem_c128* x, bem_c128* y, double alpha, void* cuda_stream);

/* One time-domain operator step, y_time = cqm_inverse(V(s_l) cqm_forward(x_time)) (the
 * bench's step; eq:omega_n P:436-441 around eq:slphelm P:529-540).  x_time, y_time: [L][M]
 * complex, input panel order, HOST (pageable or pinned) or DEVICE memory; the op must hold
 * all L = N+1 frequencies (local_l = 0..L-1).  The device part runs from a CUDA graph the
 * op captures at its first call (and again when R changes); host buffers are copied
 * through the op's device time buffers.  Asynchronous on cuda_stream for pinned/device
 * buffers.  Not while profiling is enabled (then eager). */
bem_status bem_time_step(bem_op op, const bem_c128* x_time, bem_c128* y_time, double R, void* cuda_stream);

/* Time-domain path with compressed weights (eq:fastdft
 * P:1542-1553, eq:fastrhs P:1566-1573, eq:cqmrhs P:652-680).  The op must be
 * BEM_MODE_COMBINED (every block in MACA skeleton form) and hold all L = N+1
 * frequencies (local_l = 0..L-1); else ESTATE / EINVAL.
 * bem_mot_prepare: dhat_{b,t}[n] = (R^{-n}/L) sum_l Z_b[t,l] e^{+2 pi i (nl mod L)/L}
 *   for every far and near skeleton row (the weights V^_n[b] = sum_t C_{b,t} dhat_{b,t}[n]),
 *   and stores the far pivot slices S_b(s_{k_t}) (16 sum_b r_b p^2 bytes).  Synchronous.
 * bem_conv_time: y_n = sum_{k <= min(n, kmax)} V^_{n-k} q_k, n = 0..N, with the compressed
 *   weights in the order of eq:fastrhs.  q, y: device [L][M] complex, input panel order,
 *   no overlap.  Synchronous.
 * cqm_mot_solve: marching on in time for V q = g: for n = 0..N solve
 *   Re V^_0 q_n = g_n - Re sum_{k<n} V^_{n-k} q_k by GMRES(restart) to tol (the paper
 *   factorises V^_0 once; an iterative solver is its stated alternative).
 *   g_time, phi_time: device [L][M] real.  stats over the time steps.  Synchronous;
 *   ENOCONV if some step missed tol (phi_time still written).  Stable only where the
 *   discretisation's recursion is (Courant >~ 0.5 for this collocation). */
bem_status bem_mot_prepare(bem_op op, double R, void* cuda_stream);
bem_status bem_conv_time(bem_op op, const bem_c128* q, bem_c128* y, int32_t kmax, void* cuda_stream);
bem_status cqm_mot_solve(bem_op op, const double* g_time, double* phi_time, double tol, int32_t restart,
                         int32_t max_iter, void* cuda_stream, bem_solve_stats* stats);

/* R-scaled CQM transforms (eq:omega_n P:436-441, eq:slphelm P:529-540; D2):
 *   forward:  x_freq[l] = sum_{n=0}^{N} R^n x_time[n] e^{-2 pi i n l / L}
 *   inverse:  y_time[n] = R^{-n}/L sum_{l=0}^{L-1} y_freq[l] e^{+2 pi i n l / L}
 * L = N+1; device [L][M_loc] complex each; in-place is NOT allowed.
 * Batched Bluestein FFT on the device.  Asynchronous.
 * EINVAL: M_loc < 1, N < 1, R not in (0,1], NULL pointers. */
bem_status cqm_forward(const bem_c128* x_time, bem_c128* x_freq, int64_t M_loc, int32_t N, double R,
                       void* cuda_stream);
bem_status cqm_inverse(const bem_c128* y_freq, bem_c128* y_time, int64_t M_loc, int32_t N, double R,
                       void* cuda_stream);

/* Frequency-decoupled CQM solve of the single-layer equation V phi = g
 * (Remark P:1607-1614; indirect first-kind reading D10):
 *   g^ = forward(g); for every l solve V(s_l) phi^_l = g^_l by restarted
 *   GMRES(restart) from 0, classical Gram-Schmidt with one
 *   re-orthogonalisation, stop at ||g^_l - V phi^_l|| <= tol ||g^_l||;
 *   phi = Re inverse(phi^).
 * nccl_comm = NULL: one device; g_time, phi_time device [N+1][M] real, M_loc = M,
 *   the op holds all L = N+1 frequencies in order.
 * nccl_comm = a bem_comm of G ranks (bem_comm_init; the handle type is bem_comm):
 *   rank g passes its DOF shard, g_time / phi_time device [N+1][M_loc] with
 *   M_loc = the size of [M g/G, M (g+1)/G), and its op holds exactly rank g's
 *   frequency shard (bem_shard_frequencies; EINVAL otherwise).  The two
 *   time<->frequency transposes are NCCL all-to-alls inside the call (SURVEY
 *   §8(e)); stats are reduced over the ranks (max / sum).  Collective: every rank
 *   of the communicator must call it.
 * stats (host, may be NULL).  Synchronous.  Returns BEM_ENOCONV if some
 * frequency reached max_iter (phi_time is still written), BEM_ENCCL on NCCL errors. */
bem_status cqm_solve(bem_op op, const double* g_time, double* phi_time, int64_t M_loc, double R, double tol,
                     int32_t restart, int32_t max_iter, void* nccl_comm, void* cuda_stream, bem_solve_stats* stats);

/* ---- multi-GPU frequency sharding over NCCL (Remark P:1607-1614) ----
 * Rank g of G owns the DOFs [M g/G, M (g+1)/G) of time-domain data and the frequency
 * classes {0}, {j, L-j} of bem_shard_frequencies (class i -> rank i mod G: conjugate pairs
 * kept together, every rank an even sample of the frequency circle, so the underflow cutoffs
 * of bem_op_get_work take the same share from every rank).  NCCL is loaded at run time (libnccl.so.2).
 *   bem_comm_unique_id: 128-byte ncclUniqueId, created on one rank and broadcast by
 *     the caller (e.g. torch.distributed); ENCCL when NCCL cannot be loaded.
 *   bem_comm_init: collective over the nranks processes (ncclCommInitRank); device =
 *     this rank's CUDA ordinal (the ops used with it must live there).
 *   bem_shard_frequencies: host only; owner[l] = rank holding frequency l, slot[l] =
 *     its row in that rank's local list (the op's local_l, in that order).
 *   bem_time_step_sharded: the bench's time-domain step on G ranks, collective:
 *     x_loc [L][M_loc] (this rank's DOF columns, complex, device) -> forward K4 fused
 *     with the packing of the all-to-all -> NCCL all-to-all -> apply of this rank's
 *     frequencies -> all-to-all -> inverse K4 fused with the unpacking -> y_loc
 *     [L][M_loc].  Asynchronous on cuda_stream (NCCL calls enqueue on it). */
bem_status bem_comm_unique_id(void* id_out);
bem_status bem_comm_init(const void* id, int32_t nranks, int32_t rank, int32_t device, bem_comm* out);
bem_status bem_comm_destroy(bem_comm comm); /* NULL-safe */
bem_status bem_shard_frequencies(int32_t L, int32_t G, int32_t* owner, int32_t* slot);
bem_status bem_time_step_sharded(bem_op op, const bem_c128* x_loc, bem_c128* y_loc, int64_t M_loc, double R,
                                 bem_comm comm, void* cuda_stream);

/* Transforms fused with the multi-GPU time<->frequency transpose (SURVEY
 * §8(e)).  The same R-scaled transforms as cqm_forward / cqm_inverse, but
 * row r of the frequency-domain side is addressed through a host array of
 * L = N+1 device pointers, which may point into OTHER ranks' buffers (CUDA
 * IPC handles, see bem_ipc_*; peer memory over NVLink/NVSwitch): one kernel
 * then computes the transform of this rank's DOF columns and stores frequency
 * row l straight into the rank that owns l (forward), or reads it back from
 * the owner (inverse), with no separate all-to-all.
 *   cqm_forward_rows: x_time device [N+1][M_loc] (this rank's columns) ->
 *                     out_rows[l][0..M_loc) for every l;
 *   cqm_inverse_rows: in_rows[l][0..M_loc) for every l -> y_time [N+1][M_loc].
 * The pointer arrays are copied before the call returns; rows must be
 * 16-byte aligned device (or peer-mapped) memory.  N + 1 <= 2048.
 * The caller orders the exchange (e.g. device sync + barrier) across ranks. */
bem_status cqm_forward_rows(const bem_c128* x_time, int64_t M_loc, bem_c128* const* out_rows, int32_t N, double R,
                            void* cuda_stream);
bem_status cqm_inverse_rows(bem_c128* const* in_rows, bem_c128* y_time, int64_t M_loc, int32_t N, double R,
                            void* cuda_stream);
/* CUDA IPC handles (64 bytes) for peer row tables. */
bem_status bem_ipc_get_handle(void* dev_ptr, void* handle_out);
bem_status bem_ipc_open_handle(const void* handle, int32_t device, void** dev_ptr_out);
bem_status bem_ipc_close(void* dev_ptr);
/* Plain cudaMalloc / cudaFree (buffers whose IPC handle maps exactly the buffer). */
bem_status bem_device_alloc(int64_t bytes, int32_t device, void** out);
bem_status bem_device_free(void* ptr);

/* Frequency-domain batched GMRES over the op's local frequencies (the
 * per-frequency systems of the decoupled solve, Remark P:1607-1614; reading
 * D10): for every t < n_local solve V(s_{local_l[t]}) phi_t = g_t by
 * restarted GMRES(restart) from 0 with classical Gram-Schmidt + one
 * re-orthogonalisation and Givens rotations, stopping at
 * ||g_t - V phi_t|| <= tol ||g_t||.  This is the building block of the
 * multi-GPU solve: the caller transforms, transposes (all-to-all) and calls it
 * on each rank's frequency shard (paper_2006_05186_b200/dist.py).
 * g_freq, phi_freq: device [n_local][M] complex, input panel order, distinct.
 * Synchronous.  Returns BEM_ENOCONV if some frequency reached max_iter
 * (phi_freq still written; stats says how many). */
bem_status bem_solve_multifreq(bem_op op, const bem_c128* g_freq, bem_c128* phi_freq, double tol, int32_t restart,
                               int32_t max_iter, void* cuda_stream, bem_solve_stats* stats);

/* ---- diagnostics (tests / bench only; not part of the method) ---- */
/* Pinned exp / sincos / kernel evaluated ON THE DEVICE for n host inputs
 * (checks bit-identity with the independent oracle implementation). */
bem_status bem_debug_pinned(const double* x, int64_t n, double* exp_out, double* sin_out, double* cos_out,
                            int32_t device);
/* Hot-path (K1 / K3 slice regeneration) table-driven exp (x <= 0; 0 returned
 * for x > 0) and sincos evaluated ON THE DEVICE for n host inputs: accuracy
 * check of the fast math against libm (tests).  variant: 64 or 256 (table size). */
bem_status bem_debug_fastmath(const double* x, int64_t n, double* exp_out, double* sin_out, double* cos_out,
                              int32_t device, int32_t variant);
/* MACA (the assembly's kernel and pinned arithmetic) of the listed far blocks only, no
 * skeleton kept: ranks host [nblk], pivots host [sum ranks][2] (NULL: ranks only; size it
 * with min(L, p^2) per block), *total_rank.  Sampled bit-exactness checks at sizes whose
 * full assembly takes minutes. */
bem_status bem_debug_aca_blocks(bem_tree t, const bem_c128* s, int32_t L, double aca_eps, const int32_t* blocks,
                                int32_t nblk, int32_t* ranks, int32_t* pivots, int64_t* total_rank);
/* The sharded time-domain step (bem_time_step_sharded) for G ranks in ONE process on one
 * device: ops[g] holds rank g's frequency shard, x_loc[g] / y_loc[g] rank g's DOF columns
 * [L][M_g]; the all-to-all exchanges are device copies between the ranks' buffers instead
 * of NCCL, the packing / unpacking code is the NCCL path's.  Checks the multi-rank
 * transposes where one GPU is available. */
bem_status bem_debug_sharded_step(int32_t G, bem_op* ops, const bem_c128* const* x_loc, bem_c128* const* y_loc,
                                  double R, void* cuda_stream);
/* One CTA computes D = A B^T on the 5th-generation tensor cores (tcgen05.mma kind::i8,
 * signed 8-bit operands, 32-bit integer accumulators in tensor memory): A host [128][K],
 * B host [N][K], D host [128][N] int32; K a multiple of 32 in [32, 512], N a multiple of 16
 * in [16, 128]; mode 0: A staged in tensor memory, 1: in shared memory.  Pins the operand
 * layouts of the INT8 coupling kernel (far10) against plain integer arithmetic. */
bem_status bem_debug_i8_gemm(const int8_t* A, const int8_t* B, int32_t* D, int32_t K, int32_t N, int32_t mode,
                             int32_t device);
/* The CTA-pair form (cta_group::2, M = 256) on a cluster of two CTAs: A host [256][K],
 * B host [N][K], D host [256][N]; K a multiple of 32 in [32, 512], N a multiple of 32 in
 * [32, 128].  Pins the operand split the paired far10 relies on (CTA r: A rows 128 r..,
 * B rows r N/2..). */
bem_status bem_debug_i8_gemm_pair(const int8_t* A, const int8_t* B, int32_t* D, int32_t K, int32_t N,
                                  int32_t device);
/* tcgen05 kind::i8 issue-rate microbenchmark (far10's MMA pattern: groups of 21 MMAs, M = 128,
 * K = 32, N in {32, 64, 128, 256}; mode 0: A in tensor memory, 1: A in shared memory): int8 MACs/s over
 * all SMs and tensor-core cycles per MMA on SM 0. */
bem_status bem_debug_i8_rate(int32_t N, int32_t mode, int32_t iters, int32_t device, double* macs_per_s,
                             double* cycles_per_mma);
/* FP64 DFMA throughput microbenchmark: returns achieved FLOP/s. */
bem_status bem_debug_fp64_peak(int32_t device, void* cuda_stream, double* flops_per_s);
/* mode 0: DFMA loop, 1: FP64 tensor-core mma.sync m8n8k4 loop, 2: both in one CTA. */
bem_status bem_debug_fp64_peak_ex(int32_t device, void* cuda_stream, int32_t mode, double* flops_per_s);
/* Per-kernel CUDA-event timings of the last bem_apply_multifreq issued with
 * profiling enabled (bem_op_set_profiling): ms for K1, K2up, K3, K2down, other. */
bem_status bem_op_set_profiling(bem_op op, int32_t enable);
bem_status bem_op_get_timings(bem_op op, double* ms5);
/* Work an apply of this op runs under the two underflow cutoffs (both are
 * exact to the rounding of the result: |e^{-s r}| = e^{-Re s r}, eq:fundsol P:479-482, so at
 * the strongly damped CQM frequencies the kernel underflows beyond a few mesh widths):
 *   K1 (a3): over a warp step of 32 source panels, a frequency class with Re s r_min > near_tau
 *     (default 42, env BEM_NEAR_TAU, 0 = off) is not evaluated;
 *   K3 (a5, far10): a (far block, 128-frequency tile) whose compressed fibres sum_j S(s_kj) Z[j,t]
 *     (eq:maca P:1314-1320) are bounded entrywise by far_delta / max(|s_t|, 1, 1/(4 h)) for every column t
 *     (h = the mesh's largest quadrature-node-to-centroid distance)
 *     (default far_delta = 2^-70, env BEM_FAR_SKIP_LOG2 = 70, 0 = off) is not computed.
 * far_rank_cols_*: sum over far blocks of r_b x (frequency columns), in total and under the
 * mask (equal when no mask applies); near_evals_total = 7 nnz_near n_class, near_evals_run =
 * the kernel evaluations K1 ran in the last apply issued with profiling enabled (-1: none).
 * Synchronises the device. */
typedef struct {
  int64_t far_rank_cols_total, far_rank_cols_run;
  int64_t near_evals_total, near_evals_run;
  double near_tau, far_delta;
} bem_op_work;
bem_status bem_op_get_work(bem_op op, bem_op_work* out);
/* Number of kernels one bem_apply_multifreq on this op launches. */
bem_status bem_op_launch_count(bem_op op, int32_t* n);

#ifdef __cplusplus
}
#endif
#endif /* BEM_H_ */
