// MACA assembly of the far-field coupling tensors on the device (setup step a10).
//
// Alg. 2 per admissible block b = r x c on the mode-3 unfolding
// A_b[q,l] = k(|xi_{c,nu} - xi_{r,mu}|; s_l), q = mu*p + nu (Remark P:1322-1334;
// coupling entries P:1166-1171), with the readings of DESIGN.md:
//   k_1 = 0; argmax on key(z) = re*re + im*im with the lowest index winning
//   ties; already-used slice (k) and row (q) indices are excluded (AM15);
//   C_l = 0 stops without the term; the stop rule
//   ||C_l|| ||d_l|| <= eps ||G^(l)|| uses the Gram identity
//    and is tested after the term is kept (AM13).
// Every value the ACA reads is computed with PINNED arithmetic (IEEE
// +,-,*,/,sqrt,fma only, no contraction: __d*_rn / __fma_rn intrinsics) and
// pinned reduction order (chunks of 32 summed sequentially, then left to
// right), so ranks and pivots are bit-identical to the independent CPU oracle.
// Stored per block: pivots (k_l, q_l) and Z_b = U_b^{-1} D_b^T restricted to
// the local frequencies, U_b[l][j] = d_l[k_j] (unit upper triangular), so
// that A_b ~= A_b[:,K] Z_b (eq:maca P:1314-1320 in skeleton form).
#include <algorithm>
#include <cmath>
#include <cstdio>

#include "common.cuh"

#include "pinned.cuh"
#include "zgen.cuh"

namespace bem {

namespace {

constexpr int kAcaThreads = 128;
constexpr int kMaxP = 512;         // m <= 8
constexpr int kMaxChunks = 8192;   // pp/32 upper bound for smem partials (m <= 8: 262144/32)

struct AcaArgs {
  int nfar, m, p, L, rcap, n_local;
  int ppmax, geo;  // largest unfolding row count; doubles of staged block geometry
  const int32_t* far_r;  // block row / column clusters (far or near list)
  const int32_t* far_c;
  const double* xi;
  // near blocks (combined mode): cluster ranges and cluster-ordered panel data
  const int32_t* cbegin;
  const int32_t* cend;
  const double* cen;
  const double* qn;
  const double* area;
  const double* J;
  double w[7];
  double2* Spool;                  // pivot slices V_{k_t}[b]
  unsigned long long* spool_used;
  unsigned long long spool_cap;
  int64_t* soff;
  const double2* s;
  const int32_t* local_l;
  double eps;
  double2* Cbuf;  // grid * rcap * pp
  double2* Dbuf;  // grid * rcap * L
  double2* Ebuf;  // grid * L
  double2* Pbuf;  // grid * rcap * (pp/32 + L/32 + 2): chunk partials of the batched Gram dots
  int32_t* rank;
  int32_t* pivk;
  int32_t* pivq;
  int64_t* zoff;
  double2* Zpool;  // nullable: Z_b not stored (factors-only skeleton)
  unsigned long long* pool_used;
  unsigned long long pool_cap;
  // factors-only skeleton (far blocks): F_b [r][r] row-major, F[l][j] = c_j[q_l] (j <= l, the
  // lower factor C^_b of A_b[Q,K], pivots on the diagonal) and d_l[k_j] (j > l, the unit upper U_b)
  double2* Fpool;  // nullable
  unsigned long long* fpool_used;
  unsigned long long fpool_cap;
  int64_t* foff;
  int32_t* flags;
  int32_t* next_block;
};

struct BestPair { double k; int i; };

__device__ __forceinline__ bool better(double ka, int ia, double kb, int ib) {
  return ka > kb || (ka == kb && ia < ib);
}

// block argmax of (key, index), lowest index on ties; result broadcast.
__device__ BestPair block_argmax(double k, int i, BestPair* sh) {
  for (int off = 16; off > 0; off >>= 1) {
    double ko = __shfl_down_sync(0xffffffffu, k, off);
    int io = __shfl_down_sync(0xffffffffu, i, off);
    if (better(ko, io, k, i)) { k = ko; i = io; }
  }
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) sh[w] = BestPair{k, i};
  __syncthreads();
  if (threadIdx.x == 0) {
    BestPair b = sh[0];
    for (int j = 1; j < (int)(blockDim.x >> 5); ++j)
      if (better(sh[j].k, sh[j].i, b.k, b.i)) b = sh[j];
    sh[0] = b;
  }
  __syncthreads();
  BestPair r = sh[0];
  __syncthreads();
  return r;
}

// Pinned complex reduction sum_i v(i): chunk sums (32 sequential), then left to right.
template <class F>
__device__ double2 block_psum(int n, F v, double2* part) {
  const int nch = (n + 31) >> 5;
  for (int ch = threadIdx.x; ch < nch; ch += blockDim.x) {
    double sr = 0.0, si = 0.0;
    const int e = min(n, (ch << 5) + 32);
    for (int i = ch << 5; i < e; ++i) {
      const double2 x = v(i);
      sr = __dadd_rn(sr, x.x);
      si = __dadd_rn(si, x.y);
    }
    part[ch] = make_double2(sr, si);
  }
  __syncthreads();
  __shared__ double2 tot;
  if (threadIdx.x == 0) {
    double tr = 0.0, ti = 0.0;
    for (int ch = 0; ch < nch; ++ch) { tr = __dadd_rn(tr, part[ch].x); ti = __dadd_rn(ti, part[ch].y); }
    tot = make_double2(tr, ti);
  }
  __syncthreads();
  const double2 r = tot;
  __syncthreads();
  return r;
}

template <bool NEAR>
__global__ void __launch_bounds__(kAcaThreads) aca_kernel(AcaArgs a) {
  using namespace pinned;
  extern __shared__ unsigned char smem_raw[];
  const int p = a.p, m = a.m, L = a.L;
  const int half = L / 2;
  // shared layout
  double* xr = (double*)smem_raw;             // far: p*3 row nodes; near: 3 per row panel
  double* xc = xr + 3 * p;                    // far: p*3 column nodes
  double2* part = (double2*)(xr + a.geo);     // max(ppmax, L)/32 + 1
  const int nchmax = (max(a.ppmax, L) + 31) / 32 + 1;
  double2* dk = part + nchmax;                // rcap: D[j][k]
  double2* cq = dk + a.rcap;                  // rcap: C[j][q*]
  unsigned* usedq = (unsigned*)(cq + a.rcap); // ppmax bits
  unsigned* usedk = usedq + (a.ppmax + 31) / 32;   // L bits
  double2* gcs = (double2*)(((uintptr_t)(usedk + (L + 31) / 32) + 15) & ~(uintptr_t)15);  // rcap: <c_j, c>
  double2* gds = gcs + a.rcap;                                                          // rcap: <d_j, d>
  __shared__ BestPair red[kAcaThreads / 32];
  __shared__ int s_blk, s_k, s_stop;
  __shared__ double s_nrm2;
  __shared__ long long s_off;

  double2* Cb = a.Cbuf + (size_t)blockIdx.x * a.rcap * a.ppmax;
  double2* Db = a.Dbuf + (size_t)blockIdx.x * a.rcap * L;
  double2* Eb = a.Ebuf + (size_t)blockIdx.x * L;

  for (;;) {
    if (threadIdx.x == 0) s_blk = atomicAdd(a.next_block, 1);
    __syncthreads();
    const int b = s_blk;
    __syncthreads();
    if (b >= a.nfar) break;
    const int rc = a.far_r[b], cc = a.far_c[b];
    int pp, nr = 0, nc = 0, r0 = 0, c0 = 0;
    if constexpr (NEAR) {
      r0 = a.cbegin[rc]; nr = a.cend[rc] - r0;
      c0 = a.cbegin[cc]; nc = a.cend[cc] - c0;
      pp = nr * nc;
      for (int i = threadIdx.x; i < 3 * nr; i += blockDim.x) xr[i] = a.cen[3 * (size_t)r0 + i];
      double* gc = xr + 3 * nr;  // per column panel: 21 node coordinates, area, J
      for (int i = threadIdx.x; i < 23 * nc; i += blockDim.x) {
        const int j = i / 23, e = i - 23 * j;
        gc[i] = e < 21 ? a.qn[21 * (size_t)(c0 + j) + e] : (e == 21 ? a.area[c0 + j] : a.J[c0 + j]);
      }
    } else {
      pp = p * p;
      for (int i = threadIdx.x; i < p; i += blockDim.x) {
        const double* xir = a.xi + (size_t)rc * 3 * m;
        const double* xic = a.xi + (size_t)cc * 3 * m;
        xr[3 * i + 0] = xir[i % m]; xr[3 * i + 1] = xir[m + (i / m) % m]; xr[3 * i + 2] = xir[2 * m + i / (m * m)];
        xc[3 * i + 0] = xic[i % m]; xc[3 * i + 1] = xic[m + (i / m) % m]; xc[3 * i + 2] = xic[2 * m + i / (m * m)];
      }
    }
    const int rmax = min(L, pp);
    for (int i = threadIdx.x; i < (pp + 31) / 32; i += blockDim.x) usedq[i] = 0u;
    for (int i = threadIdx.x; i < (L + 31) / 32; i += blockDim.x) usedk[i] = 0u;
    if (threadIdx.x == 0) { s_k = 0; s_nrm2 = 0.0; s_stop = 0; }
    __syncthreads();

    auto entry = [&](int q, int l) -> double2 {
      const bool mir = l > half;
      const int ll = mir ? L - l : l;
      double2 v;
      if constexpr (NEAR) {
        const int i = q / nc, j = q - i * nc;
        v = near_entry(&xr[3 * i], &xr[3 * nr + 23 * j], r0 + i == c0 + j, a.s[ll].x, a.s[ll].y, a.w);
      } else {
        const double r = dist(&xr[3 * (q / p)], &xc[3 * (q % p)]);
        v = kernel(r, a.s[ll].x, a.s[ll].y);
      }
      if (mir) v.y = -v.y;
      return v;
    };

    int ell = 0;
    bool overflow = false;
    for (;;) {
      const int k = s_k;
      if (ell == a.rcap) { overflow = true; break; }
      for (int j = threadIdx.x; j < ell; j += blockDim.x) dk[j] = Db[(size_t)j * L + k];
      __syncthreads();
      // residual slice c = A[:,k] - sum_j d_j[k] c_j
      double bk = -1.0;
      int bi = 0x7fffffff;
      double2* c = Cb + (size_t)ell * pp;
      for (int q = threadIdx.x; q < pp; q += blockDim.x) {
        double2 acc = entry(q, k);
#pragma unroll 8
        for (int j = 0; j < ell; ++j) acc = csub(acc, cmul(dk[j], Cb[(size_t)j * pp + q]));  // loads run ahead
        c[q] = acc;
        if (!((usedq[q >> 5] >> (q & 31)) & 1u)) {
          const double kk = key(acc);
          if (kk > bk) { bk = kk; bi = q; }
        }
      }
      const BestPair bq = block_argmax(bk, bi, red);
      if (bq.i == 0x7fffffff || !(bq.k > 0.0)) break;  // C_l = 0: stop without the term
      const int qs = bq.i;
      for (int j = threadIdx.x; j < ell; j += blockDim.x) cq[j] = Cb[(size_t)j * pp + qs];
      __syncthreads();
      const double2 piv = c[qs];
      // residual fibre e = A[q*,:] - sum_j c_j[q*] d_j ; d = e / piv
      double2* d = Db + (size_t)ell * L;
      double be = -1.0;
      int bl = 0x7fffffff;
      for (int l = threadIdx.x; l < L; l += blockDim.x) {
        double2 acc = entry(qs, l);
#pragma unroll 8
        for (int j = 0; j < ell; ++j) acc = csub(acc, cmul(cq[j], Db[(size_t)j * L + l]));
        Eb[l] = acc;
        d[l] = cdiv(acc, piv);
        if (l != k && !((usedk[l >> 5] >> (l & 31)) & 1u)) {
          const double kk = key(acc);
          if (kk > be) { be = kk; bl = l; }
        }
      }
      __syncthreads();
      const double nc2 = block_psum(pp, [&](int q) { const double v = key(c[q]); return make_double2(v, 0.0); }, part).x;
      const double nd2 = block_psum(L, [&](int l) { const double v = key(d[l]); return make_double2(v, 0.0); }, part).x;
      // Gram cross terms <c_j, c> <d_j, d> for all j < ell at once: every dot product keeps the
      // pinned order (sequential within chunks of 32, then left to right over the chunk sums),
      // but the (j, chunk) partials of all j are computed in one parallel pass (2 barriers
      // instead of 6 per j; the per-j serial tails run in parallel over j)
      double cross = 0.0;
      if (ell > 0) {
        const int nchc = (pp + 31) >> 5, nchd = (L + 31) >> 5;
        double2* Pc = a.Pbuf + (size_t)blockIdx.x * a.rcap * ((a.ppmax + 31) / 32 + nchd);
        double2* Pd = Pc + (size_t)a.rcap * nchc;
        for (int w = threadIdx.x; w < ell * nchc; w += blockDim.x) {
          const int j = w / nchc, ch = w - j * nchc;
          const double2* cj = Cb + (size_t)j * pp;
          double sr = 0.0, si = 0.0;
          const int e = min(pp, (ch << 5) + 32);
#pragma unroll 8
          for (int i = ch << 5; i < e; ++i) {
            const double2 x = cmulconj(cj[i], c[i]);
            sr = __dadd_rn(sr, x.x);
            si = __dadd_rn(si, x.y);
          }
          Pc[(size_t)j * nchc + ch] = make_double2(sr, si);
        }
        for (int w = threadIdx.x; w < ell * nchd; w += blockDim.x) {
          const int j = w / nchd, ch = w - j * nchd;
          const double2* dj = Db + (size_t)j * L;
          double sr = 0.0, si = 0.0;
          const int e = min(L, (ch << 5) + 32);
#pragma unroll 8
          for (int i = ch << 5; i < e; ++i) {
            const double2 x = cmulconj(dj[i], d[i]);
            sr = __dadd_rn(sr, x.x);
            si = __dadd_rn(si, x.y);
          }
          Pd[(size_t)j * nchd + ch] = make_double2(sr, si);
        }
        __syncthreads();
        for (int j = threadIdx.x; j < ell; j += blockDim.x) {
          double tr = 0.0, ti = 0.0;
          for (int ch = 0; ch < nchc; ++ch) { tr = __dadd_rn(tr, Pc[(size_t)j * nchc + ch].x); ti = __dadd_rn(ti, Pc[(size_t)j * nchc + ch].y); }
          gcs[j] = make_double2(tr, ti);
          tr = 0.0; ti = 0.0;
          for (int ch = 0; ch < nchd; ++ch) { tr = __dadd_rn(tr, Pd[(size_t)j * nchd + ch].x); ti = __dadd_rn(ti, Pd[(size_t)j * nchd + ch].y); }
          gds[j] = make_double2(tr, ti);
        }
        __syncthreads();
        for (int j = 0; j < ell; ++j)  // every thread, same order: the value is only used by thread 0
          cross = add(cross, sub(mul(gcs[j].x, gds[j].x), mul(gcs[j].y, gds[j].y)));
      }
      const BestPair bn = block_argmax(be, bl, red);
      if (threadIdx.x == 0) {
        double nrm2 = add(s_nrm2, add(mul(nc2, nd2), mul(2.0, cross)));
        if (nrm2 < 0.0) nrm2 = 0.0;
        s_nrm2 = nrm2;
        a.pivk[(size_t)b * a.rcap + ell] = k;
        a.pivq[(size_t)b * a.rcap + ell] = qs;
        usedq[qs >> 5] |= 1u << (qs & 31);
        usedk[k >> 5] |= 1u << (k & 31);
        const int rank = ell + 1;
        const bool stop = mul(__dsqrt_rn(nc2), __dsqrt_rn(nd2)) <= mul(a.eps, __dsqrt_rn(nrm2)) || rank == rmax ||
                          bn.i == 0x7fffffff;
        s_stop = stop ? 1 : 0;
        if (!stop) s_k = bn.i;
      }
      __syncthreads();
      ++ell;
      if (s_stop) break;
    }
    // write rank, allocate Z (and F), back substitution Z = U^{-1} D^T on local columns
    __shared__ long long s_foff;
    if (threadIdx.x == 0) {
      s_foff = -1;
      if (overflow) {
        atomicOr(a.flags, 1);
        a.rank[b] = -1;
        a.zoff[b] = -1;
        s_off = -1;
      } else {
        a.rank[b] = ell;
        s_off = -1;
        if (a.Zpool != nullptr) {
          const unsigned long long need = (unsigned long long)ell * (unsigned long long)a.n_local;
          const unsigned long long off = atomicAdd(a.pool_used, need);
          if (off + need > a.pool_cap) atomicOr(a.flags, 2); else s_off = (long long)off;
        }
        a.zoff[b] = s_off;
        if (a.Fpool != nullptr) {
          const unsigned long long need = (unsigned long long)ell * (unsigned long long)ell;
          const unsigned long long fo = atomicAdd(a.fpool_used, need);
          if (fo + need > a.fpool_cap) atomicOr(a.flags, 8); else s_foff = (long long)fo;
          a.foff[b] = s_foff;
        }
      }
    }
    __syncthreads();
    const long long off = s_off;
    if (s_foff >= 0) {
      const int r = ell;
      const int32_t* kp = a.pivk + (size_t)b * a.rcap;
      const int32_t* qp = a.pivq + (size_t)b * a.rcap;
      for (int idx = threadIdx.x; idx < r * r; idx += blockDim.x) {
        const int i = idx / r, j = idx - i * r;
        a.Fpool[s_foff + idx] = j <= i ? Cb[(size_t)j * pp + qp[i]] : Db[(size_t)i * L + kp[j]];
      }
    }
    if (off >= 0) {
      const int r = ell;
      const int32_t* kp = a.pivk + (size_t)b * a.rcap;
      for (int t = threadIdx.x; t < a.n_local; t += blockDim.x) {
        const int lt = a.local_l[t];
        for (int l = r - 1; l >= 0; --l) {
          double2 acc = Db[(size_t)l * L + lt];
          for (int j = l + 1; j < r; ++j)
            acc = csub(acc, cmul(Db[(size_t)l * L + kp[j]], a.Zpool[off + (size_t)j * a.n_local + t]));
          a.Zpool[off + (size_t)l * a.n_local + t] = acc;
        }
      }
    }
    if constexpr (NEAR) {
      // pivot slices V_{k_t}[b] (raw tensor columns, the apply's C_b), re-evaluated
      __shared__ long long s_soff;
      if (threadIdx.x == 0) {
        s_soff = -1;
        if (off >= 0) {
          const unsigned long long need = (unsigned long long)ell * (unsigned long long)pp;
          const unsigned long long so = atomicAdd(a.spool_used, need);
          if (so + need > a.spool_cap) atomicOr(a.flags, 4); else s_soff = (long long)so;
        }
        a.soff[b] = s_soff;
      }
      __syncthreads();
      const long long so = s_soff;
      if (so >= 0) {
        const int32_t* kp = a.pivk + (size_t)b * a.rcap;
        for (int idx = threadIdx.x; idx < ell * pp; idx += blockDim.x) {
          const int t = idx / pp, q = idx - t * pp;
          a.Spool[so + idx] = entry(q, kp[t]);
        }
      }
    }
    __syncthreads();
  }
}

// Stored-Z skeleton (the default when it fits): Z_b[:, t] for every far block and local
// frequency t, regenerated from the factors F_b (zgen.cuh; bit-identical to the ACA's own
// back substitution).  One CTA per block (grid-stride), threads over the local columns.
__global__ void __launch_bounds__(256) zgen_all_kernel(zgen::Src a, int nfar, const int32_t* rank, const int32_t* local_l,
                                                    int n_local, const int64_t* zoff, double2* Z, int cap) {
  extern __shared__ double2 work[];
  for (int b = blockIdx.x; b < nfar; b += gridDim.x) {
    double2* Zb = Z + zoff[b];
    zgen::block_columns(
        a, b, rank[b], 0, n_local, [&](int t) { return local_l[t]; }, work, cap,
        [&](int j, int t, double2 v) { Zb[(int64_t)j * n_local + t] = v; });
  }
}

__global__ void debug_pinned_kernel(const double* x, int64_t n, double* e, double* sn, double* cs) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  e[i] = pinned::exp_(x[i]);
  pinned::sincos_(x[i], &sn[i], &cs[i]);
}

}  // namespace
}  // namespace bem

using namespace bem;

namespace {
// near = false: far blocks (P+, coupling tensors); near = true: near blocks (P-,
// combined mode), whose pivot slices are stored as well.
bem_status run_aca(Op& op, cudaStream_t st, bool near, bool store_z, const std::vector<int32_t>* subset = nullptr) {
  Tree& t = *op.tree;
  const int nblk = subset ? (int)subset->size() : near ? (int)t.near_r.size() : (int)t.far_r.size();
  DBuf<int32_t> sub_r, sub_c;  // far blocks of `subset` only (diagnostic: bem_debug_aca_blocks)
  if (subset) {
    std::vector<int32_t> hr, hc;
    for (int b : *subset) { hr.push_back(t.far_r[b]); hc.push_back(t.far_c[b]); }
    BEM_CK(sub_r.upload(hr));
    BEM_CK(sub_c.upload(hc));
  }
  std::vector<int32_t>& ranks_out = near ? op.nranks : op.ranks;
  ranks_out.assign(nblk, 0);
  if (nblk == 0) return BEM_OK;
  const int p = t.p, L = op.L;
  const int ppmax = near ? t.max_leaf * t.max_leaf : p * p;
  const int geo = near ? 26 * t.max_leaf : 6 * p;
  int nsm = 148;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, t.device);
  // scratch rank cap and Z-pool size: generous first guesses (a retry recomputes the
  // whole ACA: config 5 hit both the old 96 rank cap and the 40-per-block pool
  // estimate), the pool is shrunk to its exact size afterwards
  int rcap = std::min(std::min(L, ppmax), 128);
  const bool store_f = !near && !subset;  // factors-only skeleton of the far blocks (always kept: small)
  unsigned long long cap = store_z ? (unsigned long long)nblk * 64ull * (unsigned long long)op.n_local : 0ull;
  unsigned long long fcap = store_f ? (unsigned long long)nblk * 48ull * 48ull : 0ull;
  unsigned long long scap = 0;
  if (near) {
    scap = 0;
    for (int b = 0; b < nblk; ++b)
      scap += 40ull * (unsigned long long)(t.end[t.near_r[b]] - t.begin[t.near_r[b]]) *
              (unsigned long long)(t.end[t.near_c[b]] - t.begin[t.near_c[b]]);
  }
  {
    size_t fr = 0, tot = 0;
    if (cudaMemGetInfo(&fr, &tot) == cudaSuccess) {
      const size_t scratch = (size_t)std::max(1, std::min(nblk, nsm * op.aca_ctas_per_sm)) * rcap * ((size_t)ppmax + L) * 16;
      const unsigned long long lim = fr > scratch ? (unsigned long long)((fr - scratch) * 0.7 / 16) : 0ull;
      if (lim > 0 && cap + scap + fcap > lim) {
        const double f = (double)lim / (double)(cap + scap + fcap);
        cap = (unsigned long long)(cap * f);
        scap = (unsigned long long)(scap * f);
        fcap = (unsigned long long)(fcap * f);
      }
    }
  }
  DBuf<int32_t> flags, counter;
  DBuf<unsigned long long> used;
  BEM_CK(flags.alloc(1));
  BEM_CK(counter.alloc(1));
  BEM_CK(used.alloc(3));
  DBuf<int32_t>& d_rank = near ? op.d_nrank : op.d_rank;
  DBuf<int32_t>& d_pivk = near ? op.d_npivk : op.d_pivk;
  DBuf<int32_t>& d_pivq = near ? op.d_npivq : op.d_pivq;
  DBuf<int64_t>& d_zoff = near ? op.d_nzoff : op.d_zoff;
  DBuf<double>& d_Z = near ? op.d_nZ : op.d_Z;
  BEM_CK(d_rank.alloc(nblk));
  BEM_CK(d_zoff.alloc(nblk));
  if (store_f) BEM_CK(op.d_foff.alloc(nblk));
  if (near) BEM_CK(op.d_nsoff.alloc(nblk));
  std::vector<double> wq(7);
  {
    const double r15 = std::sqrt(15.0);
    const double w1 = (155.0 + r15) / 1200.0, w2 = (155.0 - r15) / 1200.0;
    const double W[7] = {9.0 / 40.0, w1, w1, w1, w2, w2, w2};  // the 7-point rule of host.cu (C1)
    for (int q = 0; q < 7; ++q) wq[q] = W[q];
  }
  for (int attempt = 0; attempt < 8; ++attempt) {
    const int grid = std::max(1, std::min(nblk, nsm * op.aca_ctas_per_sm));
    DBuf<double> Cbuf, Dbuf, Ebuf, Pbuf;
    BEM_CK(Pbuf.alloc((size_t)grid * rcap * ((ppmax + 31) / 32 + (L + 31) / 32) * 2));
    BEM_CK(Cbuf.alloc((size_t)grid * rcap * ppmax * 2));
    BEM_CK(Dbuf.alloc((size_t)grid * rcap * L * 2));
    BEM_CK(Ebuf.alloc((size_t)grid * L * 2));
    BEM_CK(d_pivk.alloc((size_t)nblk * rcap));
    BEM_CK(d_pivq.alloc((size_t)nblk * rcap));
    BEM_CK(d_Z.alloc((size_t)cap * 2));
    if (store_f) BEM_CK(op.d_F.alloc((size_t)fcap * 2));
    if (near) BEM_CK(op.d_nS.alloc((size_t)scap * 2));
    BEM_CK(cudaMemsetAsync(flags.p, 0, sizeof(int32_t), st));
    BEM_CK(cudaMemsetAsync(counter.p, 0, sizeof(int32_t), st));
    BEM_CK(cudaMemsetAsync(used.p, 0, 3 * sizeof(unsigned long long), st));
    AcaArgs a{};
    a.nfar = nblk; a.m = t.m; a.p = p; a.L = L; a.rcap = rcap; a.n_local = op.n_local;
    a.ppmax = ppmax; a.geo = geo;
    a.far_r = subset ? sub_r.p : near ? t.d_near_r.p : t.d_far_r.p;
    a.far_c = subset ? sub_c.p : near ? t.d_near_c.p : t.d_far_c.p;
    a.xi = t.d_xi.p;
    a.cbegin = t.d_begin.p; a.cend = t.d_end.p; a.cen = t.d_cen.p; a.qn = t.d_qn.p; a.area = t.d_area.p;
    a.J = t.d_J.p;
    for (int q = 0; q < 7; ++q) a.w[q] = wq[q];
    a.Spool = near ? (double2*)op.d_nS.p : nullptr; a.spool_used = used.p + 1; a.spool_cap = scap;
    a.soff = near ? op.d_nsoff.p : nullptr;
    a.s = (const double2*)op.d_s.p; a.local_l = op.d_local_l.p; a.eps = op.eps;
    a.Cbuf = (double2*)Cbuf.p; a.Dbuf = (double2*)Dbuf.p; a.Ebuf = (double2*)Ebuf.p; a.Pbuf = (double2*)Pbuf.p;
    a.rank = d_rank.p; a.pivk = d_pivk.p; a.pivq = d_pivq.p; a.zoff = d_zoff.p;
    a.Zpool = store_z ? (double2*)d_Z.p : nullptr; a.pool_used = used.p; a.pool_cap = cap; a.flags = flags.p;
    a.Fpool = store_f ? (double2*)op.d_F.p : nullptr; a.fpool_used = used.p + 2; a.fpool_cap = fcap;
    a.foff = store_f ? op.d_foff.p : nullptr;
    a.next_block = counter.p;
    const int nchmax = (std::max(ppmax, L) + 31) / 32 + 1;
    const size_t smem = sizeof(double) * geo + sizeof(double2) * (nchmax + 2 * rcap) +
                        sizeof(unsigned) * ((ppmax + 31) / 32 + (L + 31) / 32) + 64 + sizeof(double2) * 2 * rcap + 16;
    if (near) {
      BEM_CK(cudaFuncSetAttribute(aca_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      aca_kernel<true><<<grid, kAcaThreads, smem, st>>>(a);
    } else {
      BEM_CK(cudaFuncSetAttribute(aca_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      aca_kernel<false><<<grid, kAcaThreads, smem, st>>>(a);
    }
    BEM_CK(cudaGetLastError());
    int32_t hflags = 0;
    unsigned long long hused[3] = {0, 0, 0};
    BEM_CK(cudaMemcpyAsync(&hflags, flags.p, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    BEM_CK(cudaMemcpyAsync(hused, used.p, 3 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
    BEM_CK(cudaStreamSynchronize(st));
    if (hflags & 1) {  // a rank reached the scratch capacity: grow and redo
      rcap = std::min(std::min(L, ppmax), rcap * 2);
      continue;
    }
    if (hflags & 14) {  // Z / slice / factor pool too small: exact sizes are now known
      if (hflags & 2) cap = hused[0];
      if (hflags & 4) scap = hused[1];
      if (hflags & 8) fcap = hused[2];
      continue;
    }
    if (near) op.nrcap = rcap; else op.rcap = rcap;
    BEM_CK(cudaMemcpy(ranks_out.data(), d_rank.p, sizeof(int32_t) * nblk, cudaMemcpyDeviceToHost));
    auto shrink = [&](DBuf<double>& buf, unsigned long long used_n, unsigned long long cap_n) -> cudaError_t {
      if (!(used_n < cap_n && (cap_n - used_n) * 16ull > (64ull << 20))) return cudaSuccess;
      DBuf<double> z;
      cudaError_t e = z.alloc((size_t)std::max<unsigned long long>(used_n, 1) * 2);
      if (e != cudaSuccess) return e;
      e = cudaMemcpyAsync(z.p, buf.p, (size_t)used_n * 16, cudaMemcpyDeviceToDevice, st);
      if (e == cudaSuccess) e = cudaStreamSynchronize(st);
      if (e == cudaSuccess) buf = std::move(z);
      return e;
    };
    BEM_CK(shrink(d_Z, hused[0], cap));
    if (store_f) BEM_CK(shrink(op.d_F, hused[2], fcap));
    if (!near) op.z_stored = store_z;
    if (near) BEM_CK(shrink(op.d_nS, hused[1], scap));
    return BEM_OK;
  }
  set_error("bem_assemble_h2_aca: ACA did not fit after repeated growth");
  return BEM_ENOMEM;
}
}  // namespace

extern "C" bem_status bem_assemble_h2_aca(bem_tree th, const bem_c128* s, int32_t L, const int32_t* local_l,
                                          int32_t n_local, double aca_eps, int32_t mode, void* cuda_stream,
                                          bem_op* out) {
  BEM_REQ(th && out, "bem_assemble_h2_aca: NULL tree/out");
  BEM_REQ(s != nullptr && L >= 1, "bem_assemble_h2_aca: need s and L >= 1");
  BEM_REQ(aca_eps > 0.0, "bem_assemble_h2_aca: aca_eps must be > 0");
  const int skel = mode & (BEM_SKEL_Z | BEM_SKEL_FACTORS);
  BEM_REQ((mode & ~(0xff | BEM_SKEL_Z | BEM_SKEL_FACTORS)) == 0 && skel != (BEM_SKEL_Z | BEM_SKEL_FACTORS),
          "bem_assemble_h2_aca: bad mode flags 0x%x", mode);
  mode &= 0xff;
  BEM_REQ(mode == BEM_MODE_H2ACA || mode == BEM_MODE_H2ONLY || mode == BEM_MODE_DENSE || mode == BEM_MODE_COMBINED,
          "bem_assemble_h2_aca: unknown mode %d", mode);
  BEM_REQ(!(mode == BEM_MODE_COMBINED && skel == BEM_SKEL_FACTORS),
          "bem_assemble_h2_aca: BEM_MODE_COMBINED keeps the stored Z (the MoT weights read it)");
  // the operator evaluates l > L/2 as the conjugate of L - l (ACA mirroring, conjugate
  // frequency classes of K1 / K3'): s must be exactly conjugation-symmetric
  for (int l = 1; 2 * l < L; ++l)
    BEM_REQ(s[L - l].re == s[l].re && s[L - l].im == -s[l].im,
            "bem_assemble_h2_aca: s[%d] != conj(s[%d]) (s must satisfy s_{L-l} = conj(s_l), as cqm_frequencies gives)",
            L - l, l);
  *out = nullptr;
  Tree& t = th->t;
  if (t.device < 0) {
    set_error("bem_assemble_h2_aca: tree was built host-only (device = -1)");
    return BEM_ESTATE;
  }
  std::vector<int32_t> loc;
  if (local_l == nullptr) {
    loc.resize(L);
    for (int l = 0; l < L; ++l) loc[l] = l;
  } else {
    BEM_REQ(n_local >= 1 && n_local <= L, "bem_assemble_h2_aca: n_local out of range");
    loc.assign(local_l, local_l + n_local);
    std::vector<char> seen(L, 0);
    for (int v : loc) {
      BEM_REQ(v >= 0 && v < L, "bem_assemble_h2_aca: local index %d out of range", v);
      BEM_REQ(!seen[v], "bem_assemble_h2_aca: duplicate local index %d", v);
      seen[v] = 1;
    }
  }
  DeviceGuard dg(t.device);
  Nvtx nv("a10 bem_assemble_h2_aca");
  cudaStream_t st = (cudaStream_t)cuda_stream;
  bem_op_s* h = new bem_op_s();
  Op& op = h->o;
  op.tree = &t; op.L = L; op.n_local = (int)loc.size(); op.mode = mode; op.eps = aca_eps; op.local_l = loc;
  if (const char* e = getenv("BEM_FAR_GENERIC")) op.force_generic = atoi(e) != 0;
  if (const char* e = getenv("BEM_FAR_KERNEL")) op.far_kernel = atoi(e);
  if (const char* e = getenv("BEM_FAR8_KC")) op.far8_kc = atoi(e);
  if (const char* e = getenv("BEM_FAR8_M3")) op.far8_m3 = atoi(e) != 0;
  if (const char* e = getenv("BEM_FAR8_DT")) op.far8_dt = atoi(e) != 0;
  if (const char* e = getenv("BEM_SOLVE_MASK")) op.use_solve_mask = atoi(e) != 0;
  if (const char* e = getenv("BEM_K1_FUSE")) op.k1_fuse = atoi(e) != 0;
  if (const char* e = getenv("BEM_K1_WARPS")) op.k1_warps = std::min(3, std::max(1, atoi(e)));
  if (const char* e = getenv("BEM_FAR10_PERSIST")) op.far10_persist = atoi(e) != 0;
  if (const char* e = getenv("BEM_NEAR_TAU")) op.near_tau = atof(e);  // 0: no K1 underflow cutoff
  if (const char* e = getenv("BEM_FAR_SKIP_LOG2")) op.far_delta = atoi(e) != 0 ? ldexp(1.0, -abs(atoi(e))) : 0.0;  // 0: no mask
  auto fail = [&](bem_status stt) { delete h; return stt; };
  std::vector<double> sh(2 * (size_t)L);
  for (int l = 0; l < L; ++l) { sh[2 * l] = s[l].re; sh[2 * l + 1] = s[l].im; }
  if (op.d_s.upload(sh) != cudaSuccess || op.d_local_l.upload(loc) != cudaSuccess) {
    set_error("bem_assemble_h2_aca: upload failed");
    return fail(BEM_ECUDA);
  }
  // near-field frequency classes: pair (l, L-l) when both are local
  std::vector<int32_t> pos(L, -1), c1, c2;
  for (int i = 0; i < op.n_local; ++i) pos[loc[i]] = i;
  std::vector<char> done(op.n_local, 0);
  for (int i = 0; i < op.n_local; ++i) {
    if (done[i]) continue;
    const int l = loc[i], lm = (L - l) % L;
    const int j = pos[lm];
    done[i] = 1;
    if (lm != l && j >= 0 && !done[j]) {
      // class frequency = the one with l <= L/2 (evaluated), partner = conjugate
      if (l <= L / 2) { c1.push_back(i); c2.push_back(j); } else { c1.push_back(j); c2.push_back(i); }
      done[j] = 1;
    } else {
      c1.push_back(i); c2.push_back(-1);
    }
  }
  op.n_class = (int)c1.size();
  if (op.d_class_t1.upload(c1) != cudaSuccess || op.d_class_t2.upload(c2) != cudaSuccess) {
    set_error("bem_assemble_h2_aca: upload failed");
    return fail(BEM_ECUDA);
  }
  if (mode == BEM_MODE_H2ACA || mode == BEM_MODE_COMBINED) {
    // MACA with the factors F_b only; then either the coefficients Z_b of the local
    // frequencies are stored (regenerated once from F_b here), or K3 regenerates each
    // block's Z tile in its prologue (factors-only skeleton): the
    // default stores Z when it takes at most a third of the free device memory
    bem_status rs = run_aca(op, st, false, false);
    if (rs != BEM_OK) return fail(rs);
    int64_t zrows = 0;
    for (int v : op.ranks) zrows += v;
    const size_t zbytes = (size_t)zrows * op.n_local * 16;
    bool store = skel == BEM_SKEL_Z || mode == BEM_MODE_COMBINED;
    if (skel == 0) {
      size_t fr = 0, tot = 0;
      store = cudaMemGetInfo(&fr, &tot) == cudaSuccess && zbytes <= fr / 3;
    }
    if (store) {
      std::vector<int64_t> zo(op.ranks.size());
      int64_t acc = 0;
      for (size_t b = 0; b < zo.size(); ++b) { zo[b] = acc; acc += (int64_t)op.ranks[b] * op.n_local; }
      if (op.d_zoff.upload(zo) != cudaSuccess || op.d_Z.alloc(std::max<size_t>(1, (size_t)acc * 2)) != cudaSuccess) {
        set_error("bem_assemble_h2_aca: stored Z (%.2f GB) does not fit", zbytes / 1e9);
        return fail(BEM_ENOMEM);
      }
      zgen::Src zs{};
      zs.m = t.m; zs.p = t.p; zs.L = L; zs.far_r = t.d_far_r.p; zs.far_c = t.d_far_c.p; zs.xi = t.d_xi.p;
      zs.s = (const double2*)op.d_s.p; zs.pivk = op.d_pivk.p; zs.pivq = op.d_pivq.p; zs.foff = op.d_foff.p;
      zs.F = (const double2*)op.d_F.p; zs.rcap = op.rcap;
      const int nfar = (int)op.ranks.size();
      if (nfar > 0) {
        constexpr int kSm = 64 * 1024;
        cudaFuncSetAttribute(zgen_all_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSm);
        zgen_all_kernel<<<std::min(nfar, 148 * 3), 256, kSm, st>>>(zs, nfar, op.d_rank.p, op.d_local_l.p, op.n_local,
                                                                    op.d_zoff.p, (double2*)op.d_Z.p,
                                                                    kSm / (int)sizeof(double2));
        if (cudaGetLastError() != cudaSuccess) {
          set_error("bem_assemble_h2_aca: zgen launch failed");
          return fail(BEM_ECUDA);
        }
      }
    }
    op.z_stored = store;
  }
  if (mode == BEM_MODE_COMBINED) {
    if (t.max_leaf > 64) {  // K1m stages 3 slice buffers of 32 x max_leaf complex per CTA
      set_error("bem_assemble_h2_aca: BEM_MODE_COMBINED needs leaves of at most 64 panels (largest: %d)", t.max_leaf);
      return fail(BEM_EINVAL);
    }
    bem_status rs = run_aca(op, st, true, true);
    if (rs != BEM_OK) return fail(rs);
    // K1m launch order: row leaves by descending near-field MACA work (LPT)
    std::vector<std::pair<int64_t, int32_t>> w;
    for (int li = 0; li < t.n_leaves; ++li) {
      int64_t c = 0;
      for (int bi = t.nb_ptr[li]; bi < t.nb_ptr[li + 1]; ++bi) {
        const int b = t.nb_sorted[bi];
        c += (int64_t)op.nranks[b] * (t.end[t.near_c[b]] - t.begin[t.near_c[b]]);
      }
      w.push_back({-c, li});
    }
    std::stable_sort(w.begin(), w.end());
    std::vector<int32_t> ord;
    for (auto& e : w) ord.push_back(e.second);
    if (op.d_nm_order.upload(ord) != cudaSuccess) {
      set_error("bem_assemble_h2_aca: upload failed");
      return fail(BEM_ECUDA);
    }
  }
  if (mode != BEM_MODE_DENSE && !t.far_r.empty()) {
    std::vector<std::pair<int64_t, int32_t>> w;
    for (int c = 0; c < t.C; ++c) {
      int64_t cost = 0;
      for (int bi = t.far_ptr[c]; bi < t.far_ptr[c + 1]; ++bi)
        cost += op.ranks.empty() ? 1 : op.ranks[t.far_sorted[bi]] + 1;
      if (t.far_ptr[c + 1] > t.far_ptr[c]) w.push_back({-cost, c});
    }
    std::sort(w.begin(), w.end());
    std::vector<int32_t> rows;
    for (auto& e : w) rows.push_back(e.second);
    op.n_far_rows = (int)rows.size();
    if (op.d_far_rows.upload(rows) != cudaSuccess) {
      set_error("bem_assemble_h2_aca: upload failed");
      return fail(BEM_ECUDA);
    }
    {
      // split rows into block-range segments of bounded cost (load balance of K3)
      int nsm = 148;
      cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, t.device);
      // block weight: ACA rank (H2ACA: r_b slice products) or 1 (H2ONLY: one p x p evaluation per frequency)
      const bool aca = mode == BEM_MODE_H2ACA || mode == BEM_MODE_COMBINED;
      auto wgt = [&](int b) -> int64_t { return aca ? op.ranks[b] : 1; };
      int64_t total = 0;
      for (int b = 0; b < (int)t.far_r.size(); ++b) total += wgt(b);
      int64_t cap = std::max<int64_t>(1, total / (8 * (int64_t)nsm));  // ~8 segments per SM (r01: config 2 K3 9.02 -> 8.77 ms vs 4 per SM)
      // H2ONLY: the CTA's 4 warps take every 4th block of a segment, so keep >= 16 blocks
      // per segment (<= 25% warp imbalance at the end-of-CTA barrier); the class tiles
      // already give many CTAs
      if (!aca) cap = std::max<int64_t>(cap, std::max<int64_t>(16, total / (2 * (int64_t)nsm)));
      if (const char* e = getenv("BEM_SEG_CAP")) cap = std::max<int64_t>(1, atoll(e));
      struct Seg { int64_t cost; int row, bi0, bi1, slot; };
      std::vector<Seg> segs;
      std::vector<int32_t> srows, sptr{0};
      for (int c = 0; c < t.C; ++c) {
        const int b0 = t.far_ptr[c], b1 = t.far_ptr[c + 1];
        if (b1 == b0) continue;
        int start = b0;
        int64_t acc = 0;
        for (int bi = b0; bi < b1; ++bi) {
          const int64_t w = wgt(t.far_sorted[bi]);
          if (acc > 0 && acc + w > cap) {
            segs.push_back({acc, c, start, bi, (int)segs.size()});
            start = bi;
            acc = 0;
          }
          acc += w;
        }
        segs.push_back({acc, c, start, b1, (int)segs.size()});
        srows.push_back(c);
        sptr.push_back((int32_t)segs.size());
      }
      std::vector<Seg> order = segs;
      std::stable_sort(order.begin(), order.end(), [](const Seg& x, const Seg& y) { return x.cost > y.cost; });
      std::vector<int32_t> flat;
      for (auto& sg : order) { flat.push_back(sg.row); flat.push_back(sg.bi0); flat.push_back(sg.bi1); flat.push_back(sg.slot); }
      op.n_segs = (int)segs.size();
      op.n_seg_rows = (int)srows.size();
      if (op.d_segs.upload(flat) != cudaSuccess || op.d_seg_rows.upload(srows) != cudaSuccess ||
          op.d_seg_ptr.upload(sptr) != cudaSuccess ||
          op.d_part.alloc((size_t)op.n_segs * op.n_local * t.p * 2) != cudaSuccess) {
        set_error("bem_assemble_h2_aca: segment upload/allocation failed");
        return fail(BEM_ENOMEM);
      }
    }
  }
  if (mode == BEM_MODE_DENSE) {
    std::vector<int32_t> jb(t.n_leaves, 0), je(t.n_leaves, (int32_t)t.M), jl(t.M);
    for (int64_t i = 0; i < t.M; ++i) jl[i] = (int32_t)i;
    if (op.d_dn_jb.upload(jb) != cudaSuccess || op.d_dn_je.upload(je) != cudaSuccess ||
        op.d_dn_j.upload(jl) != cudaSuccess) {
      set_error("bem_assemble_h2_aca: upload failed");
      return fail(BEM_ECUDA);
    }
  }
  {
    bem_status rs = far_prepare(op);  // K3 Z-tile scratch (factors-only skeleton)
    if (rs != BEM_OK) return fail(rs);
  }
  const int64_t M = t.M;
  const size_t nl = (size_t)op.n_local;
  if (op.d_xc.alloc(nl * M * 2) != cudaSuccess || op.d_yc.alloc(nl * M * 2) != cudaSuccess) {
    set_error("bem_assemble_h2_aca: workspace allocation failed");
    return fail(BEM_ENOMEM);
  }
  if (mode != BEM_MODE_DENSE) {
    if (op.d_xhat.alloc((size_t)t.C * nl * t.p * 2) != cudaSuccess ||
        op.d_yhat.alloc((size_t)t.C * nl * t.p * 2) != cudaSuccess) {
      set_error("bem_assemble_h2_aca: workspace allocation failed");
      return fail(BEM_ENOMEM);
    }
  }
  if (cudaStreamSynchronize(st) != cudaSuccess) {
    set_error("bem_assemble_h2_aca: %s", cudaGetErrorString(cudaGetLastError()));
    return fail(BEM_ECUDA);
  }
  t.refcount++;
  *out = h;
  return BEM_OK;
}

// MACA of a subset of the far blocks only (the assembly's kernel and arithmetic, no
// skeleton kept): ranks and pivots of every listed block, for sampled bit-exactness
// checks at sizes whose full assembly takes minutes (config 5).
extern "C" bem_status bem_debug_aca_blocks(bem_tree th, const bem_c128* s, int32_t L, double aca_eps,
                                           const int32_t* blocks, int32_t nblk, int32_t* ranks, int32_t* pivots,
                                           int64_t* total_rank) {
  BEM_REQ(th && s && blocks && ranks && L >= 1 && nblk >= 1 && aca_eps > 0.0, "bem_debug_aca_blocks: bad arguments");
  Tree& t = th->t;
  BEM_REQ(t.device >= 0, "bem_debug_aca_blocks: host-only tree");
  std::vector<int32_t> sub(blocks, blocks + nblk);
  for (int b : sub) BEM_REQ(b >= 0 && b < (int)t.far_r.size(), "bem_debug_aca_blocks: block %d out of range", b);
  DeviceGuard dg(t.device);
  Op op;
  op.tree = &t; op.L = L; op.n_local = 1; op.mode = BEM_MODE_H2ACA; op.eps = aca_eps; op.local_l = {0};
  std::vector<double> sh(2 * (size_t)L);
  for (int l = 0; l < L; ++l) { sh[2 * l] = s[l].re; sh[2 * l + 1] = s[l].im; }
  BEM_CK(op.d_s.upload(sh));
  BEM_CK(op.d_local_l.upload(op.local_l));
  bem_status rs = run_aca(op, nullptr, false, false, &sub);
  if (rs != BEM_OK) return rs;
  std::vector<int32_t> pk((size_t)nblk * op.rcap), pq((size_t)nblk * op.rcap);
  BEM_CK(cudaMemcpy(pk.data(), op.d_pivk.p, sizeof(int32_t) * pk.size(), cudaMemcpyDeviceToHost));
  BEM_CK(cudaMemcpy(pq.data(), op.d_pivq.p, sizeof(int32_t) * pq.size(), cudaMemcpyDeviceToHost));
  int64_t tot = 0;
  for (int i = 0; i < nblk; ++i) {
    ranks[i] = op.ranks[i];
    for (int j = 0; j < op.ranks[i]; ++j) {
      if (pivots) {
        pivots[2 * tot] = pk[(size_t)i * op.rcap + j];
        pivots[2 * tot + 1] = pq[(size_t)i * op.rcap + j];
      }
      ++tot;
    }
  }
  if (total_rank) *total_rank = tot;
  return BEM_OK;
}

extern "C" bem_status bem_op_get_info(bem_op oh, bem_op_info* out) {
  BEM_REQ(oh && out, "bem_op_get_info: NULL argument");
  const Op& op = oh->o;
  const bool aca = op.mode == BEM_MODE_H2ACA || op.mode == BEM_MODE_COMBINED;
  out->mode = op.mode;
  out->skeleton = aca ? (op.z_stored ? 1 : 2) : 0;
  out->n_local = op.n_local;
  int rmax = 0;
  int64_t tot = 0;
  for (int v : op.ranks) { rmax = std::max(rmax, v); tot += v; }
  out->rmax = rmax;
  out->total_rank = tot;
  out->z_bytes = (int64_t)op.d_Z.n * 8;
  out->f_bytes = (int64_t)op.d_F.n * 8;
  const size_t dbl = op.d_s.n + op.d_Z.n + op.d_F.n + op.d_zs.n + op.d_part.n + op.d_nZ.n + op.d_nS.n + op.d_Df.n +
                     op.d_Dn.n + op.d_fS.n + op.d_g0f.n + op.d_g0n.n + op.d_conv_part.n + op.d_xc.n + op.d_yc.n +
                     op.d_xhat.n + op.d_yhat.n + op.step.tx.n + op.step.xf.n + op.step.yf.n + op.step.ty.n;
  const size_t i32 = op.d_local_l.n + op.d_class_t1.n + op.d_class_t2.n + op.d_dn_jb.n + op.d_dn_je.n + op.d_dn_j.n +
                     op.d_rank.n + op.d_pivk.n + op.d_pivq.n + op.d_far_rows.n + op.d_segs.n + op.d_seg_rows.n +
                     op.d_seg_ptr.n + op.d_nrank.n + op.d_npivk.n + op.d_npivq.n + op.d_nm_order.n + op.d_nm_counter.n;
  const size_t i64 = op.d_zoff.n + op.d_foff.n + op.d_ztoff.n + op.d_nzoff.n + op.d_nsoff.n + op.d_fsoff.n + op.d_g0noff.n;
  out->device_bytes = (int64_t)(8 * dbl + 4 * i32 + 8 * i64 + 8 * op.d_xmax.n);
  out->far_kernel = aca ? far_kernel_selected(op) : 0;
  out->reserved_ = 0;
  return BEM_OK;
}

extern "C" bem_status bem_aca_export(bem_op oh, int32_t* ranks, int32_t* pivots, int64_t* total_rank) {
  BEM_REQ(oh, "bem_aca_export: NULL op");
  Op& op = oh->o;
  if (op.mode != BEM_MODE_H2ACA && op.mode != BEM_MODE_COMBINED) {
    set_error("bem_aca_export: operator was not assembled with BEM_MODE_H2ACA / BEM_MODE_COMBINED");
    return BEM_ESTATE;
  }
  const int nfar = (int)op.ranks.size();
  int64_t tot = 0;
  for (int r : op.ranks) tot += r;
  if (total_rank) *total_rank = tot;
  if (ranks) std::copy(op.ranks.begin(), op.ranks.end(), ranks);
  if (pivots && nfar > 0) {
    DeviceGuard dg(op.tree->device);
    std::vector<int32_t> pk((size_t)nfar * op.rcap), pq((size_t)nfar * op.rcap);
    BEM_CK(cudaMemcpy(pk.data(), op.d_pivk.p, sizeof(int32_t) * pk.size(), cudaMemcpyDeviceToHost));
    BEM_CK(cudaMemcpy(pq.data(), op.d_pivq.p, sizeof(int32_t) * pq.size(), cudaMemcpyDeviceToHost));
    int64_t o = 0;
    for (int b = 0; b < nfar; ++b)
      for (int j = 0; j < op.ranks[b]; ++j) {
        pivots[2 * o] = pk[(size_t)b * op.rcap + j];
        pivots[2 * o + 1] = pq[(size_t)b * op.rcap + j];
        ++o;
      }
  }
  return BEM_OK;
}

extern "C" bem_status bem_aca_export_near(bem_op oh, int32_t* ranks, int32_t* pivots, int64_t* total_rank) {
  BEM_REQ(oh, "bem_aca_export_near: NULL op");
  Op& op = oh->o;
  if (op.mode != BEM_MODE_COMBINED) {
    set_error("bem_aca_export_near: operator was not assembled with BEM_MODE_COMBINED");
    return BEM_ESTATE;
  }
  const int nb = (int)op.nranks.size();
  int64_t tot = 0;
  for (int r : op.nranks) tot += r;
  if (total_rank) *total_rank = tot;
  if (ranks) std::copy(op.nranks.begin(), op.nranks.end(), ranks);
  if (pivots && nb > 0) {
    DeviceGuard dg(op.tree->device);
    std::vector<int32_t> pk((size_t)nb * op.nrcap), pq((size_t)nb * op.nrcap);
    BEM_CK(cudaMemcpy(pk.data(), op.d_npivk.p, sizeof(int32_t) * pk.size(), cudaMemcpyDeviceToHost));
    BEM_CK(cudaMemcpy(pq.data(), op.d_npivq.p, sizeof(int32_t) * pq.size(), cudaMemcpyDeviceToHost));
    int64_t o = 0;
    for (int b = 0; b < nb; ++b)
      for (int j = 0; j < op.nranks[b]; ++j) {
        pivots[2 * o] = pk[(size_t)b * op.nrcap + j];
        pivots[2 * o + 1] = pq[(size_t)b * op.nrcap + j];
        ++o;
      }
  }
  return BEM_OK;
}

extern "C" bem_status bem_op_destroy(bem_op oh) {
  if (!oh) return BEM_OK;
  DeviceGuard dg(oh->o.tree->device);
  shard_ws_release(&oh->o);
  oh->o.tree->refcount--;
  for (auto& e : oh->o.ev)
    if (e) cudaEventDestroy(e);
  if (oh->o.side) cudaStreamDestroy(oh->o.side);
  if (oh->o.ev_fork) cudaEventDestroy(oh->o.ev_fork);
  if (oh->o.ev_join) cudaEventDestroy(oh->o.ev_join);
  delete oh;
  return BEM_OK;
}

extern "C" bem_status bem_debug_pinned(const double* x, int64_t n, double* e, double* sn, double* cs,
                                       int32_t device) {
  BEM_REQ(x && e && sn && cs && n >= 0, "bem_debug_pinned: bad arguments");
  if (n == 0) return BEM_OK;
  DeviceGuard dg(device);
  DBuf<double> dx, de, ds, dc;
  BEM_CK(dx.alloc(n)); BEM_CK(de.alloc(n)); BEM_CK(ds.alloc(n)); BEM_CK(dc.alloc(n));
  BEM_CK(cudaMemcpy(dx.p, x, sizeof(double) * n, cudaMemcpyHostToDevice));
  debug_pinned_kernel<<<(unsigned)((n + 255) / 256), 256>>>(dx.p, n, de.p, ds.p, dc.p);
  BEM_CK(cudaGetLastError());
  BEM_CK(cudaMemcpy(e, de.p, sizeof(double) * n, cudaMemcpyDeviceToHost));
  BEM_CK(cudaMemcpy(sn, ds.p, sizeof(double) * n, cudaMemcpyDeviceToHost));
  BEM_CK(cudaMemcpy(cs, dc.p, sizeof(double) * n, cudaMemcpyDeviceToHost));
  return BEM_OK;
}
