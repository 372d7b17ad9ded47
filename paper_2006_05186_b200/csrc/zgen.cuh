// Factors-only MACA skeleton: the frequency coefficients Z_b of a far block
// regenerated from its stored factors (SURVEY §8(c) C10 "skeleton (CUR) form",
// AM17; eq:maca P:1314-1320).
//
// The ACA (Alg. 2) of block b with pivots (k_l, q_l), l < r, is an
// LU factorisation of the pivot submatrix A_b[Q,K] = C^_b U_b with
//   C^_b[l][j] = c_j[q_l]  (j <= l; the pivots c_l[q_l] on the diagonal),
//   U_b[l][j]  = d_l[k_j]  (j > l; unit upper triangular),
// stored together as F_b [r][r] row-major.  The ACA's rows d_l at frequency l
// are the forward substitution of the pivot fibre A_b[Q, l]:
//   d_l = (A_b[q_l, l] - sum_{j<l} C^_b[l][j] d_j) / C^_b[l][l],
// and Z_b[:, l] = U_b^{-1} d[:, l] (back substitution), so that
//   A_b[:, l] ~= sum_j Z_b[j, l] A_b[:, k_j]      (eq:maca, skeleton form).
// Both substitutions run in the ACA's pinned arithmetic (pinned.cuh) and the fibre
// entries are the pinned kernel of the ACA with the same conjugate mirroring; the
// forward substitution keeps the ACA's term order, so d is bit-identical to the
// ACA's; the back substitution subtracts in decreasing j (the oracle: increasing j),
// a rounding-level difference far below the 1e-10 parity tolerance.
#pragma once
#include "pinned.cuh"

namespace bem {
namespace zgen {
namespace {

struct Src {
  int m, p, L;
  const int32_t* far_r;
  const int32_t* far_c;
  const double* xi;      // C * 3 * m Chebyshev nodes per axis
  const double2* s;      // all L frequencies
  const int32_t* pivk;   // [nfar][rcap]
  const int32_t* pivq;   // [nfar][rcap]
  const int64_t* foff;   // F_b offsets (complex units)
  const double2* F;
  int rcap;
};

__device__ __forceinline__ void node3(const double* xi, int m, int mu, double* o) {
  o[0] = xi[mu % m];
  o[1] = xi[m + (mu / m) % m];
  o[2] = xi[2 * m + mu / (m * m)];
}

// A_b[q, l] in the ACA's pinned arithmetic (aca.cu entry()): l > L/2 is the
// conjugate of l' = L - l (values are defined by mirroring).
__device__ __forceinline__ double2 fibre(const Src& a, int rc, int cc, int q, int l) {
  const int half = a.L / 2;
  const bool mir = l > half;
  const int ll = mir ? a.L - l : l;
  double xr[3], xc[3];
  node3(a.xi + (int64_t)rc * 3 * a.m, a.m, q / a.p, xr);
  node3(a.xi + (int64_t)cc * 3 * a.m, a.m, q % a.p, xc);
  const double2 sv = a.s[ll];
  double2 v = pinned::kernel(pinned::dist(xr, xc), sv.x, sv.y);
  if (mir) v.y = -v.y;
  return v;
}

// Z_b for a set of frequency columns, computed by the whole CTA (every thread calls it):
// columns in batches of nb = cap / r in the shared buffer work [r][nb]:
//   1. the pivot fibres A_b[q_i, l] of the batch, spread over all threads;
//   2. forward substitution, right-looking: after step j the rows i > j have subtracted
//      C^[i][j] d_j, so each d_i accumulates its terms in increasing j -- exactly the
//      ACA's own order (aca.cu computes the same d); one barrier per step;
//   3. back substitution, right-looking: Z_j is final once the rows j' > j have been
//      subtracted (in decreasing j'), then every row i < j subtracts U[i][j] Z_j;
//   4. out(j, c, Z_b[j, c]) for every row j and column c of the batch.
// col_l(c) = the global frequency of column c, or -1 for a zero (padding / masked)
// column.  The stored-Z regeneration (aca.cu) and the factors-only tile pass (far.cu)
// both call this function, so the two skeleton modes agree bit for bit.
template <class ColFn, class OutFn>
__device__ __forceinline__ void block_columns(const Src& a, int b, int r, int c_begin, int c_end, ColFn col_l,
                                              double2* work, int cap, OutFn out) {
  using namespace pinned;
  if (r <= 0) return;
  const int rc = a.far_r[b], cc = a.far_c[b];
  const double2* F = a.F + a.foff[b];
  const int32_t* qp = a.pivq + (int64_t)b * a.rcap;
  const int nb = max(1, min(c_end - c_begin, cap / r));
  for (int c0 = c_begin; c0 < c_end; c0 += nb) {
    const int nc = min(nb, c_end - c0);
    for (int e = threadIdx.x; e < r * nc; e += blockDim.x) {
      const int i = e / nc, cl = e - i * nc;
      const int l = col_l(c0 + cl);
      BEM_DASSERT(i * nb + cl < cap && l < a.L);
      work[i * nb + cl] = l >= 0 ? fibre(a, rc, cc, qp[i], l) : make_double2(0.0, 0.0);
    }
    __syncthreads();
    for (int cl = threadIdx.x; cl < nc; cl += blockDim.x) work[cl] = cdiv(work[cl], F[0]);
    __syncthreads();
    for (int j = 0; j + 1 < r; ++j) {  // forward: rows i > j subtract C^[i][j] d_j; row j+1 then divides
      const int n = (r - j - 1) * nc;
      for (int e = threadIdx.x; e < n; e += blockDim.x) {
        const int i = j + 1 + e / nc, cl = e % nc;
        double2 v = csub(work[i * nb + cl], cmul(F[(int64_t)i * r + j], work[j * nb + cl]));
        if (i == j + 1) v = cdiv(v, F[(int64_t)i * r + i]);
        work[i * nb + cl] = v;
      }
      __syncthreads();
    }
    for (int j = r - 1; j >= 1; --j) {  // backward: rows i < j subtract U[i][j] Z_j
      const int n = j * nc;
      for (int e = threadIdx.x; e < n; e += blockDim.x) {
        const int i = e / nc, cl = e % nc;
        work[i * nb + cl] = csub(work[i * nb + cl], cmul(F[(int64_t)i * r + j], work[j * nb + cl]));
      }
      __syncthreads();
    }
    for (int e = threadIdx.x; e < r * nc; e += blockDim.x) {
      const int jj = e / nc, cl = e - jj * nc;
      out(jj, c0 + cl, work[jj * nb + cl]);
    }
    __syncthreads();
  }
}

}  // namespace
}  // namespace zgen
}  // namespace bem
