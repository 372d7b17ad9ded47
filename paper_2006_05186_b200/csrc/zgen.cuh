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
// Both substitutions run in the ACA's pinned arithmetic and operation order
// (pinned.cuh; aca.cu computes exactly these d_l and Z), and the fibre entries
// are the pinned kernel of the ACA with the same conjugate mirroring, so the
// regenerated Z is bit-identical to the one the ACA itself would store.
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

// Z_b[:, l] for one frequency column, z[i * stride] already holding the pivot fibre
// A_b[q_i, l] (fibre(), or zero for a padding column): forward substitution to d, then
// back substitution to Z, in place.  Each row's dot product is split over four
// interleaved partial sums (j mod 4), combined as ((s0 + s1) + (s2 + s3)) and then
// subtracted: a fixed pinned order (bit-reproducible; the stored-Z and the factors-only
// paths share this function), with a dependency chain a quarter as long as a
// sequential sum.  (The ACA's own d rows use the sequential order; the difference is
// rounding-level, far below the 1e-10 parity tolerance.)
__device__ __forceinline__ double2 dot4(const double2* __restrict__ Fi, const double2* z, int64_t stride, int j0,
                                        int j1) {
  using namespace pinned;
  double2 s[4] = {make_double2(0.0, 0.0), make_double2(0.0, 0.0), make_double2(0.0, 0.0), make_double2(0.0, 0.0)};
  int j = j0;
  for (; j + 4 <= j1; j += 4) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const double2 pr = cmul(Fi[j + u], z[(j + u) * stride]);
      s[u] = make_double2(add(s[u].x, pr.x), add(s[u].y, pr.y));
    }
  }
  for (int u = 0; j < j1; ++j, ++u) {
    const double2 pr = cmul(Fi[j], z[j * stride]);
    s[u] = make_double2(add(s[u].x, pr.x), add(s[u].y, pr.y));
  }
  return make_double2(add(add(s[0].x, s[1].x), add(s[2].x, s[3].x)), add(add(s[0].y, s[1].y), add(s[2].y, s[3].y)));
}

// (not inlined: keeps the coupling kernel's hot-loop register allocation unchanged)
__device__ __forceinline__ void solve(const Src& a, int b, int r, double2* z, int64_t stride) {
  using namespace pinned;
  const double2* F = a.F + a.foff[b];
  for (int i = 0; i < r; ++i)  // forward: d_i = (A[q_i, l] - sum_{j<i} C^[i][j] d_j) / C^[i][i]
    z[i * stride] = cdiv(csub(z[i * stride], dot4(F + (int64_t)i * r, z, stride, 0, i)), F[(int64_t)i * r + i]);
  for (int i = r - 2; i >= 0; --i)  // backward: Z_i = d_i - sum_{j>i} U[i][j] Z_j
    z[i * stride] = csub(z[i * stride], dot4(F + (int64_t)i * r, z, stride, i + 1, r));
}

// the whole column: fibres, then the substitutions; l < 0 writes a zero column (padding)
__device__ __forceinline__ void column(const Src& a, int b, int r, int l, double2* z, int64_t stride) {
  if (l < 0) {
    for (int j = 0; j < r; ++j) z[j * stride] = make_double2(0.0, 0.0);
    return;
  }
  const int rc = a.far_r[b], cc = a.far_c[b];
  const int32_t* qp = a.pivq + (int64_t)b * a.rcap;
  for (int i = 0; i < r; ++i) z[i * stride] = fibre(a, rc, cc, qp[i], l);
  solve(a, b, r, z, stride);
}

}  // namespace
}  // namespace zgen
}  // namespace bem
