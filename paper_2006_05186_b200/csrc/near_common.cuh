// K1 near-field building blocks shared by the standalone kernels (near.cu) and the near-field
// warps fused into the K3 far10 kernel (farq.cu). See near.cu for the formulas.
#pragma once
#include "common.cuh"
#include "fastmath.cuh"

namespace bem {

struct NearArgs {
  int64_t M;
  int n_class;
  const int32_t* leaf_of;
  const int32_t* near_jb;
  const int32_t* near_je;
  const int32_t* near_j;
  const int32_t* near_gb = nullptr;  // with gsuf: the cutoff's early exit (nullable)
  const unsigned* gsuf = nullptr;    // float bits of the squared suffix distances (rounded down)
  int64_t gsuf_n = 0;                // its entries (bounds checks)
  const double* cen;
  const double* qn;
  const double* qw;
  const double* nrm;  // unit normals (double layer)
  const double* selfJ;
  const double2* s;
  const int32_t* local_l;
  const int32_t* class_t1;
  const int32_t* class_t2;
  const int32_t* mask;  // nullable: per local frequency, 0 = skip (output 0)
  const double2* xc;
  double2* yc;
  double tau = 0.0;  // underflow cutoff on Re s * r (0: off)
  double hmax = 0.0;  // largest quadrature-node-to-centroid distance of the mesh (the cutoff's slack)
  unsigned long long* evals = nullptr;  // profiling: += kernel evaluations run (nullable)
};

__device__ __forceinline__ void cmac(double2& acc, double2 a, double2 b) {
  acc.x = fma(a.x, b.x, acc.x);
  acc.x = fma(-a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y);
  acc.y = fma(a.y, b.x, acc.y);
}
__device__ __forceinline__ void cmac_conj(double2& acc, double2 a, double2 b) {  // acc += conj(a) b
  acc.x = fma(a.x, b.x, acc.x);
  acc.x = fma(a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y);
  acc.y = fma(-a.y, b.x, acc.y);
}


namespace {

// self entry V[i,i](s) = J/4pi + sum_q (w_q |T_i|/4pi) phi(s, r_q): computed once per target and
// class, spread over the lanes of the warp (self_node per node q >= 1)
// one node's share of the self entry: qw_q phi(s, r_q) / ... (q >= 1); libdevice functions
__device__ __forceinline__ double2 self_node(const double* qn, const double* qw, const double* c, int q, double sre,
                                             double sim) {
  const double dx = c[0] - qn[3 * q], dy = c[1] - qn[3 * q + 1], dz = c[2] - qn[3 * q + 2];
  const double r = sqrt(dx * dx + dy * dy + dz * dz);
  const double xr = -sre * r, yr = -sim * r;
  double sn, cs, sh, ch;
  sincos(yr, &sn, &cs);
  sincos(0.5 * yr, &sh, &ch);
  const double re = expm1(xr) * cs - 2.0 * sh * sh;  // Re(e^z - 1), cancellation-free
  const double im = exp(xr) * sn;
  return make_double2(qw[q] / r * re, qw[q] / r * im);
}

// DL: double-layer kernel d/dn_y e^{-sr}/(4 pi r) (NEXT-1): per node the factor
// (x - y).n_y / r^3 and (1 + s r) e^{-s r}; the self panel contributes 0.
// x is loaded after the node loop (r01: 128 instead of 164 registers, 4 CTAs per SM).
// one warp: target k, frequency classes c0 .. c0 + F - 1 (etab / sctab: the exp / sincos tables
// in shared memory)
// CUT: the underflow cutoff below is compiled in (a.tau <= 0 then means no cutoff)
template <int F, bool DL = false, bool CUT = !DL>
__device__ __forceinline__ void near_item(const NearArgs& a, int64_t k, int c0, const double* etab,
                                          const double2* sctab) {
  const int lane = threadIdx.x & 31;
  if (k >= a.M) return;
  double sre[F], sim[F];
  int64_t o1[F], o2[F];
#pragma unroll
  for (int f = 0; f < F; ++f) {
    const int c = c0 + f;
    const bool on = c < a.n_class &&
                    (a.mask == nullptr || a.mask[a.class_t1[c]] || (a.class_t2[c] >= 0 && a.mask[a.class_t2[c]]));
    if (c < a.n_class && !on) {  // converged frequencies (GMRES mask): write zeros, skip the work
      const int t1 = a.class_t1[c], t2 = a.class_t2[c];
      if (lane == 0) {
        a.yc[(int64_t)t1 * a.M + k] = make_double2(0.0, 0.0);
        if (t2 >= 0) a.yc[(int64_t)t2 * a.M + k] = make_double2(0.0, 0.0);
      }
    }
    if (on) {
      const int t1 = a.class_t1[c], t2 = a.class_t2[c];
      const double2 sv = a.s[a.local_l[t1]];
      sre[f] = sv.x; sim[f] = sv.y;
      o1[f] = (int64_t)t1 * a.M;
      o2[f] = t2 >= 0 ? (int64_t)t2 * a.M : -1;
    } else {
      sre[f] = 0.0; sim[f] = 0.0; o1[f] = -1; o2[f] = -1;
    }
  }
  bool any = false;
#pragma unroll
  for (int f = 0; f < F; ++f) any |= o1[f] >= 0;
  if (!any) return;
  double2 acc1[F], acc2[F];
#pragma unroll
  for (int f = 0; f < F; ++f) { acc1[f] = make_double2(0.0, 0.0); acc2[f] = make_double2(0.0, 0.0); }
  const double cx = a.cen[3 * k], cy = a.cen[3 * k + 1], cz = a.cen[3 * k + 2];
  const int li = a.leaf_of[k];
  const int jb = a.near_jb[li], je = a.near_je[li];
  // Underflow cutoff ("K1 underflow cutoff"): |e^{-s r}| = e^{-Re s r}, so a class
  // whose Re s r_min exceeds a.tau over the 32 sources of a warp step adds less than e^{-tau}
  // (tau = 42: 6e-19) of the kernel's 1/(4 pi r) scale -- below the rounding of the row sum.
  // r_min >= min_j |c_k - c_j| - hmax (source centroids, hmax = the largest node-to-centroid
  // distance of the mesh): the step is left out when min_j |c_k - c_j|^2 > rc^2, rc = tau /
  // min_f Re s_f + hmax, compared as float bit patterns (distances rounded down, rc^2 up; no
  // square root, one register of state: the loop sits at its 128-register budget and a test
  // with its operands in double cost 10 % per evaluated step, this one 4 %).  a.gsuf carries per
  // step the smallest squared distance of the target leaf's box to any later source centroid:
  // past rc^2 the loop ends.  The decision is warp-uniform and all-or-nothing for the F classes
  // of the tile (neighbours in Re s: a per-class decision would leave out 0.5 % more at config 4
  // and costs the kernel its instruction-level parallelism), so nothing diverges.
  unsigned rc2bits = 0x7f800000u;  // +inf: run every step
  unsigned nact = 0;
  {
    double smin = 1e300;  // smallest Re s of the tile's active classes
#pragma unroll
    for (int f = 0; f < F; ++f)
      if (o1[f] >= 0) { smin = fmin(smin, sre[f]); ++nact; }
    if (CUT && a.tau > 0.0 && smin > 0.0) {
      const double rc = a.tau / smin + a.hmax;
      const double rc2 = rc * rc * (1.0 + 1e-6);
      if (rc2 < 1e30) rc2bits = __float_as_uint(__double2float_ru(rc2));
    }
  }
  unsigned nev = 0;  // kernel evaluations of this lane (profiling)
  int jn = jb + lane < je ? a.near_j[jb + lane] : 0;
  int gi = CUT && a.gsuf != nullptr ? a.near_gb[li] : -1;  // this step's entry of a.gsuf
  for (int j0 = jb; j0 < je; j0 += 32) {
    const int jj = j0 + lane;
    const int j = jn;  // index loaded one step ahead (one dependent global load fewer per source)
    if (jj + 32 < je) jn = a.near_j[jj + 32];
    const bool use = jj < je && j != k;  // self panel below
    if (CUT) {
      BEM_DASSERT(gi < a.gsuf_n);
      if (gi >= 0 && a.gsuf[gi++] > rc2bits) break;  // every later source is out of reach too
      float d2 = 1e30f;
      if (use) {
        const double ddx = cx - a.cen[3 * (int64_t)j], ddy = cy - a.cen[3 * (int64_t)j + 1], ddz = cz - a.cen[3 * (int64_t)j + 2];
        d2 = __double2float_rd(ddx * ddx + ddy * ddy + ddz * ddz);
      }
      // warp minimum through the (monotone) bit pattern of the non-negative float
      if (__reduce_min_sync(0xffffffffu, __float_as_uint(d2)) > rc2bits) continue;
    }
    const double* qn = a.qn + 21 * (int64_t)j;
    const double* qw = a.qw + 7 * (int64_t)j;
    if (!use) continue;
    nev += 7u * nact;
    double2 x1[F], x2[F];
    double2 v[F];
#pragma unroll
    for (int f = 0; f < F; ++f) v[f] = make_double2(0.0, 0.0);
    double nx = 0.0, ny = 0.0, nz = 0.0;
    if (DL) { nx = a.nrm[3 * (int64_t)j]; ny = a.nrm[3 * (int64_t)j + 1]; nz = a.nrm[3 * (int64_t)j + 2]; }
#pragma unroll 7
    for (int q = 0; q < 7; ++q) {
      const double dx = cx - qn[3 * q], dy = cy - qn[3 * q + 1], dz = cz - qn[3 * q + 2];
      const double d2 = dx * dx + dy * dy + dz * dz;
      const double ir = rsqrt(d2);
      const double r = d2 * ir;
      const double w = DL ? qw[q] * ((dx * nx + dy * ny) + dz * nz) * (ir * ir * ir) : qw[q] * ir;
#pragma unroll
      for (int f = 0; f < F; ++f) {
        const double e = fast::exp_neg_tab(-sre[f] * r, etab) * w;
        double sn, cs;
        fast::sincos_tab(sim[f] * r, sctab, &sn, &cs);
        if (DL) {  // (1 + s r) e^{-s r}: (alpha + i beta)(cos - i sin) E
          const double ea = e * fma(sre[f], r, 1.0), eb = e * (sim[f] * r);
          v[f].x = fma(ea, cs, fma(eb, sn, v[f].x));
          v[f].y = fma(eb, cs, fma(-ea, sn, v[f].y));
        } else {
          v[f].x = fma(e, cs, v[f].x);
          v[f].y = fma(-e, sn, v[f].y);
        }
      }
    }
#pragma unroll
    for (int f = 0; f < F; ++f) {
      x1[f] = o1[f] >= 0 ? a.xc[o1[f] + j] : make_double2(0.0, 0.0);
      x2[f] = o2[f] >= 0 ? a.xc[o2[f] + j] : make_double2(0.0, 0.0);
    }
#pragma unroll
    for (int f = 0; f < F; ++f) {
      cmac(acc1[f], v[f], x1[f]);
      cmac_conj(acc2[f], v[f], x2[f]);
    }
  }
  if (!DL) {
    // self panel, spread over the warp: lane (f, q-1) for q = 1..6 evaluates one
    // node of class f (libdevice expm1 / sincos); the lane with q = 1 also adds
    // J and the centroid node phi(s,0) = -s.  Summed by the reduction below.
    const double c[3] = {cx, cy, cz};
    const double* qnk = a.qn + 21 * k;
    const double* qwk = a.qw + 7 * k;
#pragma unroll
    for (int f = 0; f < F; ++f) {
      if (o1[f] < 0 || lane < 6 * f || lane >= 6 * f + 6) continue;
      const int q = 1 + lane - 6 * f;
      double2 v = self_node(qnk, qwk, c, q, sre[f], sim[f]);
      if (q == 1) {
        v.x += a.selfJ[k] - qwk[0] * sre[f];
        v.y -= qwk[0] * sim[f];
      }
      cmac(acc1[f], v, a.xc[o1[f] + k]);
      if (o2[f] >= 0) cmac_conj(acc2[f], v, a.xc[o2[f] + k]);
    }
  }
#pragma unroll
  for (int f = 0; f < F; ++f) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      acc1[f].x += __shfl_xor_sync(0xffffffffu, acc1[f].x, off);
      acc1[f].y += __shfl_xor_sync(0xffffffffu, acc1[f].y, off);
      acc2[f].x += __shfl_xor_sync(0xffffffffu, acc2[f].x, off);
      acc2[f].y += __shfl_xor_sync(0xffffffffu, acc2[f].y, off);
    }
  }
  if (a.evals != nullptr) {
    if (!DL && lane == 0) {  // the self panel's rule
#pragma unroll
      for (int f = 0; f < F; ++f) nev += o1[f] >= 0 ? 7u : 0u;
    }
    nev = __reduce_add_sync(0xffffffffu, nev);
    if (lane == 0) atomicAdd(a.evals, (unsigned long long)nev);
  }
#pragma unroll
  for (int f = 0; f < F; ++f) {
    if (lane == 2 * f && o1[f] >= 0) a.yc[o1[f] + k] = acc1[f];
    if (lane == 2 * f + 1 && o2[f] >= 0) a.yc[o2[f] + k] = acc2[f];
  }
}


}  // namespace

// the NearArgs of an op's single-layer near field and its class tile F (near.cu); launch of
// the standalone kernel taking (target, class tile) items from *ctr until n_items
void near_args(Op& op, const double2* xc, double2* yc, NearArgs& na, int& F);
bem_status launch_near_tail(const NearArgs& na, int F, unsigned* ctr, cudaStream_t st);

}  // namespace bem
