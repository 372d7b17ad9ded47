// Pinned, bit-reproducible FP64 arithmetic of the ACA: IEEE
// +,-,*,/,sqrt,fma only through __d*_rn / __fma_rn intrinsics (no contraction),
// Cody-Waite exp / sincos with fixed Taylor polynomials, complex ops with every
// product and sum an explicit IEEE op.  Used by the MACA assembly (aca.cu) and
// by the factors-only skeleton (zgen.cuh: the pivot fibres regenerated per
// apply), so both reproduce the ACA's D_b rows bit for bit.  (Written
// independently of the oracle's own pinned functions; tests compare them.)
#pragma once
#include <cuda_runtime.h>

namespace bem {
namespace pinned {
namespace {

__device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double fma(double a, double b, double c) { return __fma_rn(a, b, c); }

__device__ __forceinline__ double pow2i(int k) { return __longlong_as_double((long long)(k + 1023) << 52); }

__device__ double exp_(double x) {
  if (x < -746.0) return 0.0;
  if (x > 709.5) return __longlong_as_double(0x7ff0000000000000LL);
  const double t = fma(x, 0x1.71547652b82fep+0, 0x1.8p+52);
  const double kd = sub(t, 0x1.8p+52);
  double r = fma(kd, -0x1.62e42fee00000p-1, x);
  r = fma(kd, -0x1.a39ef35793c76p-33, r);
  double q = 0x1.6124613a86d09p-33;  // 1/13!
  q = fma(q, r, 0x1.1eed8eff8d898p-29);
  q = fma(q, r, 0x1.ae64567f544e4p-26);
  q = fma(q, r, 0x1.27e4fb7789f5cp-22);
  q = fma(q, r, 0x1.71de3a556c734p-19);
  q = fma(q, r, 0x1.a01a01a01a01ap-16);
  q = fma(q, r, 0x1.a01a01a01a01ap-13);
  q = fma(q, r, 0x1.6c16c16c16c17p-10);
  q = fma(q, r, 0x1.1111111111111p-7);
  q = fma(q, r, 0x1.5555555555555p-5);
  q = fma(q, r, 0x1.5555555555555p-3);
  q = fma(q, r, 0x1.0000000000000p-1);
  q = fma(q, r, 0x1.0000000000000p+0);
  q = fma(q, r, 0x1.0000000000000p+0);
  const int k = (int)kd;
  if (k >= -1021) return mul(q, pow2i(k));
  return mul(mul(q, pow2i(k + 200)), pow2i(-200));
}

__device__ void sincos_(double th, double* sn, double* cs) {
  const double t = fma(th, 0x1.45f306dc9c883p-1, 0x1.8p+52);
  const double qd = sub(t, 0x1.8p+52);
  double r = fma(qd, -0x1.921fb54400000p+0, th);
  r = fma(qd, -0x1.0b4611a600000p-34, r);
  r = fma(qd, -0x1.3198a2e000000p-69, r);
  const double z = mul(r, r);
  double ps = 0x1.952c77030ad4ap-49;   // 1/17!
  ps = fma(ps, z, -0x1.ae7f3e733b81fp-41);
  ps = fma(ps, z, 0x1.6124613a86d09p-33);
  ps = fma(ps, z, -0x1.ae64567f544e4p-26);
  ps = fma(ps, z, 0x1.71de3a556c734p-19);
  ps = fma(ps, z, -0x1.a01a01a01a01ap-13);
  ps = fma(ps, z, 0x1.1111111111111p-7);
  ps = fma(ps, z, -0x1.5555555555555p-3);
  ps = fma(ps, z, 0x1.0000000000000p+0);
  const double s = mul(r, ps);
  double pc = -0x1.6827863b97d97p-53;  // -1/18!
  pc = fma(pc, z, 0x1.ae7f3e733b81fp-45);
  pc = fma(pc, z, -0x1.93974a8c07c9dp-37);
  pc = fma(pc, z, 0x1.1eed8eff8d898p-29);
  pc = fma(pc, z, -0x1.27e4fb7789f5cp-22);
  pc = fma(pc, z, 0x1.a01a01a01a01ap-16);
  pc = fma(pc, z, -0x1.6c16c16c16c17p-10);
  pc = fma(pc, z, 0x1.5555555555555p-5);
  pc = fma(pc, z, -0x1.0000000000000p-1);
  pc = fma(pc, z, 0x1.0000000000000p+0);
  switch ((int)((long long)qd & 3)) {
    case 0: *sn = s; *cs = pc; break;
    case 1: *sn = pc; *cs = -s; break;
    case 2: *sn = -s; *cs = -pc; break;
    default: *sn = -pc; *cs = s; break;
  }
}

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(sub(mul(a.x, b.x), mul(a.y, b.y)), add(mul(a.x, b.y), mul(a.y, b.x)));
}
__device__ __forceinline__ double2 cmulconj(double2 a, double2 b) {  // a * conj(b)
  return make_double2(add(mul(a.x, b.x), mul(a.y, b.y)), sub(mul(a.y, b.x), mul(a.x, b.y)));
}
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(sub(a.x, b.x), sub(a.y, b.y)); }
__device__ __forceinline__ double2 cdiv(double2 a, double2 c) {
  const double den = add(mul(c.x, c.x), mul(c.y, c.y));
  return make_double2(__ddiv_rn(add(mul(a.x, c.x), mul(a.y, c.y)), den),
                      __ddiv_rn(sub(mul(a.y, c.x), mul(a.x, c.y)), den));
}
__device__ __forceinline__ double key(double2 a) { return add(mul(a.x, a.x), mul(a.y, a.y)); }

// k(r; s) = e^{-s r}/(4 pi r): E = exp(-(Re s * r)), th = Im s * r,
// inv = 1/(4pi r), value = ((E cos th) inv, -((E sin th) inv)).
__device__ __forceinline__ double2 kernel(double r, double sre, double sim) {
  const double E = exp_(-mul(sre, r));
  double sn, cs;
  sincos_(mul(sim, r), &sn, &cs);
  const double inv = __ddiv_rn(1.0, mul(0x1.921fb54442d18p+3, r));
  return make_double2(mul(mul(E, cs), inv), -mul(mul(E, sn), inv));
}

__device__ __forceinline__ double dist(const double* a, const double* b) {
  const double dx = sub(b[0], a[0]), dy = sub(b[1], a[1]), dz = sub(b[2], a[2]);
  return __dsqrt_rn(add(add(mul(dx, dx), mul(dy, dy)), mul(dz, dz)));
}

// 1/k!, k = 0..19, correctly rounded (pinned expm1 of the self entry).
__device__ __constant__ double kInvFact[20] = {
    0x1.0000000000000p+0, 0x1.0000000000000p+0, 0x1.0000000000000p-1, 0x1.5555555555555p-3,
    0x1.5555555555555p-5, 0x1.1111111111111p-7, 0x1.6c16c16c16c17p-10, 0x1.a01a01a01a01ap-13,
    0x1.a01a01a01a01ap-16, 0x1.71de3a556c734p-19, 0x1.27e4fb7789f5cp-22, 0x1.ae64567f544e4p-26,
    0x1.1eed8eff8d898p-29, 0x1.6124613a86d09p-33, 0x1.93974a8c07c9dp-37, 0x1.ae7f3e733b81fp-41,
    0x1.ae7f3e733b81fp-45, 0x1.952c77030ad4ap-49, 0x1.6827863b97d97p-53, 0x1.2f49b46814157p-57};

// expm1: |x| < 1/2 -> x * sum_{k=1..19} x^{k-1}/k! (Horner in fma), else exp(x) - 1.
__device__ double expm1_(double x) {
  if (x > -0.5 && x < 0.5) {
    double q = kInvFact[19];
    for (int j = 18; j >= 1; --j) q = fma(q, x, kInvFact[j]);
    return mul(x, q);
  }
  return sub(exp_(x), 1.0);
}

// phi(s,r) = (e^{-sr} - 1)/r, r > 0: Re = expm1(x) cos y - 2 sin^2(y/2), Im = e^x sin y, x + iy = -s r.
__device__ double2 phi(double r, double sre, double sim) {
  const double x = -mul(sre, r), y = -mul(sim, r);
  double sy, cy, sh, ch;
  sincos_(y, &sy, &cy);
  sincos_(mul(0.5, y), &sh, &ch);
  const double re = sub(mul(expm1_(x), cy), mul(2.0, mul(sh, sh)));
  const double im = mul(exp_(x), sy);
  return make_double2(__ddiv_rn(re, r), __ddiv_rn(im, r));
}

// Collocation entry V(s)[i,j] (C3; the NEAR procedure of Alg. 3) in pinned
// arithmetic.  ci: centroid of panel i; cj: 21 node coordinates, |T_j|, J(T_j) of panel j.
__device__ double2 near_entry(const double* ci, const double* cj, bool self, double sre, double sim,
                              const double* w) {
  double ar = 0.0, ai = 0.0;
  const double area = cj[21];
  if (!self) {
    for (int q = 0; q < 7; ++q) {
      const double2 k = kernel(dist(ci, cj + 3 * q), sre, sim);
      const double wa = mul(w[q], area);
      ar = add(ar, mul(wa, k.x));
      ai = add(ai, mul(wa, k.y));
    }
    return make_double2(ar, ai);
  }
  ar = add(ar, mul(w[0], -sre));  // node 0 is the centroid: phi = -s
  ai = add(ai, mul(w[0], -sim));
  for (int q = 1; q < 7; ++q) {
    const double2 f = phi(dist(ci, cj + 3 * q), sre, sim);
    ar = add(ar, mul(w[q], f.x));
    ai = add(ai, mul(w[q], f.y));
  }
  constexpr double kInv4Pi = 0x1.45f306dc9c883p-4;
  return make_double2(mul(add(cj[22], mul(area, ar)), kInv4Pi), mul(mul(area, ai), kInv4Pi));
}

}  // namespace
}  // namespace pinned
}  // namespace bem
