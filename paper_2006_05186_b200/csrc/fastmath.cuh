// Branch-free FP64 exp / sincos for the hot kernels (K1 near field, K3 pivot
// slice regeneration).  Not used by the ACA (which needs the pinned,
// bit-reproducible versions in aca.cu); accuracy ~1-2 ulp over the ranges the
// configs produce (exp argument in [-708, 0], |theta| <= 1e5), checked
// against the oracle by the parity tests.
//
// exp:    x = k ln2 + r (Cody-Waite, |r| <= ln2/2), Taylor degree 12, the
//         power 2^k added to the exponent field (no multiply; x >= -708 keeps
//         the result normal, smaller arguments are clamped -- their
//         contribution is below 1e-300).
// sincos: theta = q pi/2 + r (3-part Cody-Waite), minimax polynomials on
//         |r| <= pi/4 (the classical fdlibm kernel coefficients), quadrant by
//         selects.
#pragma once

namespace bem {
namespace fast {

__device__ __forceinline__ double exp_neg(double x) {
  x = fmax(x, -708.0);
  const double t = fma(x, 1.4426950408889634074, 6755399441055744.0);
  const double kd = t - 6755399441055744.0;
  double r = fma(kd, -6.93147180369123816490e-01, x);
  r = fma(kd, -1.90821492927058770002e-10, r);
  double p = 2.08767569878680989792e-09;     // 1/12!
  p = fma(p, r, 2.50521083854417187751e-08);  // 1/11!
  p = fma(p, r, 2.75573192239858906526e-07);  // 1/10!
  p = fma(p, r, 2.75573192239858906526e-06);  // 1/9!
  p = fma(p, r, 2.48015873015873015873e-05);  // 1/8!
  p = fma(p, r, 1.98412698412698412698e-04);  // 1/7!
  p = fma(p, r, 1.38888888888888888889e-03);  // 1/6!
  p = fma(p, r, 8.33333333333333333333e-03);  // 1/5!
  p = fma(p, r, 4.16666666666666666667e-02);  // 1/4!
  p = fma(p, r, 1.66666666666666666667e-01);  // 1/3!
  p = fma(p, r, 0.5);
  p = fma(p, r, 1.0);
  p = fma(p, r, 1.0);
  const int k = __double2loint(t);
  return __hiloint2double(__double2hiint(p) + (k << 20), __double2loint(p));
}

__device__ __forceinline__ void sincos_(double th, double* sn, double* cs) {
  const double t = fma(th, 6.36619772367581382433e-01, 6755399441055744.0);
  const double qd = t - 6755399441055744.0;
  const int q = __double2loint(t);
  double r = fma(qd, -1.57079632673412561417e+00, th);
  r = fma(qd, -6.07710050650619224932e-11, r);
  r = fma(qd, -2.02226624879595063154e-21, r);
  const double z = r * r;
  double ps = 1.58969099521155010221e-10;
  ps = fma(ps, z, -2.50507602534068634195e-08);
  ps = fma(ps, z, 2.75573137070700676789e-06);
  ps = fma(ps, z, -1.98412698298579493134e-04);
  ps = fma(ps, z, 8.33333333332248946124e-03);
  ps = fma(ps, z, -1.66666666666666324348e-01);
  const double s = fma(r * z, ps, r);
  double pc = -1.13596475577881948265e-11;
  pc = fma(pc, z, 2.08757232129817482790e-09);
  pc = fma(pc, z, -2.75573143513906633035e-07);
  pc = fma(pc, z, 2.48015872894767294178e-05);
  pc = fma(pc, z, -1.38888888888741095749e-03);
  pc = fma(pc, z, 4.16666666666666019037e-02);
  const double c = fma(z * z, pc, fma(z, -0.5, 1.0));
  const bool swap = q & 1;
  const double so = swap ? c : s;
  const double co = swap ? s : c;
  // quadrant signs as integer sign-bit flips (keeps the FP64 pipe free)
  const int sflip = (q & 2) << 30, cflip = ((q + 1) & 2) << 30;
  *sn = __hiloint2double(__double2hiint(so) ^ sflip, __double2loint(so));
  *cs = __hiloint2double(__double2hiint(co) ^ cflip, __double2loint(co));
}

}  // namespace fast
}  // namespace bem
