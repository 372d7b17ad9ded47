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
//         selects and integer sign flips.
// The coefficients live in __constant__ memory so the DFMAs take them as
// constant-bank operands (no per-iteration immediate materialisation).
#pragma once

namespace bem {
namespace fast {

static __constant__ double kExpC[13] = {
    2.08767569878680989792e-09, 2.50521083854417187751e-08, 2.75573192239858906526e-07,
    2.75573192239858906526e-06, 2.48015873015873015873e-05, 1.98412698412698412698e-04,
    1.38888888888888888889e-03, 8.33333333333333333333e-03, 4.16666666666666666667e-02,
    1.66666666666666666667e-01, 0.5, 1.0, 1.0};
static __constant__ double kSinC[6] = {1.58969099521155010221e-10, -2.50507602534068634195e-08,
                                2.75573137070700676789e-06, -1.98412698298579493134e-04,
                                8.33333333332248946124e-03, -1.66666666666666324348e-01};
static __constant__ double kCosC[6] = {-1.13596475577881948265e-11, 2.08757232129817482790e-09,
                                -2.75573143513906633035e-07, 2.48015872894767294178e-05,
                                -1.38888888888741095749e-03, 4.16666666666666019037e-02};
static __constant__ double kRed[8] = {
    1.4426950408889634074,  -6.93147180369123816490e-01, -1.90821492927058770002e-10,  // exp
    6.36619772367581382433e-01, -1.57079632673412561417e+00, -6.07710050650619224932e-11,
    -2.02226624879595063154e-21,  // sincos
    6755399441055744.0};

static __constant__ double kExp2Tab[64] = {
    0x1.0000000000000p+0, 0x1.02c9a3e778061p+0, 0x1.059b0d3158574p+0, 0x1.0874518759bc8p+0,
    0x1.0b5586cf9890fp+0, 0x1.0e3ec32d3d1a2p+0, 0x1.11301d0125b51p+0, 0x1.1429aaea92de0p+0,
    0x1.172b83c7d517bp+0, 0x1.1a35beb6fcb75p+0, 0x1.1d4873168b9aap+0, 0x1.2063b88628cd6p+0,
    0x1.2387a6e756238p+0, 0x1.26b4565e27cddp+0, 0x1.29e9df51fdee1p+0, 0x1.2d285a6e4030bp+0,
    0x1.306fe0a31b715p+0, 0x1.33c08b26416ffp+0, 0x1.371a7373aa9cbp+0, 0x1.3a7db34e59ff7p+0,
    0x1.3dea64c123422p+0, 0x1.4160a21f72e2ap+0, 0x1.44e086061892dp+0, 0x1.486a2b5c13cd0p+0,
    0x1.4bfdad5362a27p+0, 0x1.4f9b2769d2ca7p+0, 0x1.5342b569d4f82p+0, 0x1.56f4736b527dap+0,
    0x1.5ab07dd485429p+0, 0x1.5e76f15ad2148p+0, 0x1.6247eb03a5585p+0, 0x1.6623882552225p+0,
    0x1.6a09e667f3bcdp+0, 0x1.6dfb23c651a2fp+0, 0x1.71f75e8ec5f74p+0, 0x1.75feb564267c9p+0,
    0x1.7a11473eb0187p+0, 0x1.7e2f336cf4e62p+0, 0x1.82589994cce13p+0, 0x1.868d99b4492edp+0,
    0x1.8ace5422aa0dbp+0, 0x1.8f1ae99157736p+0, 0x1.93737b0cdc5e5p+0, 0x1.97d829fde4e50p+0,
    0x1.9c49182a3f090p+0, 0x1.a0c667b5de565p+0, 0x1.a5503b23e255dp+0, 0x1.a9e6b5579fdbfp+0,
    0x1.ae89f995ad3adp+0, 0x1.b33a2b84f15fbp+0, 0x1.b7f76f2fb5e47p+0, 0x1.bcc1e904bc1d2p+0,
    0x1.c199bdd85529cp+0, 0x1.c67f12e57d14bp+0, 0x1.cb720dcef9069p+0, 0x1.d072d4a07897cp+0,
    0x1.d5818dcfba487p+0, 0x1.da9e603db3285p+0, 0x1.dfc97337b9b5fp+0, 0x1.e502ee78b3ff6p+0,
    0x1.ea4afa2a490dap+0, 0x1.efa1bee615a27p+0, 0x1.f50765b6e4540p+0, 0x1.fa7c1819e90d8p+0};
static __constant__ double kExpT[6] = {8.33333333333333333333e-03, 4.16666666666666666667e-02,
                                         1.66666666666666666667e-01, 0.5, 1.0, 1.0};

__device__ __forceinline__ double exp_neg(double x) {
  x = fmax(x, -708.0);
  const double t = fma(x, kRed[0], kRed[7]);
  const double kd = t - kRed[7];
  double r = fma(kd, kRed[1], x);
  r = fma(kd, kRed[2], r);
  double p = kExpC[0];
#pragma unroll
  for (int i = 1; i < 13; ++i) p = fma(p, r, kExpC[i]);
  const int k = __double2loint(t);
  return __hiloint2double(__double2hiint(p) + (k << 20), __double2loint(p));
}

// Table-driven variant: x = (64 k + j) ln2/64 + r, |r| <= ln2/128 (|x| < 1e13),
// e^x = 2^k * T[j] * poly5(r), T[j] = 2^(j/64) (host-rounded, in shared
// memory); truncation error r^6/720 < 4e-17.  Caller provides the table.
static __constant__ double kET[4] = {92.332482616893656473, 6755399441055744.0,  // 64/ln2, magic
                                      -0x1.62e42ff000000p-7,                   // -ln2/64, high 32 bits (kd * hi exact)
                                      6.563929801064195e-13};                  // ln2/64 low part (hi - ln2/64)

__device__ __forceinline__ double exp_neg_tab(double x, const double* __restrict__ T) {
  const double t = fma(x, kET[0], kET[1]);
  const double kd = t - kET[1];
  double r = fma(kd, kET[2], x);
  r = fma(kd, kET[3], r);
  double p = kExpT[0];
#pragma unroll
  for (int i = 1; i < 6; ++i) p = fma(p, r, kExpT[i]);
  const int ki = __double2loint(t);
  p *= T[ki & 63];
  // exponent clamp in the integer pipe: x < -707 returns ~1e-307 instead of 0
  // (negligible) without an FP64 fmax
  return __hiloint2double(__double2hiint(p) + (max(ki >> 6, -1020) << 20), __double2loint(p));
}

__device__ __forceinline__ void sincos_(double th, double* sn, double* cs) {
  const double t = fma(th, kRed[3], kRed[7]);
  const double qd = t - kRed[7];
  const int q = __double2loint(t);
  double r = fma(qd, kRed[4], th);
  r = fma(qd, kRed[5], r);
  r = fma(qd, kRed[6], r);
  const double z = r * r;
  double ps = kSinC[0];
#pragma unroll
  for (int i = 1; i < 6; ++i) ps = fma(ps, z, kSinC[i]);
  const double s = fma(r * z, ps, r);
  double pc = kCosC[0];
#pragma unroll
  for (int i = 1; i < 6; ++i) pc = fma(pc, z, kCosC[i]);
  const double c = fma(z * z, pc, fma(z, -0.5, 1.0));
  const bool swap = q & 1;
  const double so = swap ? c : s;
  const double co = swap ? s : c;
  // quadrant signs as integer sign-bit flips (keeps the FP64 pipe free)
  const int sflip = (q & 2) << 30, cflip = ((q + 1) & 2) << 30;
  *sn = __hiloint2double(__double2hiint(so) ^ sflip, __double2loint(so));
  *cs = __hiloint2double(__double2hiint(co) ^ cflip, __double2loint(co));
}


// Table-driven sincos: th = k pi/32 + r (2-part Cody-Waite with the fdlibm
// pio2_1 / pio2_1t split scaled by 1/16; kd * hi is exact for |k| < 2^20,
// i.e. |th| < 1e5), |r| <= pi/64; Taylor sin to r^7 and cos to r^8
// (truncation < 1e-16 relative); (cos, sin)(k pi/32) from a 64-entry table
// (correctly rounded, caller stages it in shared memory) -- the table also
// carries the quadrant, so there is no select/sign logic.
static __constant__ double2 kSinCosTab[64] = {
    {0x1.0000000000000p+0, 0x0.0p+0}, {0x1.fd88da3d12526p-1, 0x1.917a6bc29b42cp-4},
    {0x1.f6297cff75cb0p-1, 0x1.8f8b83c69a60bp-3}, {0x1.e9f4156c62ddap-1, 0x1.294062ed59f06p-2},
    {0x1.d906bcf328d46p-1, 0x1.87de2a6aea963p-2}, {0x1.c38b2f180bdb1p-1, 0x1.e2b5d3806f63bp-2},
    {0x1.a9b66290ea1a3p-1, 0x1.1c73b39ae68c8p-1}, {0x1.8bc806b151741p-1, 0x1.44cf325091dd6p-1},
    {0x1.6a09e667f3bcdp-1, 0x1.6a09e667f3bcdp-1}, {0x1.44cf325091dd6p-1, 0x1.8bc806b151741p-1},
    {0x1.1c73b39ae68c8p-1, 0x1.a9b66290ea1a3p-1}, {0x1.e2b5d3806f63bp-2, 0x1.c38b2f180bdb1p-1},
    {0x1.87de2a6aea963p-2, 0x1.d906bcf328d46p-1}, {0x1.294062ed59f06p-2, 0x1.e9f4156c62ddap-1},
    {0x1.8f8b83c69a60bp-3, 0x1.f6297cff75cb0p-1}, {0x1.917a6bc29b42cp-4, 0x1.fd88da3d12526p-1},
    {0x0.0p+0, 0x1.0000000000000p+0}, {-0x1.917a6bc29b42cp-4, 0x1.fd88da3d12526p-1},
    {-0x1.8f8b83c69a60bp-3, 0x1.f6297cff75cb0p-1}, {-0x1.294062ed59f06p-2, 0x1.e9f4156c62ddap-1},
    {-0x1.87de2a6aea963p-2, 0x1.d906bcf328d46p-1}, {-0x1.e2b5d3806f63bp-2, 0x1.c38b2f180bdb1p-1},
    {-0x1.1c73b39ae68c8p-1, 0x1.a9b66290ea1a3p-1}, {-0x1.44cf325091dd6p-1, 0x1.8bc806b151741p-1},
    {-0x1.6a09e667f3bcdp-1, 0x1.6a09e667f3bcdp-1}, {-0x1.8bc806b151741p-1, 0x1.44cf325091dd6p-1},
    {-0x1.a9b66290ea1a3p-1, 0x1.1c73b39ae68c8p-1}, {-0x1.c38b2f180bdb1p-1, 0x1.e2b5d3806f63bp-2},
    {-0x1.d906bcf328d46p-1, 0x1.87de2a6aea963p-2}, {-0x1.e9f4156c62ddap-1, 0x1.294062ed59f06p-2},
    {-0x1.f6297cff75cb0p-1, 0x1.8f8b83c69a60bp-3}, {-0x1.fd88da3d12526p-1, 0x1.917a6bc29b42cp-4},
    {-0x1.0000000000000p+0, 0x0.0p+0}, {-0x1.fd88da3d12526p-1, -0x1.917a6bc29b42cp-4},
    {-0x1.f6297cff75cb0p-1, -0x1.8f8b83c69a60bp-3}, {-0x1.e9f4156c62ddap-1, -0x1.294062ed59f06p-2},
    {-0x1.d906bcf328d46p-1, -0x1.87de2a6aea963p-2}, {-0x1.c38b2f180bdb1p-1, -0x1.e2b5d3806f63bp-2},
    {-0x1.a9b66290ea1a3p-1, -0x1.1c73b39ae68c8p-1}, {-0x1.8bc806b151741p-1, -0x1.44cf325091dd6p-1},
    {-0x1.6a09e667f3bcdp-1, -0x1.6a09e667f3bcdp-1}, {-0x1.44cf325091dd6p-1, -0x1.8bc806b151741p-1},
    {-0x1.1c73b39ae68c8p-1, -0x1.a9b66290ea1a3p-1}, {-0x1.e2b5d3806f63bp-2, -0x1.c38b2f180bdb1p-1},
    {-0x1.87de2a6aea963p-2, -0x1.d906bcf328d46p-1}, {-0x1.294062ed59f06p-2, -0x1.e9f4156c62ddap-1},
    {-0x1.8f8b83c69a60bp-3, -0x1.f6297cff75cb0p-1}, {-0x1.917a6bc29b42cp-4, -0x1.fd88da3d12526p-1},
    {0x0.0p+0, -0x1.0000000000000p+0}, {0x1.917a6bc29b42cp-4, -0x1.fd88da3d12526p-1},
    {0x1.8f8b83c69a60bp-3, -0x1.f6297cff75cb0p-1}, {0x1.294062ed59f06p-2, -0x1.e9f4156c62ddap-1},
    {0x1.87de2a6aea963p-2, -0x1.d906bcf328d46p-1}, {0x1.e2b5d3806f63bp-2, -0x1.c38b2f180bdb1p-1},
    {0x1.1c73b39ae68c8p-1, -0x1.a9b66290ea1a3p-1}, {0x1.44cf325091dd6p-1, -0x1.8bc806b151741p-1},
    {0x1.6a09e667f3bcdp-1, -0x1.6a09e667f3bcdp-1}, {0x1.8bc806b151741p-1, -0x1.44cf325091dd6p-1},
    {0x1.a9b66290ea1a3p-1, -0x1.1c73b39ae68c8p-1}, {0x1.c38b2f180bdb1p-1, -0x1.e2b5d3806f63bp-2},
    {0x1.d906bcf328d46p-1, -0x1.87de2a6aea963p-2}, {0x1.e9f4156c62ddap-1, -0x1.294062ed59f06p-2},
    {0x1.f6297cff75cb0p-1, -0x1.8f8b83c69a60bp-3}, {0x1.fd88da3d12526p-1, -0x1.917a6bc29b42cp-4}};

// constant-bank operands (DFMA takes c[][] directly; immediates would be
// rematerialised through uniform registers every iteration)
static __constant__ double kSCT[12] = {
    10.185916357881301489, 6755399441055744.0, -0x1.921fb54400000p-4, -0x1.0b4611a626331p-38,  // 32/pi, magic, -pi/32 hi, lo
    -1.98412698412698412698e-04, 8.33333333333333333333e-03, -1.66666666666666666667e-01,      // sin r^7, r^5, r^3
    2.48015873015873015873e-05, -1.38888888888888888889e-03, 4.16666666666666666667e-02, -0.5, 1.0};  // cos

__device__ __forceinline__ void sincos_tab(double th, const double2* __restrict__ T, double* sn, double* cs) {
  const double t = fma(th, kSCT[0], kSCT[1]);
  const double kd = t - kSCT[1];
  double r = fma(kd, kSCT[2], th);
  r = fma(kd, kSCT[3], r);
  const double z = r * r;
  const double ps = fma(z, fma(z, kSCT[4], kSCT[5]), kSCT[6]);
  const double sr = fma(r * z, ps, r);
  const double cr = fma(z, fma(z, fma(z, fma(z, kSCT[7], kSCT[8]), kSCT[9]), kSCT[10]), kSCT[11]);
  const double2 cs_k = T[__double2loint(t) & 63];
  *sn = fma(cs_k.y, cr, cs_k.x * sr);
  *cs = fma(cs_k.x, cr, -(cs_k.y * sr));
}

}  // namespace fast
}  // namespace bem
