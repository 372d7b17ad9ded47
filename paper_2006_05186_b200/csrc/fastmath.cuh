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


// ---- 256-entry variants (K1 / K3 hot loops): one polynomial term fewer in
// exp and two in sincos than the 64-entry versions, same accuracy class.
// exp: x = (256 k + j) ln2/256 + r, |r| <= ln2/512, degree-4 Taylor
// (truncation r^5/120 < 4e-17); T[j] = 2^(j/256) correctly rounded.
static __constant__ double kExp2Tab256[256] = {
    0x1.0000000000000p+0, 0x1.00b1afa5abcbfp+0, 0x1.0163da9fb3335p+0, 0x1.02168143b0281p+0,
    0x1.02c9a3e778061p+0, 0x1.037d42e11bbccp+0, 0x1.04315e86e7f85p+0, 0x1.04e5f72f654b1p+0,
    0x1.059b0d3158574p+0, 0x1.0650a0e3c1f89p+0, 0x1.0706b29ddf6dep+0, 0x1.07bd42b72a836p+0,
    0x1.0874518759bc8p+0, 0x1.092bdf66607e0p+0, 0x1.09e3ecac6f383p+0, 0x1.0a9c79b1f3919p+0,
    0x1.0b5586cf9890fp+0, 0x1.0c0f145e46c85p+0, 0x1.0cc922b7247f7p+0, 0x1.0d83b23395decp+0,
    0x1.0e3ec32d3d1a2p+0, 0x1.0efa55fdfa9c5p+0, 0x1.0fb66affed31bp+0, 0x1.1073028d7233ep+0,
    0x1.11301d0125b51p+0, 0x1.11edbab5e2ab6p+0, 0x1.12abdc06c31ccp+0, 0x1.136a814f204abp+0,
    0x1.1429aaea92de0p+0, 0x1.14e95934f312ep+0, 0x1.15a98c8a58e51p+0, 0x1.166a45471c3c2p+0,
    0x1.172b83c7d517bp+0, 0x1.17ed48695bbc0p+0, 0x1.18af9388c8deap+0, 0x1.1972658375d2fp+0,
    0x1.1a35beb6fcb75p+0, 0x1.1af99f8138a1cp+0, 0x1.1bbe084045cd4p+0, 0x1.1c82f95281c6bp+0,
    0x1.1d4873168b9aap+0, 0x1.1e0e75eb44027p+0, 0x1.1ed5022fcd91dp+0, 0x1.1f9c18438ce4dp+0,
    0x1.2063b88628cd6p+0, 0x1.212be3578a819p+0, 0x1.21f49917ddc96p+0, 0x1.22bdda27912d1p+0,
    0x1.2387a6e756238p+0, 0x1.2451ffb82140ap+0, 0x1.251ce4fb2a63fp+0, 0x1.25e85711ece75p+0,
    0x1.26b4565e27cddp+0, 0x1.2780e341ddf29p+0, 0x1.284dfe1f56381p+0, 0x1.291ba7591bb70p+0,
    0x1.29e9df51fdee1p+0, 0x1.2ab8a66d10f13p+0, 0x1.2b87fd0dad990p+0, 0x1.2c57e39771b2fp+0,
    0x1.2d285a6e4030bp+0, 0x1.2df961f641589p+0, 0x1.2ecafa93e2f56p+0, 0x1.2f9d24abd886bp+0,
    0x1.306fe0a31b715p+0, 0x1.31432edeeb2fdp+0, 0x1.32170fc4cd831p+0, 0x1.32eb83ba8ea32p+0,
    0x1.33c08b26416ffp+0, 0x1.3496266e3fa2dp+0, 0x1.356c55f929ff1p+0, 0x1.36431a2de883bp+0,
    0x1.371a7373aa9cbp+0, 0x1.37f26231e754ap+0, 0x1.38cae6d05d866p+0, 0x1.39a401b7140efp+0,
    0x1.3a7db34e59ff7p+0, 0x1.3b57fbfec6cf4p+0, 0x1.3c32dc313a8e5p+0, 0x1.3d0e544ede173p+0,
    0x1.3dea64c123422p+0, 0x1.3ec70df1c5175p+0, 0x1.3fa4504ac801cp+0, 0x1.40822c367a024p+0,
    0x1.4160a21f72e2ap+0, 0x1.423fb2709468ap+0, 0x1.431f5d950a897p+0, 0x1.43ffa3f84b9d4p+0,
    0x1.44e086061892dp+0, 0x1.45c2042a7d232p+0, 0x1.46a41ed1d0057p+0, 0x1.4786d668b3237p+0,
    0x1.486a2b5c13cd0p+0, 0x1.494e1e192aed2p+0, 0x1.4a32af0d7d3dep+0, 0x1.4b17dea6db7d7p+0,
    0x1.4bfdad5362a27p+0, 0x1.4ce41b817c114p+0, 0x1.4dcb299fddd0dp+0, 0x1.4eb2d81d8abffp+0,
    0x1.4f9b2769d2ca7p+0, 0x1.508417f4531eep+0, 0x1.516daa2cf6642p+0, 0x1.5257de83f4eefp+0,
    0x1.5342b569d4f82p+0, 0x1.542e2f4f6ad27p+0, 0x1.551a4ca5d920fp+0, 0x1.56070dde910d2p+0,
    0x1.56f4736b527dap+0, 0x1.57e27dbe2c4cfp+0, 0x1.58d12d497c7fdp+0, 0x1.59c0827ff07ccp+0,
    0x1.5ab07dd485429p+0, 0x1.5ba11fba87a03p+0, 0x1.5c9268a5946b7p+0, 0x1.5d84590998b93p+0,
    0x1.5e76f15ad2148p+0, 0x1.5f6a320dceb71p+0, 0x1.605e1b976dc09p+0, 0x1.6152ae6cdf6f4p+0,
    0x1.6247eb03a5585p+0, 0x1.633dd1d1929fdp+0, 0x1.6434634ccc320p+0, 0x1.652b9febc8fb7p+0,
    0x1.6623882552225p+0, 0x1.671c1c70833f6p+0, 0x1.68155d44ca973p+0, 0x1.690f4b19e9538p+0,
    0x1.6a09e667f3bcdp+0, 0x1.6b052fa75173ep+0, 0x1.6c012750bdabfp+0, 0x1.6cfdcddd47645p+0,
    0x1.6dfb23c651a2fp+0, 0x1.6ef9298593ae5p+0, 0x1.6ff7df9519484p+0, 0x1.70f7466f42e87p+0,
    0x1.71f75e8ec5f74p+0, 0x1.72f8286ead08ap+0, 0x1.73f9a48a58174p+0, 0x1.74fbd35d7cbfdp+0,
    0x1.75feb564267c9p+0, 0x1.77024b1ab6e09p+0, 0x1.780694fde5d3fp+0, 0x1.790b938ac1cf6p+0,
    0x1.7a11473eb0187p+0, 0x1.7b17b0976cfdbp+0, 0x1.7c1ed0130c132p+0, 0x1.7d26a62ff86f0p+0,
    0x1.7e2f336cf4e62p+0, 0x1.7f3878491c491p+0, 0x1.80427543e1a12p+0, 0x1.814d2add106d9p+0,
    0x1.82589994cce13p+0, 0x1.8364c1eb941f7p+0, 0x1.8471a4623c7adp+0, 0x1.857f4179f5b21p+0,
    0x1.868d99b4492edp+0, 0x1.879cad931a436p+0, 0x1.88ac7d98a6699p+0, 0x1.89bd0a478580fp+0,
    0x1.8ace5422aa0dbp+0, 0x1.8be05bad61778p+0, 0x1.8cf3216b5448cp+0, 0x1.8e06a5e0866d9p+0,
    0x1.8f1ae99157736p+0, 0x1.902fed0282c8ap+0, 0x1.9145b0b91ffc6p+0, 0x1.925c353aa2fe2p+0,
    0x1.93737b0cdc5e5p+0, 0x1.948b82b5f98e5p+0, 0x1.95a44cbc8520fp+0, 0x1.96bdd9a7670b3p+0,
    0x1.97d829fde4e50p+0, 0x1.98f33e47a22a2p+0, 0x1.9a0f170ca07bap+0, 0x1.9b2bb4d53fe0dp+0,
    0x1.9c49182a3f090p+0, 0x1.9d674194bb8d5p+0, 0x1.9e86319e32323p+0, 0x1.9fa5e8d07f29ep+0,
    0x1.a0c667b5de565p+0, 0x1.a1e7aed8eb8bbp+0, 0x1.a309bec4a2d33p+0, 0x1.a42c980460ad8p+0,
    0x1.a5503b23e255dp+0, 0x1.a674a8af46052p+0, 0x1.a799e1330b358p+0, 0x1.a8bfe53c12e59p+0,
    0x1.a9e6b5579fdbfp+0, 0x1.ab0e521356ebap+0, 0x1.ac36bbfd3f37ap+0, 0x1.ad5ff3a3c2774p+0,
    0x1.ae89f995ad3adp+0, 0x1.afb4ce622f2ffp+0, 0x1.b0e07298db666p+0, 0x1.b20ce6c9a8952p+0,
    0x1.b33a2b84f15fbp+0, 0x1.b468415b749b1p+0, 0x1.b59728de5593ap+0, 0x1.b6c6e29f1c52ap+0,
    0x1.b7f76f2fb5e47p+0, 0x1.b928cf22749e4p+0, 0x1.ba5b030a1064ap+0, 0x1.bb8e0b79a6f1fp+0,
    0x1.bcc1e904bc1d2p+0, 0x1.bdf69c3f3a207p+0, 0x1.bf2c25bd71e09p+0, 0x1.c06286141b33dp+0,
    0x1.c199bdd85529cp+0, 0x1.c2d1cd9fa652cp+0, 0x1.c40ab5fffd07ap+0, 0x1.c544778fafb22p+0,
    0x1.c67f12e57d14bp+0, 0x1.c7ba88988c933p+0, 0x1.c8f6d9406e7b5p+0, 0x1.ca3405751c4dbp+0,
    0x1.cb720dcef9069p+0, 0x1.ccb0f2e6d1675p+0, 0x1.cdf0b555dc3fap+0, 0x1.cf3155b5bab74p+0,
    0x1.d072d4a07897cp+0, 0x1.d1b532b08c968p+0, 0x1.d2f87080d89f2p+0, 0x1.d43c8eacaa1d6p+0,
    0x1.d5818dcfba487p+0, 0x1.d6c76e862e6d3p+0, 0x1.d80e316c98398p+0, 0x1.d955d71ff6075p+0,
    0x1.da9e603db3285p+0, 0x1.dbe7cd63a8315p+0, 0x1.dd321f301b460p+0, 0x1.de7d5641c0658p+0,
    0x1.dfc97337b9b5fp+0, 0x1.e11676b197d17p+0, 0x1.e264614f5a129p+0, 0x1.e3b333b16ee12p+0,
    0x1.e502ee78b3ff6p+0, 0x1.e653924676d76p+0, 0x1.e7a51fbc74c83p+0, 0x1.e8f7977cdb740p+0,
    0x1.ea4afa2a490dap+0, 0x1.eb9f4867cca6ep+0, 0x1.ecf482d8e67f1p+0, 0x1.ee4aaa2188510p+0,
    0x1.efa1bee615a27p+0, 0x1.f0f9c1cb6412ap+0, 0x1.f252b376bba97p+0, 0x1.f3ac948dd7274p+0,
    0x1.f50765b6e4540p+0, 0x1.f6632798844f8p+0, 0x1.f7bfdad9cbe14p+0, 0x1.f91d802243c89p+0,
    0x1.fa7c1819e90d8p+0, 0x1.fbdba3692d514p+0, 0x1.fd3c22b8f71f1p+0, 0x1.fe9d96b2a23d9p+0};
static __constant__ double kET256[4] = {369.32993046757462595,   // 256/ln2
                                        6755399441055744.0,      // 1.5 * 2^52
                                        -0x1.62e42ff000000p-9,  // -(ln2/256) rounded to 32 bits (kd * hi exact)
                                        0x1.718432a1b0e26p-43};  // -(ln2/256 - hi)
static __constant__ double kExpT4[5] = {4.16666666666666666667e-02, 1.66666666666666666667e-01, 0.5, 1.0, 1.0};

__device__ __forceinline__ double exp_neg_tab256(double x, const double* __restrict__ T) {
  const double t = fma(x, kET256[0], kET256[1]);
  const double kd = t - kET256[1];
  double r = fma(kd, kET256[2], x);
  r = fma(kd, kET256[3], r);
  double p = kExpT4[0];
#pragma unroll
  for (int i = 1; i < 5; ++i) p = fma(p, r, kExpT4[i]);
  const int ki = __double2loint(t);
  p *= T[ki & 255];
  return __hiloint2double(__double2hiint(p) + (max(ki >> 8, -1020) << 20), __double2loint(p));
}

// sincos: th = k pi/128 + r, |r| <= pi/256 (2-part Cody-Waite, pio2_1 / 64 split);
// sin r to r^5 (truncation r^7/5040 < 1e-17), cos r to r^6 (z^4/8! < 2e-20).
static __constant__ double2 kSinCosTab256[256] = {
    {0x1.0000000000000p+0, 0x0.0p+0}, {0x1.ffd886084cd0dp-1, 0x1.92155f7a3667ep-6},
    {0x1.ff621e3796d7ep-1, 0x1.91f65f10dd814p-5}, {0x1.fe9cdad01883ap-1, 0x1.2d52092ce19f6p-4},
    {0x1.fd88da3d12526p-1, 0x1.917a6bc29b42cp-4}, {0x1.fc26470e19fd3p-1, 0x1.f564e56a9730ep-4},
    {0x1.fa7557f08a517p-1, 0x1.2c8106e8e613ap-3}, {0x1.f8764fa714ba9p-1, 0x1.5e214448b3fc6p-3},
    {0x1.f6297cff75cb0p-1, 0x1.8f8b83c69a60bp-3}, {0x1.f38f3ac64e589p-1, 0x1.c0b826a7e4f63p-3},
    {0x1.f0a7efb9230d7p-1, 0x1.f19f97b215f1bp-3}, {0x1.ed740e7684963p-1, 0x1.111d262b1f677p-2},
    {0x1.e9f4156c62ddap-1, 0x1.294062ed59f06p-2}, {0x1.e6288ec48e112p-1, 0x1.4135c94176601p-2},
    {0x1.e212104f686e5p-1, 0x1.58f9a75ab1fddp-2}, {0x1.ddb13b6ccc23cp-1, 0x1.7088530fa459fp-2},
    {0x1.d906bcf328d46p-1, 0x1.87de2a6aea963p-2}, {0x1.d4134d14dc93ap-1, 0x1.9ef7943a8ed8ap-2},
    {0x1.ced7af43cc773p-1, 0x1.b5d1009e15cc0p-2}, {0x1.c954b213411f5p-1, 0x1.cc66e9931c45ep-2},
    {0x1.c38b2f180bdb1p-1, 0x1.e2b5d3806f63bp-2}, {0x1.bd7c0ac6f952ap-1, 0x1.f8ba4dbf89abap-2},
    {0x1.b728345196e3ep-1, 0x1.073879922ffeep-1}, {0x1.b090a58150200p-1, 0x1.11eb3541b4b23p-1},
    {0x1.a9b66290ea1a3p-1, 0x1.1c73b39ae68c8p-1}, {0x1.a29a7a0462782p-1, 0x1.26d054cdd12dfp-1},
    {0x1.9b3e047f38741p-1, 0x1.30ff7fce17035p-1}, {0x1.93a22499263fbp-1, 0x1.3affa292050b9p-1},
    {0x1.8bc806b151741p-1, 0x1.44cf325091dd6p-1}, {0x1.83b0e0bff976ep-1, 0x1.4e6cabbe3e5e9p-1},
    {0x1.7b5df226aafafp-1, 0x1.57d69348ceca0p-1}, {0x1.72d0837efff96p-1, 0x1.610b7551d2cdfp-1},
    {0x1.6a09e667f3bcdp-1, 0x1.6a09e667f3bcdp-1}, {0x1.610b7551d2cdfp-1, 0x1.72d0837efff96p-1},
    {0x1.57d69348ceca0p-1, 0x1.7b5df226aafafp-1}, {0x1.4e6cabbe3e5e9p-1, 0x1.83b0e0bff976ep-1},
    {0x1.44cf325091dd6p-1, 0x1.8bc806b151741p-1}, {0x1.3affa292050b9p-1, 0x1.93a22499263fbp-1},
    {0x1.30ff7fce17035p-1, 0x1.9b3e047f38741p-1}, {0x1.26d054cdd12dfp-1, 0x1.a29a7a0462782p-1},
    {0x1.1c73b39ae68c8p-1, 0x1.a9b66290ea1a3p-1}, {0x1.11eb3541b4b23p-1, 0x1.b090a58150200p-1},
    {0x1.073879922ffeep-1, 0x1.b728345196e3ep-1}, {0x1.f8ba4dbf89abap-2, 0x1.bd7c0ac6f952ap-1},
    {0x1.e2b5d3806f63bp-2, 0x1.c38b2f180bdb1p-1}, {0x1.cc66e9931c45ep-2, 0x1.c954b213411f5p-1},
    {0x1.b5d1009e15cc0p-2, 0x1.ced7af43cc773p-1}, {0x1.9ef7943a8ed8ap-2, 0x1.d4134d14dc93ap-1},
    {0x1.87de2a6aea963p-2, 0x1.d906bcf328d46p-1}, {0x1.7088530fa459fp-2, 0x1.ddb13b6ccc23cp-1},
    {0x1.58f9a75ab1fddp-2, 0x1.e212104f686e5p-1}, {0x1.4135c94176601p-2, 0x1.e6288ec48e112p-1},
    {0x1.294062ed59f06p-2, 0x1.e9f4156c62ddap-1}, {0x1.111d262b1f677p-2, 0x1.ed740e7684963p-1},
    {0x1.f19f97b215f1bp-3, 0x1.f0a7efb9230d7p-1}, {0x1.c0b826a7e4f63p-3, 0x1.f38f3ac64e589p-1},
    {0x1.8f8b83c69a60bp-3, 0x1.f6297cff75cb0p-1}, {0x1.5e214448b3fc6p-3, 0x1.f8764fa714ba9p-1},
    {0x1.2c8106e8e613ap-3, 0x1.fa7557f08a517p-1}, {0x1.f564e56a9730ep-4, 0x1.fc26470e19fd3p-1},
    {0x1.917a6bc29b42cp-4, 0x1.fd88da3d12526p-1}, {0x1.2d52092ce19f6p-4, 0x1.fe9cdad01883ap-1},
    {0x1.91f65f10dd814p-5, 0x1.ff621e3796d7ep-1}, {0x1.92155f7a3667ep-6, 0x1.ffd886084cd0dp-1},
    {0x0.0p+0, 0x1.0000000000000p+0}, {-0x1.92155f7a3667ep-6, 0x1.ffd886084cd0dp-1},
    {-0x1.91f65f10dd814p-5, 0x1.ff621e3796d7ep-1}, {-0x1.2d52092ce19f6p-4, 0x1.fe9cdad01883ap-1},
    {-0x1.917a6bc29b42cp-4, 0x1.fd88da3d12526p-1}, {-0x1.f564e56a9730ep-4, 0x1.fc26470e19fd3p-1},
    {-0x1.2c8106e8e613ap-3, 0x1.fa7557f08a517p-1}, {-0x1.5e214448b3fc6p-3, 0x1.f8764fa714ba9p-1},
    {-0x1.8f8b83c69a60bp-3, 0x1.f6297cff75cb0p-1}, {-0x1.c0b826a7e4f63p-3, 0x1.f38f3ac64e589p-1},
    {-0x1.f19f97b215f1bp-3, 0x1.f0a7efb9230d7p-1}, {-0x1.111d262b1f677p-2, 0x1.ed740e7684963p-1},
    {-0x1.294062ed59f06p-2, 0x1.e9f4156c62ddap-1}, {-0x1.4135c94176601p-2, 0x1.e6288ec48e112p-1},
    {-0x1.58f9a75ab1fddp-2, 0x1.e212104f686e5p-1}, {-0x1.7088530fa459fp-2, 0x1.ddb13b6ccc23cp-1},
    {-0x1.87de2a6aea963p-2, 0x1.d906bcf328d46p-1}, {-0x1.9ef7943a8ed8ap-2, 0x1.d4134d14dc93ap-1},
    {-0x1.b5d1009e15cc0p-2, 0x1.ced7af43cc773p-1}, {-0x1.cc66e9931c45ep-2, 0x1.c954b213411f5p-1},
    {-0x1.e2b5d3806f63bp-2, 0x1.c38b2f180bdb1p-1}, {-0x1.f8ba4dbf89abap-2, 0x1.bd7c0ac6f952ap-1},
    {-0x1.073879922ffeep-1, 0x1.b728345196e3ep-1}, {-0x1.11eb3541b4b23p-1, 0x1.b090a58150200p-1},
    {-0x1.1c73b39ae68c8p-1, 0x1.a9b66290ea1a3p-1}, {-0x1.26d054cdd12dfp-1, 0x1.a29a7a0462782p-1},
    {-0x1.30ff7fce17035p-1, 0x1.9b3e047f38741p-1}, {-0x1.3affa292050b9p-1, 0x1.93a22499263fbp-1},
    {-0x1.44cf325091dd6p-1, 0x1.8bc806b151741p-1}, {-0x1.4e6cabbe3e5e9p-1, 0x1.83b0e0bff976ep-1},
    {-0x1.57d69348ceca0p-1, 0x1.7b5df226aafafp-1}, {-0x1.610b7551d2cdfp-1, 0x1.72d0837efff96p-1},
    {-0x1.6a09e667f3bcdp-1, 0x1.6a09e667f3bcdp-1}, {-0x1.72d0837efff96p-1, 0x1.610b7551d2cdfp-1},
    {-0x1.7b5df226aafafp-1, 0x1.57d69348ceca0p-1}, {-0x1.83b0e0bff976ep-1, 0x1.4e6cabbe3e5e9p-1},
    {-0x1.8bc806b151741p-1, 0x1.44cf325091dd6p-1}, {-0x1.93a22499263fbp-1, 0x1.3affa292050b9p-1},
    {-0x1.9b3e047f38741p-1, 0x1.30ff7fce17035p-1}, {-0x1.a29a7a0462782p-1, 0x1.26d054cdd12dfp-1},
    {-0x1.a9b66290ea1a3p-1, 0x1.1c73b39ae68c8p-1}, {-0x1.b090a58150200p-1, 0x1.11eb3541b4b23p-1},
    {-0x1.b728345196e3ep-1, 0x1.073879922ffeep-1}, {-0x1.bd7c0ac6f952ap-1, 0x1.f8ba4dbf89abap-2},
    {-0x1.c38b2f180bdb1p-1, 0x1.e2b5d3806f63bp-2}, {-0x1.c954b213411f5p-1, 0x1.cc66e9931c45ep-2},
    {-0x1.ced7af43cc773p-1, 0x1.b5d1009e15cc0p-2}, {-0x1.d4134d14dc93ap-1, 0x1.9ef7943a8ed8ap-2},
    {-0x1.d906bcf328d46p-1, 0x1.87de2a6aea963p-2}, {-0x1.ddb13b6ccc23cp-1, 0x1.7088530fa459fp-2},
    {-0x1.e212104f686e5p-1, 0x1.58f9a75ab1fddp-2}, {-0x1.e6288ec48e112p-1, 0x1.4135c94176601p-2},
    {-0x1.e9f4156c62ddap-1, 0x1.294062ed59f06p-2}, {-0x1.ed740e7684963p-1, 0x1.111d262b1f677p-2},
    {-0x1.f0a7efb9230d7p-1, 0x1.f19f97b215f1bp-3}, {-0x1.f38f3ac64e589p-1, 0x1.c0b826a7e4f63p-3},
    {-0x1.f6297cff75cb0p-1, 0x1.8f8b83c69a60bp-3}, {-0x1.f8764fa714ba9p-1, 0x1.5e214448b3fc6p-3},
    {-0x1.fa7557f08a517p-1, 0x1.2c8106e8e613ap-3}, {-0x1.fc26470e19fd3p-1, 0x1.f564e56a9730ep-4},
    {-0x1.fd88da3d12526p-1, 0x1.917a6bc29b42cp-4}, {-0x1.fe9cdad01883ap-1, 0x1.2d52092ce19f6p-4},
    {-0x1.ff621e3796d7ep-1, 0x1.91f65f10dd814p-5}, {-0x1.ffd886084cd0dp-1, 0x1.92155f7a3667ep-6},
    {-0x1.0000000000000p+0, 0x0.0p+0}, {-0x1.ffd886084cd0dp-1, -0x1.92155f7a3667ep-6},
    {-0x1.ff621e3796d7ep-1, -0x1.91f65f10dd814p-5}, {-0x1.fe9cdad01883ap-1, -0x1.2d52092ce19f6p-4},
    {-0x1.fd88da3d12526p-1, -0x1.917a6bc29b42cp-4}, {-0x1.fc26470e19fd3p-1, -0x1.f564e56a9730ep-4},
    {-0x1.fa7557f08a517p-1, -0x1.2c8106e8e613ap-3}, {-0x1.f8764fa714ba9p-1, -0x1.5e214448b3fc6p-3},
    {-0x1.f6297cff75cb0p-1, -0x1.8f8b83c69a60bp-3}, {-0x1.f38f3ac64e589p-1, -0x1.c0b826a7e4f63p-3},
    {-0x1.f0a7efb9230d7p-1, -0x1.f19f97b215f1bp-3}, {-0x1.ed740e7684963p-1, -0x1.111d262b1f677p-2},
    {-0x1.e9f4156c62ddap-1, -0x1.294062ed59f06p-2}, {-0x1.e6288ec48e112p-1, -0x1.4135c94176601p-2},
    {-0x1.e212104f686e5p-1, -0x1.58f9a75ab1fddp-2}, {-0x1.ddb13b6ccc23cp-1, -0x1.7088530fa459fp-2},
    {-0x1.d906bcf328d46p-1, -0x1.87de2a6aea963p-2}, {-0x1.d4134d14dc93ap-1, -0x1.9ef7943a8ed8ap-2},
    {-0x1.ced7af43cc773p-1, -0x1.b5d1009e15cc0p-2}, {-0x1.c954b213411f5p-1, -0x1.cc66e9931c45ep-2},
    {-0x1.c38b2f180bdb1p-1, -0x1.e2b5d3806f63bp-2}, {-0x1.bd7c0ac6f952ap-1, -0x1.f8ba4dbf89abap-2},
    {-0x1.b728345196e3ep-1, -0x1.073879922ffeep-1}, {-0x1.b090a58150200p-1, -0x1.11eb3541b4b23p-1},
    {-0x1.a9b66290ea1a3p-1, -0x1.1c73b39ae68c8p-1}, {-0x1.a29a7a0462782p-1, -0x1.26d054cdd12dfp-1},
    {-0x1.9b3e047f38741p-1, -0x1.30ff7fce17035p-1}, {-0x1.93a22499263fbp-1, -0x1.3affa292050b9p-1},
    {-0x1.8bc806b151741p-1, -0x1.44cf325091dd6p-1}, {-0x1.83b0e0bff976ep-1, -0x1.4e6cabbe3e5e9p-1},
    {-0x1.7b5df226aafafp-1, -0x1.57d69348ceca0p-1}, {-0x1.72d0837efff96p-1, -0x1.610b7551d2cdfp-1},
    {-0x1.6a09e667f3bcdp-1, -0x1.6a09e667f3bcdp-1}, {-0x1.610b7551d2cdfp-1, -0x1.72d0837efff96p-1},
    {-0x1.57d69348ceca0p-1, -0x1.7b5df226aafafp-1}, {-0x1.4e6cabbe3e5e9p-1, -0x1.83b0e0bff976ep-1},
    {-0x1.44cf325091dd6p-1, -0x1.8bc806b151741p-1}, {-0x1.3affa292050b9p-1, -0x1.93a22499263fbp-1},
    {-0x1.30ff7fce17035p-1, -0x1.9b3e047f38741p-1}, {-0x1.26d054cdd12dfp-1, -0x1.a29a7a0462782p-1},
    {-0x1.1c73b39ae68c8p-1, -0x1.a9b66290ea1a3p-1}, {-0x1.11eb3541b4b23p-1, -0x1.b090a58150200p-1},
    {-0x1.073879922ffeep-1, -0x1.b728345196e3ep-1}, {-0x1.f8ba4dbf89abap-2, -0x1.bd7c0ac6f952ap-1},
    {-0x1.e2b5d3806f63bp-2, -0x1.c38b2f180bdb1p-1}, {-0x1.cc66e9931c45ep-2, -0x1.c954b213411f5p-1},
    {-0x1.b5d1009e15cc0p-2, -0x1.ced7af43cc773p-1}, {-0x1.9ef7943a8ed8ap-2, -0x1.d4134d14dc93ap-1},
    {-0x1.87de2a6aea963p-2, -0x1.d906bcf328d46p-1}, {-0x1.7088530fa459fp-2, -0x1.ddb13b6ccc23cp-1},
    {-0x1.58f9a75ab1fddp-2, -0x1.e212104f686e5p-1}, {-0x1.4135c94176601p-2, -0x1.e6288ec48e112p-1},
    {-0x1.294062ed59f06p-2, -0x1.e9f4156c62ddap-1}, {-0x1.111d262b1f677p-2, -0x1.ed740e7684963p-1},
    {-0x1.f19f97b215f1bp-3, -0x1.f0a7efb9230d7p-1}, {-0x1.c0b826a7e4f63p-3, -0x1.f38f3ac64e589p-1},
    {-0x1.8f8b83c69a60bp-3, -0x1.f6297cff75cb0p-1}, {-0x1.5e214448b3fc6p-3, -0x1.f8764fa714ba9p-1},
    {-0x1.2c8106e8e613ap-3, -0x1.fa7557f08a517p-1}, {-0x1.f564e56a9730ep-4, -0x1.fc26470e19fd3p-1},
    {-0x1.917a6bc29b42cp-4, -0x1.fd88da3d12526p-1}, {-0x1.2d52092ce19f6p-4, -0x1.fe9cdad01883ap-1},
    {-0x1.91f65f10dd814p-5, -0x1.ff621e3796d7ep-1}, {-0x1.92155f7a3667ep-6, -0x1.ffd886084cd0dp-1},
    {0x0.0p+0, -0x1.0000000000000p+0}, {0x1.92155f7a3667ep-6, -0x1.ffd886084cd0dp-1},
    {0x1.91f65f10dd814p-5, -0x1.ff621e3796d7ep-1}, {0x1.2d52092ce19f6p-4, -0x1.fe9cdad01883ap-1},
    {0x1.917a6bc29b42cp-4, -0x1.fd88da3d12526p-1}, {0x1.f564e56a9730ep-4, -0x1.fc26470e19fd3p-1},
    {0x1.2c8106e8e613ap-3, -0x1.fa7557f08a517p-1}, {0x1.5e214448b3fc6p-3, -0x1.f8764fa714ba9p-1},
    {0x1.8f8b83c69a60bp-3, -0x1.f6297cff75cb0p-1}, {0x1.c0b826a7e4f63p-3, -0x1.f38f3ac64e589p-1},
    {0x1.f19f97b215f1bp-3, -0x1.f0a7efb9230d7p-1}, {0x1.111d262b1f677p-2, -0x1.ed740e7684963p-1},
    {0x1.294062ed59f06p-2, -0x1.e9f4156c62ddap-1}, {0x1.4135c94176601p-2, -0x1.e6288ec48e112p-1},
    {0x1.58f9a75ab1fddp-2, -0x1.e212104f686e5p-1}, {0x1.7088530fa459fp-2, -0x1.ddb13b6ccc23cp-1},
    {0x1.87de2a6aea963p-2, -0x1.d906bcf328d46p-1}, {0x1.9ef7943a8ed8ap-2, -0x1.d4134d14dc93ap-1},
    {0x1.b5d1009e15cc0p-2, -0x1.ced7af43cc773p-1}, {0x1.cc66e9931c45ep-2, -0x1.c954b213411f5p-1},
    {0x1.e2b5d3806f63bp-2, -0x1.c38b2f180bdb1p-1}, {0x1.f8ba4dbf89abap-2, -0x1.bd7c0ac6f952ap-1},
    {0x1.073879922ffeep-1, -0x1.b728345196e3ep-1}, {0x1.11eb3541b4b23p-1, -0x1.b090a58150200p-1},
    {0x1.1c73b39ae68c8p-1, -0x1.a9b66290ea1a3p-1}, {0x1.26d054cdd12dfp-1, -0x1.a29a7a0462782p-1},
    {0x1.30ff7fce17035p-1, -0x1.9b3e047f38741p-1}, {0x1.3affa292050b9p-1, -0x1.93a22499263fbp-1},
    {0x1.44cf325091dd6p-1, -0x1.8bc806b151741p-1}, {0x1.4e6cabbe3e5e9p-1, -0x1.83b0e0bff976ep-1},
    {0x1.57d69348ceca0p-1, -0x1.7b5df226aafafp-1}, {0x1.610b7551d2cdfp-1, -0x1.72d0837efff96p-1},
    {0x1.6a09e667f3bcdp-1, -0x1.6a09e667f3bcdp-1}, {0x1.72d0837efff96p-1, -0x1.610b7551d2cdfp-1},
    {0x1.7b5df226aafafp-1, -0x1.57d69348ceca0p-1}, {0x1.83b0e0bff976ep-1, -0x1.4e6cabbe3e5e9p-1},
    {0x1.8bc806b151741p-1, -0x1.44cf325091dd6p-1}, {0x1.93a22499263fbp-1, -0x1.3affa292050b9p-1},
    {0x1.9b3e047f38741p-1, -0x1.30ff7fce17035p-1}, {0x1.a29a7a0462782p-1, -0x1.26d054cdd12dfp-1},
    {0x1.a9b66290ea1a3p-1, -0x1.1c73b39ae68c8p-1}, {0x1.b090a58150200p-1, -0x1.11eb3541b4b23p-1},
    {0x1.b728345196e3ep-1, -0x1.073879922ffeep-1}, {0x1.bd7c0ac6f952ap-1, -0x1.f8ba4dbf89abap-2},
    {0x1.c38b2f180bdb1p-1, -0x1.e2b5d3806f63bp-2}, {0x1.c954b213411f5p-1, -0x1.cc66e9931c45ep-2},
    {0x1.ced7af43cc773p-1, -0x1.b5d1009e15cc0p-2}, {0x1.d4134d14dc93ap-1, -0x1.9ef7943a8ed8ap-2},
    {0x1.d906bcf328d46p-1, -0x1.87de2a6aea963p-2}, {0x1.ddb13b6ccc23cp-1, -0x1.7088530fa459fp-2},
    {0x1.e212104f686e5p-1, -0x1.58f9a75ab1fddp-2}, {0x1.e6288ec48e112p-1, -0x1.4135c94176601p-2},
    {0x1.e9f4156c62ddap-1, -0x1.294062ed59f06p-2}, {0x1.ed740e7684963p-1, -0x1.111d262b1f677p-2},
    {0x1.f0a7efb9230d7p-1, -0x1.f19f97b215f1bp-3}, {0x1.f38f3ac64e589p-1, -0x1.c0b826a7e4f63p-3},
    {0x1.f6297cff75cb0p-1, -0x1.8f8b83c69a60bp-3}, {0x1.f8764fa714ba9p-1, -0x1.5e214448b3fc6p-3},
    {0x1.fa7557f08a517p-1, -0x1.2c8106e8e613ap-3}, {0x1.fc26470e19fd3p-1, -0x1.f564e56a9730ep-4},
    {0x1.fd88da3d12526p-1, -0x1.917a6bc29b42cp-4}, {0x1.fe9cdad01883ap-1, -0x1.2d52092ce19f6p-4},
    {0x1.ff621e3796d7ep-1, -0x1.91f65f10dd814p-5}, {0x1.ffd886084cd0dp-1, -0x1.92155f7a3667ep-6}};
static __constant__ double kSCT256[9] = {
    40.743665431525205957, 6755399441055744.0,                    // 128/pi, 1.5 * 2^52
    -0x1.921fb54400000p+0 / 64.0, -0x1.0b4611a626331p-34 / 64.0,  // -(pi/128 hi, lo)
    8.33333333333333333333e-03, -1.66666666666666666667e-01,      // sin r^5, r^3
    -1.38888888888888888889e-03, 4.16666666666666666667e-02, -0.5};  // cos r^6, r^4, r^2

__device__ __forceinline__ void sincos_tab256(double th, const double2* __restrict__ T, double* sn, double* cs) {
  const double t = fma(th, kSCT256[0], kSCT256[1]);
  const double kd = t - kSCT256[1];
  double r = fma(kd, kSCT256[2], th);
  r = fma(kd, kSCT256[3], r);
  const double z = r * r;
  const double sr = fma(r * z, fma(z, kSCT256[4], kSCT256[5]), r);
  const double cr = fma(z, fma(z, fma(z, kSCT256[6], kSCT256[7]), kSCT256[8]), 1.0);
  const double2 cs_k = T[__double2loint(t) & 255];
  *sn = fma(cs_k.y, cr, cs_k.x * sr);
  *cs = fma(cs_k.x, cr, -(cs_k.y * sr));
}

}  // namespace fast
}  // namespace bem
