// oracle/oracle.cpp -- TEST INFRASTRUCTURE ONLY.
//
// Plain, slow, obviously-correct FP64 CPU implementation of the multi-frequency
// H^2 + ACA single-layer apply of D. Seibel, "Boundary Element Methods for the
// Wave Equation based on Hierarchical Matrices and Adaptive Cross Approximation"
// (arXiv 2006.05186, /root/reference/PAPER.md, cited as P:<line>).
//
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
// reference legs may load this library.  It shares no code, header, table or
// constant generator with the CUDA library under paper_2006_05186_b200/ ; the
// pinned arithmetic (pexp / psincos / reduction order) is written here
// independently from the specification in DESIGN.md §"Pinned arithmetic".
//
// Build: g++ -O2 -ffp-contract=off -fopenmp -shared -fPIC (see oracle/build.py).
// -ffp-contract=off is REQUIRED: the ACA pivots must be bit-identical to the
// GPU library (SURVEY.md §8(c) C10 reading 5b).
//
// Modes: DENSE (V_l fully by the collocation rule C3), H2ONLY (exact coupling
// matrices per frequency), H2ACA (couplings compressed across
// frequency by MACA, Alg. 2, eq:lrfinal P:1404-1410).
//
// Parity status per function: every function below is pinned by a
// `-m "not gpu"` test in tests/test_oracle_*.py.
#include <algorithm>
#include <cmath>
#include <complex>
#include <cstdint>
#include <cstring>
#include <vector>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef std::complex<double> cplx;
static const double PI = 3.14159265358979323846;
static const double FOURPI = 0x1.921fb54442d18p+3;

// ---------------------------------------------------------------------------
// C1. Panel geometry (flat triangles).  7-point degree-5 rule
// (north_star; the paper is silent on quadrature).
// ---------------------------------------------------------------------------
struct Rule7 {
  double lam[7][3];
  double w[7];
  Rule7() {
    double s15 = std::sqrt(15.0);
    double a1 = (9.0 - 2.0 * s15) / 21.0, b1 = (6.0 + s15) / 21.0;
    double a2 = (9.0 + 2.0 * s15) / 21.0, b2 = (6.0 - s15) / 21.0;
    double w1 = (155.0 + s15) / 1200.0, w2 = (155.0 - s15) / 1200.0;
    double t[7][3] = {{1.0 / 3.0, 1.0 / 3.0, 1.0 / 3.0},
                      {a1, b1, b1}, {b1, a1, b1}, {b1, b1, a1},
                      {a2, b2, b2}, {b2, a2, b2}, {b2, b2, a2}};
    double ww[7] = {9.0 / 40.0, w1, w1, w1, w2, w2, w2};
    for (int q = 0; q < 7; ++q) {
      for (int a = 0; a < 3; ++a) lam[q][a] = t[q][a];
      w[q] = ww[q];
    }
  }
};
static const Rule7 RULE;

struct Geometry {
  int64_t M = 0;
  std::vector<double> cen, area, node, J, lo, hi;  // cen M*3, node M*7*3, lo/hi M*3
  std::vector<double> nrm;                           // M*3 unit normal (b-a) x (c-a) / |.| (vertex order)
};

// J(T) = int_T dS(y)/|c-y| for c the centroid (in-plane point), summed over
// the three edge sub-triangles: d*(asinh(tB/d)-asinh(tA/d)).
static double self_integral(const double* A0, const double* B0, const double* C0) {
  double c[3];
  for (int a = 0; a < 3; ++a) c[a] = ((A0[a] + B0[a]) + C0[a]) / 3.0;
  const double* V[3] = {A0, B0, C0};
  double J = 0.0;
  for (int e = 0; e < 3; ++e) {
    const double* A = V[e];
    const double* B = V[(e + 1) % 3];
    double u[3], len = 0.0;
    for (int a = 0; a < 3; ++a) { u[a] = B[a] - A[a]; len += u[a] * u[a]; }
    len = std::sqrt(len);
    for (int a = 0; a < 3; ++a) u[a] /= len;
    double tA = 0.0, tB = 0.0;
    for (int a = 0; a < 3; ++a) { tA += (A[a] - c[a]) * u[a]; tB += (B[a] - c[a]) * u[a]; }
    double d2 = 0.0;
    for (int a = 0; a < 3; ++a) { double f = A[a] - tA * u[a] - c[a]; d2 += f * f; }
    double d = std::sqrt(d2);
    J += d * (std::asinh(tB / d) - std::asinh(tA / d));
  }
  return J;
}

static void make_geometry(const double* V, const int32_t* T, int64_t M, Geometry& g) {
  g.M = M;
  g.cen.resize(M * 3); g.area.resize(M); g.node.resize(M * 21); g.J.resize(M);
  g.lo.resize(M * 3); g.hi.resize(M * 3); g.nrm.resize(M * 3);
  for (int64_t i = 0; i < M; ++i) {
    const double* a = V + 3 * (int64_t)T[3 * i + 0];
    const double* b = V + 3 * (int64_t)T[3 * i + 1];
    const double* c = V + 3 * (int64_t)T[3 * i + 2];
    for (int k = 0; k < 3; ++k) {
      g.cen[3 * i + k] = ((a[k] + b[k]) + c[k]) / 3.0;
      g.lo[3 * i + k] = std::min(std::min(a[k], b[k]), c[k]);
      g.hi[3 * i + k] = std::max(std::max(a[k], b[k]), c[k]);
    }
    double e1[3], e2[3];
    for (int k = 0; k < 3; ++k) { e1[k] = b[k] - a[k]; e2[k] = c[k] - a[k]; }
    double cr[3] = {e1[1] * e2[2] - e1[2] * e2[1], e1[2] * e2[0] - e1[0] * e2[2],
                    e1[0] * e2[1] - e1[1] * e2[0]};
    g.area[i] = 0.5 * std::sqrt((cr[0] * cr[0] + cr[1] * cr[1]) + cr[2] * cr[2]);
    for (int k = 0; k < 3; ++k) g.nrm[3 * i + k] = cr[k] / (2.0 * g.area[i]);
    for (int q = 0; q < 7; ++q)
      for (int k = 0; k < 3; ++k)
        g.node[21 * i + 3 * q + k] = (q == 0) ? g.cen[3 * i + k]
            : (RULE.lam[q][0] * a[k] + RULE.lam[q][1] * b[k]) + RULE.lam[q][2] * c[k];
    g.J[i] = self_integral(a, b, c);
  }
}

// ---------------------------------------------------------------------------
// C2. Kernel k(r;s) = e^{-sr}/(4 pi r), eq:fundsol P:479-482 (libm tier).
// ---------------------------------------------------------------------------
static inline cplx kernel(double r, cplx s) {
  double E = std::exp(-(s.real() * r));
  double th = s.imag() * r;
  double inv = 1.0 / (FOURPI * r);
  return cplx(E * std::cos(th) * inv, -(E * std::sin(th)) * inv);
}

// phi(s,r) = (e^{-sr}-1)/r, phi(s,0) = -s; cancellation-free form.
static inline cplx phi_self(double r, cplx s) {
  if (r == 0.0) return -s;
  double x = -(s.real() * r), y = -(s.imag() * r);
  double sh = std::sin(0.5 * y);
  double re = std::expm1(x) * std::cos(y) - 2.0 * sh * sh;
  double im = std::exp(x) * std::sin(y);
  return cplx(re / r, im / r);
}

// C3. Collocation entry V_l[i,j] (centroid collocation, P0 density).
static cplx entry(const Geometry& g, int64_t i, int64_t j, cplx s) {
  const double* ci = &g.cen[3 * i];
  cplx acc(0.0, 0.0);
  if (i != j) {
    for (int q = 0; q < 7; ++q) {
      const double* y = &g.node[21 * j + 3 * q];
      double dx = ci[0] - y[0], dy = ci[1] - y[1], dz = ci[2] - y[2];
      double r = std::sqrt((dx * dx + dy * dy) + dz * dz);
      acc += RULE.w[q] * kernel(r, s) * FOURPI;  // e^{-sr}/r
    }
    return acc * (g.area[j] / FOURPI);
  }
  for (int q = 0; q < 7; ++q) {
    const double* y = &g.node[21 * j + 3 * q];
    double dx = ci[0] - y[0], dy = ci[1] - y[1], dz = ci[2] - y[2];
    double r = std::sqrt((dx * dx + dy * dy) + dz * dz);
    acc += RULE.w[q] * phi_self(r, s);
  }
  return (g.J[i] + g.area[i] * acc) / FOURPI;
}

// NEXT-1: double-layer operator K(s) of eq:wavebio (P:301-303,
// gamma_{1,y} applied to the fundamental solution), collocation analogue:
//   dk(x,y,n_y;s) = d/dn_y e^{-s|x-y|}/(4 pi |x-y|) = -(1+s r) e^{-s r} ((y-x).n_y)/(4 pi r^3),
//   K_l[i,j] = |T_j| sum_q w_q dk(c_i, y_{j,q}, n_j; s_l)  (i != j),
//   K_l[i,i] = 0 (flat panel: (y - c_i).n_i = 0 on the panel's own plane).
static cplx entry_dl(const Geometry& g, int64_t i, int64_t j, cplx s) {
  if (i == j) return cplx(0.0, 0.0);
  const double* ci = &g.cen[3 * i];
  const double* n = &g.nrm[3 * j];
  cplx acc(0.0, 0.0);
  for (int q = 0; q < 7; ++q) {
    const double* y = &g.node[21 * j + 3 * q];
    double dx = y[0] - ci[0], dy = y[1] - ci[1], dz = y[2] - ci[2];
    double r = std::sqrt((dx * dx + dy * dy) + dz * dz);
    double dn = (dx * n[0] + dy * n[1]) + dz * n[2];
    acc += RULE.w[q] * (-(1.0 + s * r) * std::exp(-s * r) * (dn / (r * r * r)));
  }
  return acc * (g.area[j] / FOURPI);
}

// ---------------------------------------------------------------------------
// Pinned arithmetic: used for every value the
// ACA reads, so that pivots are bit-reproducible (SURVEY C10 reading 5b).
// Only IEEE +,-,*,/,sqrt and fma; no contraction (-ffp-contract=off).
// ---------------------------------------------------------------------------
static const double P_SHIFT = 0x1.8p+52;
static const double P_INVLN2 = 0x1.71547652b82fep+0;
static const double P_LN2HI = 0x1.62e42fee00000p-1;
static const double P_LN2LO = 0x1.a39ef35793c76p-33;
static const double P_2OPI = 0x1.45f306dc9c883p-1;
static const double P_PIO2_1 = 0x1.921fb54400000p+0;
static const double P_PIO2_2 = 0x1.0b4611a600000p-34;
static const double P_PIO2_3 = 0x1.3198a2e000000p-69;
// 1/k!, k = 0..19, correctly rounded.
static const double P_INVFACT[20] = {
    0x1.0000000000000p+0, 0x1.0000000000000p+0, 0x1.0000000000000p-1, 0x1.5555555555555p-3,
    0x1.5555555555555p-5, 0x1.1111111111111p-7, 0x1.6c16c16c16c17p-10, 0x1.a01a01a01a01ap-13,
    0x1.a01a01a01a01ap-16, 0x1.71de3a556c734p-19, 0x1.27e4fb7789f5cp-22, 0x1.ae64567f544e4p-26,
    0x1.1eed8eff8d898p-29, 0x1.6124613a86d09p-33, 0x1.93974a8c07c9dp-37, 0x1.ae7f3e733b81fp-41,
    0x1.ae7f3e733b81fp-45, 0x1.952c77030ad4ap-49, 0x1.6827863b97d97p-53, 0x1.2f49b46814157p-57};

static inline double pow2i(int k) {  // exact 2^k for -1022 <= k <= 1023
  uint64_t bits = (uint64_t)(k + 1023) << 52;
  double d;
  std::memcpy(&d, &bits, 8);
  return d;
}

static double pexp(double x) {
  if (x < -746.0) return 0.0;
  if (x > 709.5) return HUGE_VAL;
  double t = std::fma(x, P_INVLN2, P_SHIFT);
  double kd = t - P_SHIFT;
  double r = std::fma(kd, -P_LN2HI, x);
  r = std::fma(kd, -P_LN2LO, r);
  double p = P_INVFACT[13];
  for (int j = 12; j >= 0; --j) p = std::fma(p, r, P_INVFACT[j]);
  int k = (int)kd;
  if (k >= -1021) return p * pow2i(k);
  return (p * pow2i(k + 200)) * pow2i(-200);
}

static void psincos(double th, double* sn, double* cs) {
  double t = std::fma(th, P_2OPI, P_SHIFT);
  double qd = t - P_SHIFT;
  double r = std::fma(qd, -P_PIO2_1, th);
  r = std::fma(qd, -P_PIO2_2, r);
  r = std::fma(qd, -P_PIO2_3, r);
  double z = r * r;
  // sin r = r * sum_{k=0..8} (-1)^k z^k/(2k+1)!
  double ps = P_INVFACT[17];
  ps = std::fma(ps, z, -P_INVFACT[15]);
  ps = std::fma(ps, z, P_INVFACT[13]);
  ps = std::fma(ps, z, -P_INVFACT[11]);
  ps = std::fma(ps, z, P_INVFACT[9]);
  ps = std::fma(ps, z, -P_INVFACT[7]);
  ps = std::fma(ps, z, P_INVFACT[5]);
  ps = std::fma(ps, z, -P_INVFACT[3]);
  ps = std::fma(ps, z, P_INVFACT[1]);
  double s = r * ps;
  // cos r = sum_{k=0..9} (-1)^k z^k/(2k)!
  double pc = -P_INVFACT[18];
  pc = std::fma(pc, z, P_INVFACT[16]);
  pc = std::fma(pc, z, -P_INVFACT[14]);
  pc = std::fma(pc, z, P_INVFACT[12]);
  pc = std::fma(pc, z, -P_INVFACT[10]);
  pc = std::fma(pc, z, P_INVFACT[8]);
  pc = std::fma(pc, z, -P_INVFACT[6]);
  pc = std::fma(pc, z, P_INVFACT[4]);
  pc = std::fma(pc, z, -P_INVFACT[2]);
  pc = std::fma(pc, z, P_INVFACT[0]);
  double c = pc;
  switch ((int)((int64_t)qd & 3)) {
    case 0: *sn = s; *cs = c; break;
    case 1: *sn = c; *cs = -s; break;
    case 2: *sn = -s; *cs = -c; break;
    default: *sn = -c; *cs = s; break;
  }
}

struct C2 { double re, im; };
static inline C2 pmul(C2 a, C2 b) { return {a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re}; }
static inline C2 pmulconj(C2 a, C2 b) { return {a.re * b.re + a.im * b.im, a.im * b.re - a.re * b.im}; }
static inline C2 psub(C2 a, C2 b) { return {a.re - b.re, a.im - b.im}; }
static inline C2 pdiv(C2 a, C2 c) {
  double den = c.re * c.re + c.im * c.im;
  return {(a.re * c.re + a.im * c.im) / den, (a.im * c.re - a.re * c.im) / den};
}
static inline double pkey(C2 a) { return a.re * a.re + a.im * a.im; }

static C2 pkernel(double r, C2 s) {
  double E = pexp(-(s.re * r));
  double sn, cs;
  psincos(s.im * r, &sn, &cs);
  double inv = 1.0 / (FOURPI * r);
  return {(E * cs) * inv, -((E * sn) * inv)};
}

// Pinned expm1 (self entry of the NEAR tensor, Alg. 3 P:1414-1453 / NEXT-4):
// |x| < 1/2: x * sum_{k=1..19} x^{k-1}/k! (Horner in fma); else pexp(x) - 1.
static double pexpm1(double x) {
  if (x > -0.5 && x < 0.5) {
    double q = P_INVFACT[19];
    for (int j = 18; j >= 1; --j) q = std::fma(q, x, P_INVFACT[j]);
    return x * q;
  }
  return pexp(x) - 1.0;
}

// Pinned phi(s,r) = (e^{-sr}-1)/r, r > 0, in the cancellation-free form of C3:
// Re = expm1(x) cos y - 2 sin^2(y/2), Im = e^x sin y, z = x + iy = -s r.
static C2 pphi(double r, C2 s) {
  double x = -(s.re * r), y = -(s.im * r);
  double sy, cy, sh, chh;
  psincos(y, &sy, &cy);
  psincos(0.5 * y, &sh, &chh);
  double re = pexpm1(x) * cy - 2.0 * (sh * sh);
  double im = pexp(x) * sy;
  return {re / r, im / r};
}

static const double INV4PI = 0x1.45f306dc9c883p-4;  // 1/(4 pi), correctly rounded

// Pinned collocation entry V(s)[i,j] of C3 (the NEAR procedure of Alg. 3,
// P:1444-1450, collocation reading): every value the near-field MACA reads.
//   i != j: sum_{q=0..6} (w_q |T_j|) * pkernel(|y_{j,q} - c_i|; s), q ascending;
//   i == j: ((J_i + |T_i| acc.re) / 4pi, (|T_i| acc.im) / 4pi) with
//           acc = sum_q w_q phi_q, phi_0 = -s (node 0 is the centroid), phi_q = pphi(r_q, s).
static C2 pentry(const Geometry& g, int64_t i, int64_t j, C2 s) {
  const double* ci = &g.cen[3 * i];
  double ar = 0.0, ai = 0.0;
  if (i != j) {
    for (int q = 0; q < 7; ++q) {
      const double* y = &g.node[21 * j + 3 * q];
      double dx = y[0] - ci[0], dy = y[1] - ci[1], dz = y[2] - ci[2];
      double r = std::sqrt((dx * dx + dy * dy) + dz * dz);
      C2 k = pkernel(r, s);
      double wa = RULE.w[q] * g.area[j];
      ar = ar + wa * k.re;
      ai = ai + wa * k.im;
    }
    return {ar, ai};
  }
  ar = ar + RULE.w[0] * (-s.re);
  ai = ai + RULE.w[0] * (-s.im);
  for (int q = 1; q < 7; ++q) {
    const double* y = &g.node[21 * j + 3 * q];
    double dx = y[0] - ci[0], dy = y[1] - ci[1], dz = y[2] - ci[2];
    double r = std::sqrt((dx * dx + dy * dy) + dz * dz);
    C2 f = pphi(r, s);
    ar = ar + RULE.w[q] * f.re;
    ai = ai + RULE.w[q] * f.im;
  }
  return {(g.J[i] + g.area[i] * ar) * INV4PI, (g.area[i] * ai) * INV4PI};
}

// Pinned summation: sequential within chunks of 32, then left to right.
// (Four chunks are summed side by side -- each still strictly in order -- so the
// loop has independent chains; the result is the same as chunk after chunk.)
static double psum(const std::vector<double>& v) {
  double tot = 0.0;
  size_t n = v.size();
  size_t c0 = 0;
  for (; c0 + 128 <= n; c0 += 128) {
    double s[4] = {0.0, 0.0, 0.0, 0.0};
    for (size_t i = 0; i < 32; ++i)
      for (int u = 0; u < 4; ++u) s[u] = s[u] + v[c0 + 32 * u + i];
    for (int u = 0; u < 4; ++u) tot = tot + s[u];
  }
  for (; c0 < n; c0 += 32) {
    double s = 0.0;
    size_t c1 = std::min(n, c0 + 32);
    for (size_t i = c0; i < c1; ++i) s = s + v[i];
    tot = tot + s;
  }
  return tot;
}

// ---------------------------------------------------------------------------
// C4. CQM frequencies s_l = delta(R e^{-2 pi i l/L})/dt, eq:cqm_freq
// P:443-447 with the north_star sign; L = N+1; s_{L-l} := conj(s_l).
// ---------------------------------------------------------------------------
static void frequencies(int N, double T, double R, int method, std::vector<C2>& s) {
  int L = N + 1;
  s.assign(L, C2{0.0, 0.0});
  double dt = T / (double)N;
  int half = L / 2;
  for (int l = 0; l <= half; ++l) {
    double ang = (2.0 * PI * (double)l) / (double)L;
    double zr = R * std::cos(ang), zi = -(R * std::sin(ang));
    if (l == 0) { zr = R; zi = 0.0; }
    double dr, di;
    if (method == 1) {  // BDF1: delta = 1 - zeta
      dr = 1.0 - zr; di = -zi;
    } else {            // BDF2: delta = 3/2 - 2 zeta + zeta^2/2
      double z2r = zr * zr - zi * zi, z2i = 2.0 * (zr * zi);
      dr = (1.5 - 2.0 * zr) + 0.5 * z2r;
      di = (-2.0 * zi) + 0.5 * z2i;
    }
    s[l] = C2{dr / dt, di / dt};
    if (l == 0) s[l].im = 0.0;
  }
  for (int l = half + 1; l < L; ++l) s[l] = C2{s[L - l].re, -s[L - l].im};
}

// ---------------------------------------------------------------------------
// C6. Cluster tree: tight vertex boxes, longest-axis midpoint
// bisection on centroids, stable partition, median fallback, DFS pre-order.
// ---------------------------------------------------------------------------
struct Cluster {
  int begin, end, son0, son1, level, parent;
  double lo[3], hi[3];
};

struct H2 {
  Geometry g;
  int nmin, m, p;
  double eta;
  std::vector<int> perm;  // perm[k] = input index of the k-th panel in cluster order
  std::vector<Cluster> cl;
  std::vector<int> nearR, nearC, farR, farC;
  // bases (cluster order): U[k*p+mu], W[k*p+nu]; E[c*p*p + lam*p + mu] = E_{c,parent(c)}
  std::vector<double> U, W, E, xi;  // xi[c*3*m + a*m + k]
  std::vector<double> WK;           // double-layer column basis: |T_j| sum_q w_q n_j . grad L_nu(y_q)
  // ACA result per far block
  std::vector<int> rank, pivk, pivq;
  std::vector<int64_t> pivoff, zoff;
  std::vector<C2> Z;   // per far block r x zld: the coefficients of the kept frequencies
  std::vector<int> zcol;  // zcol[l] = column of frequency l in Z (-1: not kept); zld = #kept
  int zld = 0;
  std::vector<C2> s;  // frequencies used by the ACA
  int L = 0;
  bool aca_done = false;
  // near-field MACA per near block (Alg. 3 NEAR branch, BEM_MODE_COMBINED / NEXT-4)
  std::vector<int> nrank, npivk, npivq;
  std::vector<int64_t> npivoff, nzoff;
  std::vector<C2> nZ;
  std::vector<int64_t> nsoff;  // pivot slices C_{b,t} = V_{k_t}[b] (the tensor C_b of eq:lrfinal), t-major
  std::vector<C2> nS;
  bool near_done = false;
  // time-domain weight coefficients dhat (NEXT-2), rows as in Z / nZ
  std::vector<cplx> tDf, tDn;
  bool tw_done = false;
};

static void build_cluster(H2& h, int begin, int end, int level, int parent) {
  int id = (int)h.cl.size();
  h.cl.push_back(Cluster{begin, end, -1, -1, level, parent, {0, 0, 0}, {0, 0, 0}});
  Cluster c = h.cl[id];
  for (int a = 0; a < 3; ++a) { c.lo[a] = HUGE_VAL; c.hi[a] = -HUGE_VAL; }
  for (int k = begin; k < end; ++k) {
    int i = h.perm[k];
    for (int a = 0; a < 3; ++a) {
      c.lo[a] = std::min(c.lo[a], h.g.lo[3 * i + a]);
      c.hi[a] = std::max(c.hi[a], h.g.hi[3 * i + a]);
    }
  }
  h.cl[id] = c;
  int n = end - begin;
  if (n <= h.nmin) return;
  int ax = 0;
  for (int a = 1; a < 3; ++a)
    if (c.hi[a] - c.lo[a] > c.hi[ax] - c.lo[ax]) ax = a;
  double mid = 0.5 * (c.lo[ax] + c.hi[ax]);
  std::vector<int> left, right;
  for (int k = begin; k < end; ++k) {
    int i = h.perm[k];
    if (h.g.cen[3 * i + ax] < mid) left.push_back(i); else right.push_back(i);
  }
  if (left.empty() || right.empty()) {
    std::vector<int> all(h.perm.begin() + begin, h.perm.begin() + end);
    std::stable_sort(all.begin(), all.end(), [&](int x, int y) {
      return h.g.cen[3 * x + ax] < h.g.cen[3 * y + ax];
    });
    left.assign(all.begin(), all.begin() + n / 2);
    right.assign(all.begin() + n / 2, all.end());
  }
  int k = begin;
  for (int i : left) h.perm[k++] = i;
  for (int i : right) h.perm[k++] = i;
  int split = begin + (int)left.size();
  h.cl[id].son0 = (int)h.cl.size();
  build_cluster(h, begin, split, level + 1, id);
  h.cl[id].son1 = (int)h.cl.size();
  build_cluster(h, split, end, level + 1, id);
}

// C7. Admissibility eq:qadm with squared norms, equality admissible.
static bool admissible(const Cluster& r, const Cluster& c, double eta) {
  double dr[3], dc[3], gap[3];
  for (int a = 0; a < 3; ++a) {
    dr[a] = r.hi[a] - r.lo[a];
    dc[a] = c.hi[a] - c.lo[a];
    double g1 = c.lo[a] - r.hi[a], g2 = r.lo[a] - c.hi[a];
    gap[a] = std::max(0.0, std::max(g1, g2));
  }
  double diag_r = (dr[0] * dr[0] + dr[1] * dr[1]) + dr[2] * dr[2];
  double diag_c = (dc[0] * dc[0] + dc[1] * dc[1]) + dc[2] * dc[2];
  double dist = (gap[0] * gap[0] + gap[1] * gap[1]) + gap[2] * gap[2];
  return std::max(diag_r, diag_c) <= (eta * eta) * dist;
}

static void partition(H2& h, int r, int c) {
  const Cluster& R = h.cl[r];
  const Cluster& C = h.cl[c];
  if (admissible(R, C, h.eta)) { h.farR.push_back(r); h.farC.push_back(c); return; }
  bool lr = R.son0 < 0, lc = C.son0 < 0;
  if (lr && lc) { h.nearR.push_back(r); h.nearC.push_back(c); return; }
  if (!lr && !lc) {
    int r0 = R.son0, r1 = R.son1, c0 = C.son0, c1 = C.son1;
    partition(h, r0, c0); partition(h, r0, c1); partition(h, r1, c0); partition(h, r1, c1);
  } else if (!lr) {
    int r0 = R.son0, r1 = R.son1;
    partition(h, r0, c); partition(h, r1, c);
  } else {
    int c0 = C.son0, c1 = C.son1;
    partition(h, r, c0); partition(h, r, c1);
  }
}

// ---------------------------------------------------------------------------
// C8. Chebyshev interpolation and cluster bases.
// ---------------------------------------------------------------------------
static void cluster_nodes(const Cluster& c, int m, double* xi /*3*m*/) {
  double dd[3];
  for (int a = 0; a < 3; ++a) dd[a] = c.hi[a] - c.lo[a];
  double diag = std::sqrt((dd[0] * dd[0] + dd[1] * dd[1]) + dd[2] * dd[2]);
  for (int a = 0; a < 3; ++a) {
    double lo = c.lo[a], hi = c.hi[a];
    if (hi - lo == 0.0) { lo = lo - 1e-8 * diag; hi = hi + 1e-8 * diag; }
    double mid = 0.5 * (lo + hi), half = 0.5 * (hi - lo);
    for (int k = 0; k < m; ++k) {
      double x = std::cos(((double)(2 * k + 1) * PI) / (double)(2 * m));
      xi[a * m + k] = mid + half * x;
    }
  }
}

static double lagrange1(const double* nodes, int m, int k, double t) {
  double v = 1.0;
  for (int j = 0; j < m; ++j)
    if (j != k) v *= (t - nodes[j]) / (nodes[k] - nodes[j]);
  return v;
}

// L_{c,mu}(x), mu = kx + m ky + m^2 kz
static double lagrange3(const double* xi, int m, int mu, const double* x) {
  int kx = mu % m, ky = (mu / m) % m, kz = mu / (m * m);
  return lagrange1(xi, m, kx, x[0]) * lagrange1(xi + m, m, ky, x[1]) *
         lagrange1(xi + 2 * m, m, kz, x[2]);
}

// d/dt of the 1-D Lagrange polynomial l_k(t)
static double dlagrange1(const double* nodes, int m, int k, double t) {
  double sum = 0.0;
  for (int i = 0; i < m; ++i) {
    if (i == k) continue;
    double v = 1.0 / (nodes[k] - nodes[i]);
    for (int j = 0; j < m; ++j)
      if (j != k && j != i) v *= (t - nodes[j]) / (nodes[k] - nodes[j]);
    sum += v;
  }
  return sum;
}

// n . grad L_{c,mu}(x)
static double dlagrange3n(const double* xi, int m, int mu, const double* x, const double* n) {
  int kx = mu % m, ky = (mu / m) % m, kz = mu / (m * m);
  double lx = lagrange1(xi, m, kx, x[0]), ly = lagrange1(xi + m, m, ky, x[1]), lz = lagrange1(xi + 2 * m, m, kz, x[2]);
  double gx = dlagrange1(xi, m, kx, x[0]) * ly * lz;
  double gy = lx * dlagrange1(xi + m, m, ky, x[1]) * lz;
  double gz = lx * ly * dlagrange1(xi + 2 * m, m, kz, x[2]);
  return (n[0] * gx + n[1] * gy) + n[2] * gz;
}

static void node_point(const double* xi, int m, int mu, double* out) {
  out[0] = xi[mu % m];
  out[1] = xi[m + (mu / m) % m];
  out[2] = xi[2 * m + mu / (m * m)];
}

static void build_bases(H2& h) {
  int m = h.m, p = h.p;
  int C = (int)h.cl.size();
  int64_t M = h.g.M;
  h.xi.assign((size_t)C * 3 * m, 0.0);
  for (int c = 0; c < C; ++c) cluster_nodes(h.cl[c], m, &h.xi[(size_t)c * 3 * m]);
  h.U.assign((size_t)M * p, 0.0);
  h.W.assign((size_t)M * p, 0.0);
  h.WK.assign((size_t)M * p, 0.0);
  for (int c = 0; c < C; ++c) {
    const Cluster& cc = h.cl[c];
    if (cc.son0 >= 0) continue;
    const double* xi = &h.xi[(size_t)c * 3 * m];
    for (int k = cc.begin; k < cc.end; ++k) {
      int i = h.perm[k];
      for (int mu = 0; mu < p; ++mu) {
        h.U[(size_t)k * p + mu] = lagrange3(xi, m, mu, &h.g.cen[3 * i]);
        double acc = 0.0;
        for (int q = 0; q < 7; ++q) acc += RULE.w[q] * lagrange3(xi, m, mu, &h.g.node[21 * i + 3 * q]);
        h.W[(size_t)k * p + mu] = h.g.area[i] * acc;
        double acck = 0.0;
        for (int q = 0; q < 7; ++q)
          acck += RULE.w[q] * dlagrange3n(xi, m, mu, &h.g.node[21 * i + 3 * q], &h.g.nrm[3 * i]);
        h.WK[(size_t)k * p + mu] = h.g.area[i] * acck;
      }
    }
  }
  h.E.assign((size_t)C * p * p, 0.0);
  for (int c = 0; c < C; ++c) {
    int par = h.cl[c].parent;
    if (par < 0) continue;
    const double* xs = &h.xi[(size_t)c * 3 * m];
    const double* xp = &h.xi[(size_t)par * 3 * m];
    for (int lam = 0; lam < p; ++lam) {
      double pt[3];
      node_point(xs, m, lam, pt);
      for (int mu = 0; mu < p; ++mu) h.E[(size_t)c * p * p + (size_t)lam * p + mu] = lagrange3(xp, m, mu, pt);
    }
  }
}

// ---------------------------------------------------------------------------
// C10. MACA per far block (Alg. 2) on the mode-3 unfolding
// (Remark P:1322-1334), pinned arithmetic, used pivots excluded (AM15),
// stopping rule P:1288 with the Gram identity P:1302-1308, last term kept
// (AM13).  Stored: pivots (k_l, q_l) and Z = U^{-1} D^T.
// ---------------------------------------------------------------------------
static C2 aca_entry(const double* xr, const double* xc, int m, int p, int q, const std::vector<C2>& s, int l) {
  int L = (int)s.size(), half = L / 2;
  bool mir = l > half;
  int ll = mir ? L - l : l;
  int mu = q / p, nu = q % p;
  double a[3], b[3];
  node_point(xr, m, mu, a);
  node_point(xc, m, nu, b);
  double dx = b[0] - a[0], dy = b[1] - a[1], dz = b[2] - a[2];
  double r = std::sqrt((dx * dx + dy * dy) + dz * dz);
  C2 v = pkernel(r, s[ll]);
  if (mir) v.im = -v.im;
  return v;
}

struct AcaOut {
  std::vector<int> k, q;
  std::vector<C2> Z;  // r x L
  int fragile = 0;
};

// Generic MACA on an entry callback A(q,l), q < pp, l < L (Alg. 2).
template <class Entry>
static void aca_generic(Entry A, int pp, int L, double eps, AcaOut& out, std::vector<double>* nrm_hist = nullptr,
                        std::vector<std::vector<C2>>* Cout = nullptr, std::vector<std::vector<C2>>* Dout = nullptr) {
  int rmax = std::min(L, pp);
  std::vector<std::vector<C2>> Cs, Ds;
  std::vector<char> usedq(pp, 0), usedk(L, 0);
  std::vector<C2> c(pp), e(L), d(L);
  std::vector<double> tmp, tmp2;
  int k = 0;
  double nrm2 = 0.0;
  out.k.clear(); out.q.clear(); out.Z.clear(); out.fragile = 0;
  for (;;) {
    int ell = (int)Cs.size();
    // c[q] = A(q,k) - sum_{j<ell} d_j[k] c_j[q], subtracted in increasing j for every q
    // (loop order j-outer only so that the q loop vectorises; each c[q] sees the same ops)
    for (int q = 0; q < pp; ++q) c[q] = A(q, k);
    for (int j = 0; j < ell; ++j) {
      const C2 dk = Ds[j][k];
      const C2* cj = Cs[j].data();
      for (int q = 0; q < pp; ++q) c[q] = psub(c[q], pmul(dk, cj[q]));
    }
    int qs = -1;
    double best = -1.0, second = -1.0;
    for (int q = 0; q < pp; ++q) {
      if (usedq[q]) continue;
      double kk = pkey(c[q]);
      if (kk > best) { second = best; best = kk; qs = q; }
      else if (kk > second) second = kk;
    }
    if (qs < 0 || best == 0.0) break;
    if (second >= 0.0 && best - second <= 0x1p-44 * best) out.fragile++;
    C2 piv = c[qs];
    for (int l = 0; l < L; ++l) e[l] = A(qs, l);
    for (int j = 0; j < ell; ++j) {  // e[l] -= c_j[q*] d_j[l], increasing j (as above)
      const C2 cq = Cs[j][qs];
      const C2* dj = Ds[j].data();
      for (int l = 0; l < L; ++l) e[l] = psub(e[l], pmul(cq, dj[l]));
    }
    for (int l = 0; l < L; ++l) d[l] = pdiv(e[l], piv);
    tmp.resize(pp);
    for (int q = 0; q < pp; ++q) tmp[q] = pkey(c[q]);
    double nc2 = psum(tmp);
    tmp.resize(L);
    for (int l = 0; l < L; ++l) tmp[l] = pkey(d[l]);
    double nd2 = psum(tmp);
    double cross = 0.0;
    for (int j = 0; j < ell; ++j) {
      tmp.resize(pp); tmp2.resize(pp);
      for (int q = 0; q < pp; ++q) { C2 t = pmulconj(Cs[j][q], c[q]); tmp[q] = t.re; tmp2[q] = t.im; }
      C2 gc = {psum(tmp), psum(tmp2)};
      tmp.resize(L); tmp2.resize(L);
      for (int l = 0; l < L; ++l) { C2 t = pmulconj(Ds[j][l], d[l]); tmp[l] = t.re; tmp2[l] = t.im; }
      C2 gd = {psum(tmp), psum(tmp2)};
      cross = cross + (gc.re * gd.re - gc.im * gd.im);
    }
    nrm2 = nrm2 + (nc2 * nd2 + 2.0 * cross);
    if (nrm2 < 0.0) nrm2 = 0.0;
    if (nrm_hist) nrm_hist->push_back(nrm2);
    Cs.push_back(c); Ds.push_back(d);
    out.k.push_back(k); out.q.push_back(qs);
    usedq[qs] = 1; usedk[k] = 1;
    int rank = ell + 1;
    if (std::sqrt(nc2) * std::sqrt(nd2) <= eps * std::sqrt(nrm2) || rank == rmax) break;
    int kn = -1;
    best = -1.0;
    for (int l = 0; l < L; ++l) {
      if (usedk[l]) continue;
      double kk = pkey(e[l]);
      if (kk > best) { best = kk; kn = l; }
    }
    if (kn < 0) break;
    k = kn;
  }
  // Z = U^{-1} D^T, U[l][j] = d_l[k_j] (unit upper triangular), back substitution.
  int r = (int)Ds.size();
  out.Z.assign((size_t)r * L, C2{0.0, 0.0});
  for (int l = r - 1; l >= 0; --l) {
    for (int t = 0; t < L; ++t) {
      C2 acc = Ds[l][t];
      for (int j = l + 1; j < r; ++j) acc = psub(acc, pmul(Ds[l][out.k[j]], out.Z[(size_t)j * L + t]));
      out.Z[(size_t)l * L + t] = acc;
    }
  }
  if (Cout) *Cout = Cs;
  if (Dout) *Dout = Ds;
}

static void aca_block(const double* xr, const double* xc, int m, int p, const std::vector<C2>& s, double eps,
                      AcaOut& out) {
  aca_generic([&](int q, int l) { return aca_entry(xr, xc, m, p, q, s, l); }, p * p, (int)s.size(), eps, out);
}

// ---------------------------------------------------------------------------
// C11. The apply y_l = V_l x_l in three modes (eq:lrfinal P:1404-1410).
// ---------------------------------------------------------------------------
// MODE_COMBINED: Alg. 3 in full (eq:lrfinal P:1404-1410): MACA skeletons on the
// far blocks (P+) AND on the near blocks (P-: V[b] ~ C_b x_3 D_b), NEXT-4.
enum { MODE_DENSE = 0, MODE_H2ONLY = 1, MODE_H2ACA = 2, MODE_COMBINED = 3 };

// Entry q = a_loc * n_c + k_loc, frequency l of the near block tensor V[b]
// (block b = (R, C) of P-, rows/cols in cluster order), pinned; l > L/2 is the
// conjugate of l' = L - l (C2 reading: mirrored values are defined, not evaluated).
static C2 near_aca_entry(const H2& h, size_t b, int q, const std::vector<C2>& s, int l) {
  int L = (int)s.size(), half = L / 2;
  bool mir = l > half;
  int ll = mir ? L - l : l;
  const Cluster& R = h.cl[h.nearR[b]];
  const Cluster& Cc = h.cl[h.nearC[b]];
  int nc = Cc.end - Cc.begin;
  int a = R.begin + q / nc, k = Cc.begin + q % nc;
  C2 v = pentry(h.g, h.perm[a], h.perm[k], s[ll]);
  if (mir) v.im = -v.im;
  return v;
}

// op = 0: single layer V(s_l); op = 1: double layer K(s_l) (NEXT-1): the same
// coupling tensors and ACA, column basis WK and near entries entry_dl.
static void apply_one(const H2& h, int mode, cplx s_l, int l, const std::vector<cplx>& sl_all,
                      const cplx* x_in, cplx* y_out, int op = 0) {
  auto ent = [&](int64_t i, int64_t j) { return op == 0 ? entry(h.g, i, j, s_l) : entry_dl(h.g, i, j, s_l); };
  const std::vector<double>& Wc = op == 0 ? h.W : h.WK;
  int64_t M = h.g.M;
  int p = h.p, m = h.m, C = (int)h.cl.size();
  std::vector<cplx> x(M), y(M, cplx(0.0, 0.0));
  for (int64_t k = 0; k < M; ++k) x[k] = x_in[h.perm[k]];
  if (mode == MODE_DENSE) {
    for (int64_t a = 0; a < M; ++a) {
      cplx acc(0.0, 0.0);
      for (int64_t b = 0; b < M; ++b) acc += ent(h.perm[a], h.perm[b]) * x[b];
      y[a] = acc;
    }
  } else {
    // upward pass: leaves xhat = W^T x|_c, parents xhat = sum E^T xhat_son
    std::vector<cplx> xh((size_t)C * p, cplx(0.0, 0.0)), yh((size_t)C * p, cplx(0.0, 0.0));
    for (int c = C - 1; c >= 0; --c) {  // pre-order numbering: sons have larger ids
      const Cluster& cc = h.cl[c];
      cplx* out = &xh[(size_t)c * p];
      if (cc.son0 < 0) {
        for (int nu = 0; nu < p; ++nu) {
          cplx acc(0.0, 0.0);
          for (int k = cc.begin; k < cc.end; ++k) acc += Wc[(size_t)k * p + nu] * x[k];
          out[nu] = acc;
        }
      } else {
        for (int son : {cc.son0, cc.son1}) {
          const double* Es = &h.E[(size_t)son * p * p];
          for (int mu = 0; mu < p; ++mu) {
            cplx acc(0.0, 0.0);
            for (int lam = 0; lam < p; ++lam) acc += Es[(size_t)lam * p + mu] * xh[(size_t)son * p + lam];
            out[mu] += acc;
          }
        }
      }
    }
    // coupling
    std::vector<cplx> S((size_t)p * p);
    for (size_t b = 0; b < h.farR.size(); ++b) {
      int r = h.farR[b], c = h.farC[b];
      const double* xr = &h.xi[(size_t)r * 3 * m];
      const double* xc = &h.xi[(size_t)c * 3 * m];
      std::fill(S.begin(), S.end(), cplx(0.0, 0.0));
      if (mode == MODE_H2ONLY) {
        for (int mu = 0; mu < p; ++mu)
          for (int nu = 0; nu < p; ++nu) {
            double a[3], bb[3];
            node_point(xr, m, mu, a); node_point(xc, m, nu, bb);
            double dx = bb[0] - a[0], dy = bb[1] - a[1], dz = bb[2] - a[2];
            S[(size_t)mu * p + nu] = kernel(std::sqrt((dx * dx + dy * dy) + dz * dz), s_l);
          }
      } else {
        int rb = h.rank[b];
        for (int t = 0; t < rb; ++t) {
          int kk = h.pivk[h.pivoff[b] + t];
          C2 z = h.Z[h.zoff[b] + (size_t)t * h.zld + h.zcol[l]];
          cplx zc(z.re, z.im);
          for (int mu = 0; mu < p; ++mu)
            for (int nu = 0; nu < p; ++nu) {
              double a[3], bb[3];
              node_point(xr, m, mu, a); node_point(xc, m, nu, bb);
              double dx = bb[0] - a[0], dy = bb[1] - a[1], dz = bb[2] - a[2];
              S[(size_t)mu * p + nu] += zc * kernel(std::sqrt((dx * dx + dy * dy) + dz * dz), sl_all[kk]);
            }
        }
      }
      for (int mu = 0; mu < p; ++mu) {
        cplx acc(0.0, 0.0);
        for (int nu = 0; nu < p; ++nu) acc += S[(size_t)mu * p + nu] * xh[(size_t)c * p + nu];
        yh[(size_t)r * p + mu] += acc;
      }
    }
    // downward pass: yhat_son += E yhat_parent; leaves y += U yhat
    for (int c = 0; c < C; ++c) {
      const Cluster& cc = h.cl[c];
      if (cc.parent >= 0) {
        const double* Es = &h.E[(size_t)c * p * p];
        for (int lam = 0; lam < p; ++lam) {
          cplx acc(0.0, 0.0);
          for (int mu = 0; mu < p; ++mu) acc += Es[(size_t)lam * p + mu] * yh[(size_t)cc.parent * p + mu];
          yh[(size_t)c * p + lam] += acc;
        }
      }
      if (cc.son0 < 0) {
        for (int k = cc.begin; k < cc.end; ++k) {
          cplx acc(0.0, 0.0);
          for (int mu = 0; mu < p; ++mu) acc += h.U[(size_t)k * p + mu] * yh[(size_t)c * p + mu];
          y[k] += acc;
        }
      }
    }
    // near field
    for (size_t b = 0; b < h.nearR.size(); ++b) {
      const Cluster& R = h.cl[h.nearR[b]];
      const Cluster& Cc = h.cl[h.nearC[b]];
      if (mode == MODE_COMBINED && op == 0) {
        // V_l[b] ~ sum_t Z_b[t,l] V_{k_t}[b] (skeleton form of eq:maca, pivot slices pinned)
        const int nr = R.end - R.begin, nc = Cc.end - Cc.begin;
        for (int t = 0; t < h.nrank[b]; ++t) {
          const C2* S = &h.nS[h.nsoff[b] + (size_t)t * nr * nc];  // V_{k_t}[b], row-major
          const C2 z = h.nZ[h.nzoff[b] + (size_t)t * h.L + l];
          const cplx zc(z.re, z.im);
          for (int a = R.begin; a < R.end; ++a) {
            cplx acc(0.0, 0.0);
            for (int k = Cc.begin; k < Cc.end; ++k) {
              const C2 v = S[(size_t)(a - R.begin) * nc + (k - Cc.begin)];
              acc += cplx(v.re, v.im) * x[k];
            }
            y[a] += zc * acc;
          }
        }
        continue;
      }
      for (int a = R.begin; a < R.end; ++a) {
        cplx acc(0.0, 0.0);
        for (int k = Cc.begin; k < Cc.end; ++k) acc += ent(h.perm[a], h.perm[k]) * x[k];
        y[a] += acc;
      }
    }
  }
  for (int64_t k = 0; k < M; ++k) y_out[h.perm[k]] = y[k];
}

// The same apply for several frequencies at once, parallel over row clusters /
// rows.  For every frequency the arithmetic and its order are exactly those of
// apply_one (tests check equality bit for bit); only the loop nesting differs:
// a far block's pivot slices S_b(s_{k_t}) are evaluated once and shared by the
// selected frequencies, and the row-parallel loops visit each row's blocks in
// ascending block order, as apply_one's sequential loop does.
// far_on / near_on (nullable): only these blocks contribute (a bounded sample of the
// work, for timing the oracle on workloads it cannot finish: bench.py cpu_baseline).
static void apply_multi(const H2& h, int mode, const std::vector<cplx>& sl_all, const int32_t* lsel, int nsel,
                        const cplx* x_in, cplx* y_out, int op, const char* far_on = nullptr,
                        const char* near_on = nullptr) {
  const int64_t M = h.g.M;
  const int p = h.p, m = h.m, C = (int)h.cl.size();
  const std::vector<double>& Wc = op == 0 ? h.W : h.WK;
  auto ent = [&](int64_t i, int64_t j, cplx s_l) { return op == 0 ? entry(h.g, i, j, s_l) : entry_dl(h.g, i, j, s_l); };
  std::vector<std::vector<cplx>> x(nsel), y(nsel), xh(nsel), yh(nsel);
#pragma omp parallel for schedule(dynamic, 1)
  for (int t = 0; t < nsel; ++t) {
    x[t].resize(M);
    y[t].assign(M, cplx(0.0, 0.0));
    for (int64_t k = 0; k < M; ++k) x[t][k] = x_in[(int64_t)t * M + h.perm[k]];
    if (mode == MODE_DENSE) continue;
    std::vector<cplx>& xt = xh[t];
    xt.assign((size_t)C * p, cplx(0.0, 0.0));
    yh[t].assign((size_t)C * p, cplx(0.0, 0.0));
    for (int c = C - 1; c >= 0; --c) {  // upward pass, as apply_one
      const Cluster& cc = h.cl[c];
      cplx* out = &xt[(size_t)c * p];
      if (cc.son0 < 0) {
        for (int nu = 0; nu < p; ++nu) {
          cplx acc(0.0, 0.0);
          for (int k = cc.begin; k < cc.end; ++k) acc += Wc[(size_t)k * p + nu] * x[t][k];
          out[nu] = acc;
        }
      } else {
        for (int son : {cc.son0, cc.son1}) {
          const double* Es = &h.E[(size_t)son * p * p];
          for (int mu = 0; mu < p; ++mu) {
            cplx acc(0.0, 0.0);
            for (int lam = 0; lam < p; ++lam) acc += Es[(size_t)lam * p + mu] * xt[(size_t)son * p + lam];
            out[mu] += acc;
          }
        }
      }
    }
  }
  if (mode == MODE_DENSE) {
#pragma omp parallel for schedule(dynamic, 8)
    for (int64_t a = 0; a < M; ++a)
      for (int t = 0; t < nsel; ++t) {
        const cplx s_l = sl_all[lsel[t]];
        cplx acc(0.0, 0.0);
        for (int64_t b = 0; b < M; ++b) acc += ent(h.perm[a], h.perm[b], s_l) * x[t][b];
        y[t][a] = acc;
      }
  } else {
    // coupling, parallel over row clusters
    std::vector<std::vector<int>> byrow(C);
    for (size_t b = 0; b < h.farR.size(); ++b)
      if (!far_on || far_on[b]) byrow[h.farR[b]].push_back((int)b);
    const int FCH = 32;  // frequencies per pass (bounds the per-thread S buffers)
#pragma omp parallel for schedule(dynamic, 1)
    for (int r = 0; r < C; ++r) {
      if (byrow[r].empty()) continue;
      std::vector<double> dist((size_t)p * p);
      std::vector<cplx> S((size_t)p * p * std::min(nsel, FCH));
      for (int b : byrow[r]) {
        const int c = h.farC[b];
        const double* xr = &h.xi[(size_t)r * 3 * m];
        const double* xc = &h.xi[(size_t)c * 3 * m];
        for (int mu = 0; mu < p; ++mu)
          for (int nu = 0; nu < p; ++nu) {
            double a[3], bb[3];
            node_point(xr, m, mu, a); node_point(xc, m, nu, bb);
            double dx = bb[0] - a[0], dy = bb[1] - a[1], dz = bb[2] - a[2];
            dist[(size_t)mu * p + nu] = std::sqrt((dx * dx + dy * dy) + dz * dz);
          }
        for (int t0 = 0; t0 < nsel; t0 += FCH) {
          const int nt = std::min(FCH, nsel - t0);
          std::fill(S.begin(), S.begin() + (size_t)p * p * nt, cplx(0.0, 0.0));
          if (mode == MODE_H2ONLY) {
            for (int t = 0; t < nt; ++t) {
              const cplx s_l = sl_all[lsel[t0 + t]];
              for (size_t e = 0; e < (size_t)p * p; ++e) S[(size_t)t * p * p + e] = kernel(dist[e], s_l);
            }
          } else {
            const int rb = h.rank[b];
            for (int j = 0; j < rb; ++j) {
              const int kk = h.pivk[h.pivoff[b] + j];
              for (size_t e = 0; e < (size_t)p * p; ++e) {
                const cplx kv = kernel(dist[e], sl_all[kk]);
                for (int t = 0; t < nt; ++t) {
                  const C2 z = h.Z[h.zoff[b] + (size_t)j * h.zld + h.zcol[lsel[t0 + t]]];
                  const cplx zc(z.re, z.im);
                  S[(size_t)t * p * p + e] += zc * kv;
                }
              }
            }
          }
          for (int t = 0; t < nt; ++t) {
            const cplx* St = &S[(size_t)t * p * p];
            const cplx* xc2 = &xh[t0 + t][(size_t)c * p];
            cplx* yr = &yh[t0 + t][(size_t)r * p];
            for (int mu = 0; mu < p; ++mu) {
              cplx acc(0.0, 0.0);
              for (int nu = 0; nu < p; ++nu) acc += St[(size_t)mu * p + nu] * xc2[nu];
              yr[mu] += acc;
            }
          }
        }
      }
    }
    // downward pass per frequency, as apply_one
#pragma omp parallel for schedule(dynamic, 1)
    for (int t = 0; t < nsel; ++t) {
      std::vector<cplx>& yt = yh[t];
      for (int c = 0; c < C; ++c) {
        const Cluster& cc = h.cl[c];
        if (cc.parent >= 0) {
          const double* Es = &h.E[(size_t)c * p * p];
          for (int lam = 0; lam < p; ++lam) {
            cplx acc(0.0, 0.0);
            for (int mu = 0; mu < p; ++mu) acc += Es[(size_t)lam * p + mu] * yt[(size_t)cc.parent * p + mu];
            yt[(size_t)c * p + lam] += acc;
          }
        }
        if (cc.son0 < 0) {
          for (int k = cc.begin; k < cc.end; ++k) {
            cplx acc(0.0, 0.0);
            for (int mu = 0; mu < p; ++mu) acc += h.U[(size_t)k * p + mu] * yt[(size_t)c * p + mu];
            y[t][k] += acc;
          }
        }
      }
    }
    // near field, parallel over row leaves (each row's blocks in ascending order)
    std::vector<std::vector<int>> nbyrow(C);
    for (size_t b = 0; b < h.nearR.size(); ++b)
      if (!near_on || near_on[b]) nbyrow[h.nearR[b]].push_back((int)b);
#pragma omp parallel for schedule(dynamic, 1)
    for (int rl = 0; rl < C; ++rl) {
      for (int b : nbyrow[rl]) {
        const Cluster& R = h.cl[h.nearR[b]];
        const Cluster& Cc = h.cl[h.nearC[b]];
        for (int t = 0; t < nsel; ++t) {
          const int l = lsel[t];
          if (mode == MODE_COMBINED && op == 0) {
            const int nr = R.end - R.begin, nc = Cc.end - Cc.begin;
            for (int j = 0; j < h.nrank[b]; ++j) {
              const C2* Sn = &h.nS[h.nsoff[b] + (size_t)j * nr * nc];
              const C2 z = h.nZ[h.nzoff[b] + (size_t)j * h.L + l];
              const cplx zc(z.re, z.im);
              for (int a = R.begin; a < R.end; ++a) {
                cplx acc(0.0, 0.0);
                for (int k = Cc.begin; k < Cc.end; ++k) {
                  const C2 v = Sn[(size_t)(a - R.begin) * nc + (k - Cc.begin)];
                  acc += cplx(v.re, v.im) * x[t][k];
                }
                y[t][a] += zc * acc;
              }
            }
            continue;
          }
          const cplx s_l = sl_all[l];
          for (int a = R.begin; a < R.end; ++a) {
            cplx acc(0.0, 0.0);
            for (int k = Cc.begin; k < Cc.end; ++k) acc += ent(h.perm[a], h.perm[k], s_l) * x[t][k];
            y[t][a] += acc;
          }
        }
      }
    }
  }
#pragma omp parallel for schedule(static)
  for (int t = 0; t < nsel; ++t)
    for (int64_t k = 0; k < M; ++k) y_out[(int64_t)t * M + h.perm[k]] = y[t][k];
}

// apply_one for a single frequency with the far-block coupling matrices S~_{b,l}
// and the near-block entries evaluated once (cached) and reused by every GMRES
// iteration; the arithmetic of each product and its order are those of
// apply_one, so the iterates are the same bit for bit (only far faster).
static void up_pass(const H2& h, const std::vector<cplx>& x, std::vector<cplx>& xh);
static void down_pass(const H2& h, std::vector<cplx>& yh, std::vector<cplx>& y);

struct OneFreqCache {
  std::vector<cplx> S;     // far blocks: p x p each, block order
  std::vector<cplx> Vn;    // near blocks: nr x nc each, block order
  std::vector<int64_t> noff;
  std::vector<std::vector<int>> fbyrow, nbyrow;
};

static void build_cache(const H2& h, int mode, cplx s_l, int l, const std::vector<cplx>& sl_all, OneFreqCache& k) {
  const int p = h.p, m = h.m, C = (int)h.cl.size();
  const size_t nfar = h.farR.size(), nnear = h.nearR.size();
  k.S.assign(nfar * p * p, cplx(0.0, 0.0));
#pragma omp parallel for schedule(dynamic, 16)
  for (int64_t b = 0; b < (int64_t)nfar; ++b) {
    const double* xr = &h.xi[(size_t)h.farR[b] * 3 * m];
    const double* xc = &h.xi[(size_t)h.farC[b] * 3 * m];
    cplx* S = &k.S[(size_t)b * p * p];
    for (int mu = 0; mu < p; ++mu)
      for (int nu = 0; nu < p; ++nu) {
        double a[3], bb[3];
        node_point(xr, m, mu, a); node_point(xc, m, nu, bb);
        double dx = bb[0] - a[0], dy = bb[1] - a[1], dz = bb[2] - a[2];
        const double r = std::sqrt((dx * dx + dy * dy) + dz * dz);
        if (mode == MODE_H2ONLY) {
          S[(size_t)mu * p + nu] = kernel(r, s_l);
        } else {
          for (int t = 0; t < h.rank[b]; ++t) {
            const C2 z = h.Z[h.zoff[b] + (size_t)t * h.zld + h.zcol[l]];
            S[(size_t)mu * p + nu] += cplx(z.re, z.im) * kernel(r, sl_all[h.pivk[h.pivoff[b] + t]]);
          }
        }
      }
  }
  k.noff.assign(nnear + 1, 0);
  for (size_t b = 0; b < nnear; ++b)
    k.noff[b + 1] = k.noff[b] + (int64_t)(h.cl[h.nearR[b]].end - h.cl[h.nearR[b]].begin) *
                                    (h.cl[h.nearC[b]].end - h.cl[h.nearC[b]].begin);
  k.Vn.assign((size_t)k.noff[nnear], cplx(0.0, 0.0));
#pragma omp parallel for schedule(dynamic, 16)
  for (int64_t b = 0; b < (int64_t)nnear; ++b) {
    const Cluster& R = h.cl[h.nearR[b]];
    const Cluster& Cc = h.cl[h.nearC[b]];
    const int nc = Cc.end - Cc.begin;
    for (int a = R.begin; a < R.end; ++a)
      for (int kk = Cc.begin; kk < Cc.end; ++kk)
        k.Vn[k.noff[b] + (size_t)(a - R.begin) * nc + (kk - Cc.begin)] = entry(h.g, h.perm[a], h.perm[kk], s_l);
  }
  k.fbyrow.assign(C, {});
  for (size_t b = 0; b < nfar; ++b) k.fbyrow[h.farR[b]].push_back((int)b);
  k.nbyrow.assign(C, {});
  for (size_t b = 0; b < nnear; ++b) k.nbyrow[h.nearR[b]].push_back((int)b);
}

static void apply_cached(const H2& h, const OneFreqCache& k, const cplx* x_in, cplx* y_out) {
  const int64_t M = h.g.M;
  const int p = h.p, C = (int)h.cl.size();
  std::vector<cplx> x(M), y(M, cplx(0.0, 0.0)), xh((size_t)C * p, cplx(0.0, 0.0)), yh((size_t)C * p, cplx(0.0, 0.0));
  for (int64_t i = 0; i < M; ++i) x[i] = x_in[h.perm[i]];
  up_pass(h, x, xh);
#pragma omp parallel for schedule(dynamic, 1)
  for (int r = 0; r < C; ++r)
    for (int b : k.fbyrow[r]) {
      const cplx* S = &k.S[(size_t)b * p * p];
      const int c = h.farC[b];
      for (int mu = 0; mu < p; ++mu) {
        cplx acc(0.0, 0.0);
        for (int nu = 0; nu < p; ++nu) acc += S[(size_t)mu * p + nu] * xh[(size_t)c * p + nu];
        yh[(size_t)r * p + mu] += acc;
      }
    }
  down_pass(h, yh, y);
#pragma omp parallel for schedule(dynamic, 1)
  for (int rl = 0; rl < C; ++rl)
    for (int b : k.nbyrow[rl]) {
      const Cluster& R = h.cl[h.nearR[b]];
      const Cluster& Cc = h.cl[h.nearC[b]];
      const int nc = Cc.end - Cc.begin;
      for (int a = R.begin; a < R.end; ++a) {
        cplx acc(0.0, 0.0);
        for (int kk = Cc.begin; kk < Cc.end; ++kk) acc += k.Vn[k.noff[b] + (size_t)(a - R.begin) * nc + (kk - Cc.begin)] * x[kk];
        y[a] += acc;
      }
    }
  for (int64_t i = 0; i < M; ++i) y_out[h.perm[i]] = y[i];
}

// ---------------------------------------------------------------------------
// C5. Transforms (eq:omega_n P:436-441, eq:slphelm P:529-540), reading D2.
// ---------------------------------------------------------------------------
// The twiddles e^{-+2 pi i idx/L} (idx = n l mod L) and R^n are tabulated once
// (the same values the naive loop evaluates per term); columns are processed in
// blocks of 16 and in parallel; every sum keeps its n-ascending order.
static void dft_tables(int L, double R, std::vector<cplx>& tw, std::vector<double>& Rn) {
  tw.resize(L);
  Rn.resize(L);
  for (int idx = 0; idx < L; ++idx) {
    double ang = (2.0 * PI * (double)idx) / (double)L;
    tw[idx] = cplx(std::cos(ang), std::sin(ang));
  }
  for (int n = 0; n < L; ++n) Rn[n] = std::pow(R, (double)n);
}

static void forward(const cplx* xt, cplx* xf, int64_t M, int N, double R) {
  int L = N + 1;
  std::vector<cplx> tw;
  std::vector<double> Rn;
  dft_tables(L, R, tw, Rn);
  const int64_t nb = (M + 15) / 16;
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t ib = 0; ib < nb; ++ib) {
    const int64_t i0 = ib * 16, w = std::min<int64_t>(16, M - i0);
    std::vector<cplx> xb((size_t)L * 16);
    for (int n = 0; n < L; ++n)
      for (int64_t ii = 0; ii < w; ++ii) xb[(size_t)n * 16 + ii] = xt[(int64_t)n * M + i0 + ii];
    for (int l = 0; l < L; ++l) {
      cplx acc[16];
      for (int64_t ii = 0; ii < w; ++ii) acc[ii] = cplx(0.0, 0.0);
      for (int n = 0; n < L; ++n) {
        int64_t idx = ((int64_t)n * l) % L;
        const cplx e(tw[idx].real(), -tw[idx].imag());
        for (int64_t ii = 0; ii < w; ++ii) acc[ii] += Rn[n] * xb[(size_t)n * 16 + ii] * e;
      }
      for (int64_t ii = 0; ii < w; ++ii) xf[(int64_t)l * M + i0 + ii] = acc[ii];
    }
  }
}

static void inverse(const cplx* yf, cplx* yt, int64_t M, int N, double R) {
  int L = N + 1;
  std::vector<cplx> tw;
  std::vector<double> Rn;
  dft_tables(L, R, tw, Rn);
  const int64_t nb = (M + 15) / 16;
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t ib = 0; ib < nb; ++ib) {
    const int64_t i0 = ib * 16, w = std::min<int64_t>(16, M - i0);
    std::vector<cplx> yb((size_t)L * 16);
    for (int l = 0; l < L; ++l)
      for (int64_t ii = 0; ii < w; ++ii) yb[(size_t)l * 16 + ii] = yf[(int64_t)l * M + i0 + ii];
    for (int n = 0; n < L; ++n) {
      cplx acc[16];
      for (int64_t ii = 0; ii < w; ++ii) acc[ii] = cplx(0.0, 0.0);
      for (int l = 0; l < L; ++l) {
        int64_t idx = ((int64_t)n * l) % L;
        for (int64_t ii = 0; ii < w; ++ii) acc[ii] += yb[(size_t)l * 16 + ii] * tw[idx];
      }
      const double sc = std::pow(R, -(double)n) / (double)L;
      for (int64_t ii = 0; ii < w; ++ii) yt[(int64_t)n * M + i0 + ii] = acc[ii] * sc;
    }
  }
}

// ---------------------------------------------------------------------------
// C12. GMRES(restart) per frequency, x0 = 0, CGS with one reorthogonalisation,
// complex Givens rotations; stop at ||b - A x|| <= tol ||b|| (Remark
// P:1607-1614; reading D10).
// ---------------------------------------------------------------------------
template <class Op>
static int gmres(Op op, int64_t M, const cplx* b, cplx* x, double tol, int restart, int maxit, double* relres) {
  auto nrm = [&](const std::vector<cplx>& v) {
    double s = 0.0;
    for (auto& z : v) s += std::norm(z);
    return std::sqrt(s);
  };
  std::vector<cplx> bb(b, b + M), xx(M, cplx(0.0, 0.0)), r(M), w(M);
  double bn = nrm(bb);
  int it = 0;
  *relres = 0.0;
  if (bn == 0.0) { std::fill(x, x + M, cplx(0.0, 0.0)); return 0; }
  std::vector<std::vector<cplx>> V(restart + 1, std::vector<cplx>(M));
  std::vector<cplx> H((size_t)(restart + 1) * restart), g(restart + 1), cs(restart), sn(restart);
  for (;;) {
    op(xx.data(), w.data());
    for (int64_t i = 0; i < M; ++i) r[i] = bb[i] - w[i];
    double beta = nrm(r);
    *relres = beta / bn;
    if (beta <= tol * bn || it >= maxit) break;
    for (int64_t i = 0; i < M; ++i) V[0][i] = r[i] / beta;
    std::fill(g.begin(), g.end(), cplx(0.0, 0.0));
    g[0] = beta;
    int j = 0;
    for (; j < restart; ++j) {
      op(V[j].data(), w.data());
      ++it;
      for (int pass = 0; pass < 2; ++pass) {
        std::vector<cplx> hc(j + 1);
        for (int i = 0; i <= j; ++i) {
          cplx acc(0.0, 0.0);
          for (int64_t k = 0; k < M; ++k) acc += std::conj(V[i][k]) * w[k];
          hc[i] = acc;
        }
        for (int i = 0; i <= j; ++i) {
          for (int64_t k = 0; k < M; ++k) w[k] -= hc[i] * V[i][k];
          H[(size_t)i * restart + j] += hc[i];
        }
      }
      double hn = nrm(w);
      H[(size_t)(j + 1) * restart + j] = hn;
      if (hn > 0.0)
        for (int64_t k = 0; k < M; ++k) V[j + 1][k] = w[k] / hn;
      for (int i = 0; i < j; ++i) {
        cplx a = H[(size_t)i * restart + j], bq = H[(size_t)(i + 1) * restart + j];
        H[(size_t)i * restart + j] = cs[i] * a + sn[i] * bq;
        H[(size_t)(i + 1) * restart + j] = -std::conj(sn[i]) * a + cs[i] * bq;
      }
      cplx a = H[(size_t)j * restart + j], bq = H[(size_t)(j + 1) * restart + j];
      double den = std::sqrt(std::norm(a) + std::norm(bq));
      if (den == 0.0) { cs[j] = 1.0; sn[j] = 0.0; }
      else if (std::abs(a) == 0.0) { cs[j] = 0.0; sn[j] = std::conj(bq) / std::abs(bq); }
      else {
        cs[j] = std::abs(a) / den;
        sn[j] = (a / std::abs(a)) * std::conj(bq) / den;
      }
      H[(size_t)j * restart + j] = cs[j] * a + sn[j] * bq;
      H[(size_t)(j + 1) * restart + j] = 0.0;
      g[j + 1] = -std::conj(sn[j]) * g[j];
      g[j] = cs[j] * g[j];
      if (std::abs(g[j + 1]) <= tol * bn || it >= maxit) { ++j; break; }
    }
    std::vector<cplx> yv(j);
    for (int i = j - 1; i >= 0; --i) {
      cplx acc = g[i];
      for (int k2 = i + 1; k2 < j; ++k2) acc -= H[(size_t)i * restart + k2] * yv[k2];
      yv[i] = acc / H[(size_t)i * restart + i];
    }
    for (int i = 0; i < j; ++i)
      for (int64_t k = 0; k < M; ++k) xx[k] += yv[i] * V[i][k];
    std::fill(H.begin(), H.end(), cplx(0.0, 0.0));
  }
  std::copy(xx.begin(), xx.end(), x);
  return it;
}

// ===========================================================================
// C interface (ctypes)
// ===========================================================================
extern "C" {

int orc_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

void orc_set_threads(int n) {
#ifdef _OPENMP
  if (n > 0) omp_set_num_threads(n);
#else
  (void)n;
#endif
}

void orc_geometry(const double* V, const int32_t* T, int64_t M, double* cen, double* area, double* node,
                  double* wq, double* J) {
  Geometry g;
  make_geometry(V, T, M, g);
  std::memcpy(cen, g.cen.data(), sizeof(double) * M * 3);
  std::memcpy(area, g.area.data(), sizeof(double) * M);
  std::memcpy(node, g.node.data(), sizeof(double) * M * 21);
  std::memcpy(J, g.J.data(), sizeof(double) * M);
  for (int q = 0; q < 7; ++q) wq[q] = RULE.w[q];
}

double orc_self_integral(const double* a, const double* b, const double* c) { return self_integral(a, b, c); }

void orc_kernel(double r, double sre, double sim, double* out) {
  cplx v = kernel(r, cplx(sre, sim));
  out[0] = v.real(); out[1] = v.imag();
}

void orc_kernel_pinned(double r, double sre, double sim, double* out) {
  C2 v = pkernel(r, C2{sre, sim});
  out[0] = v.re; out[1] = v.im;
}

void orc_phi_self(double r, double sre, double sim, double* out) {
  cplx v = phi_self(r, cplx(sre, sim));
  out[0] = v.real(); out[1] = v.imag();
}

void orc_pexp_n(const double* x, double* y, int64_t n) { for (int64_t i = 0; i < n; ++i) y[i] = pexp(x[i]); }
void orc_psincos_n(const double* t, double* s, double* c, int64_t n) {
  for (int64_t i = 0; i < n; ++i) psincos(t[i], &s[i], &c[i]);
}
double orc_psum(const double* v, int64_t n) { return psum(std::vector<double>(v, v + n)); }

void orc_frequencies(int32_t N, double T, double R, int32_t method, double* s_out) {
  std::vector<C2> s;
  frequencies(N, T, R, method, s);
  for (int l = 0; l <= N; ++l) { s_out[2 * l] = s[l].re; s_out[2 * l + 1] = s[l].im; }
}

// Dense matrix V(s) in input order (row i = collocation point c_i).
void orc_dense_matrix(const double* V, const int32_t* T, int64_t M, double sre, double sim, double* A) {
  Geometry g;
  make_geometry(V, T, M, g);
  cplx s(sre, sim);
#pragma omp parallel for schedule(dynamic, 4)
  for (int64_t i = 0; i < M; ++i)
    for (int64_t j = 0; j < M; ++j) {
      cplx v = entry(g, i, j, s);
      A[2 * (i * M + j)] = v.real();
      A[2 * (i * M + j) + 1] = v.imag();
    }
}

void* orc_h2_build(const double* V, const int32_t* T, int64_t M, int32_t nmin, double eta, int32_t m) {
  H2* h = new H2();
  make_geometry(V, T, M, h->g);
  h->nmin = nmin; h->eta = eta; h->m = m; h->p = m * m * m;
  h->perm.resize(M);
  for (int64_t i = 0; i < M; ++i) h->perm[i] = (int)i;
  build_cluster(*h, 0, (int)M, 0, -1);
  partition(*h, 0, 0);
  build_bases(*h);
  return h;
}

void orc_h2_destroy(void* hp) { delete (H2*)hp; }

// stats: clusters, leaves, near, far, nnz_near, depth, p
void orc_h2_stats(void* hp, int64_t* out) {
  H2& h = *(H2*)hp;
  int64_t leaves = 0, depth = 0, nnz = 0;
  for (auto& c : h.cl) { if (c.son0 < 0) ++leaves; depth = std::max<int64_t>(depth, c.level); }
  for (size_t b = 0; b < h.nearR.size(); ++b) {
    const Cluster& r = h.cl[h.nearR[b]];
    const Cluster& c = h.cl[h.nearC[b]];
    nnz += (int64_t)(r.end - r.begin) * (c.end - c.begin);
  }
  out[0] = (int64_t)h.cl.size(); out[1] = leaves; out[2] = (int64_t)h.nearR.size();
  out[3] = (int64_t)h.farR.size(); out[4] = nnz; out[5] = depth; out[6] = h.p;
}

void orc_h2_export(void* hp, int32_t* perm, int32_t* clusters, double* boxes, int32_t* nearp, int32_t* farp) {
  H2& h = *(H2*)hp;
  for (size_t k = 0; k < h.perm.size(); ++k) perm[k] = h.perm[k];
  for (size_t c = 0; c < h.cl.size(); ++c) {
    const Cluster& cc = h.cl[c];
    clusters[5 * c + 0] = cc.begin; clusters[5 * c + 1] = cc.end;
    clusters[5 * c + 2] = cc.son0; clusters[5 * c + 3] = cc.son1; clusters[5 * c + 4] = cc.level;
    for (int a = 0; a < 3; ++a) { boxes[6 * c + a] = cc.lo[a]; boxes[6 * c + 3 + a] = cc.hi[a]; }
  }
  for (size_t b = 0; b < h.nearR.size(); ++b) { nearp[2 * b] = h.nearR[b]; nearp[2 * b + 1] = h.nearC[b]; }
  for (size_t b = 0; b < h.farR.size(); ++b) { farp[2 * b] = h.farR[b]; farp[2 * b + 1] = h.farC[b]; }
}

// U, W: M x p (cluster order); E: C x p x p; xi: C x 3 x m
void orc_h2_export_bases(void* hp, double* U, double* W, double* E, double* xi) {
  H2& h = *(H2*)hp;
  if (U) std::memcpy(U, h.U.data(), sizeof(double) * h.U.size());
  if (W) std::memcpy(W, h.W.data(), sizeof(double) * h.W.size());
  if (E) std::memcpy(E, h.E.data(), sizeof(double) * h.E.size());
  if (xi) std::memcpy(xi, h.xi.data(), sizeof(double) * h.xi.size());
}

// ACA over all far blocks (or the first nblk of `blocks` if blocks != NULL:
// then only those are compressed -- used for sampled pivot checks).
// Returns sum of ranks.
// keep (may be NULL = all L): the frequencies whose Z columns are kept (memory:
// config 4 stores only the compared frequencies, not 28 GB of Z).
int64_t orc_h2_aca_keep(void* hp, const double* s_in, int32_t L, double eps, const int32_t* blocks, int64_t nblk,
                        const int32_t* keep, int32_t nkeep, int32_t* ranks, int32_t* fragile) {
  H2& h = *(H2*)hp;
  if (h.near_done && h.L != L) h.near_done = false;
  h.tw_done = false;
  h.L = L;
  h.s.resize(L);
  for (int l = 0; l < L; ++l) h.s[l] = C2{s_in[2 * l], s_in[2 * l + 1]};
  h.zcol.assign(L, -1);
  std::vector<int> kl;
  if (keep) for (int i = 0; i < nkeep; ++i) { if (h.zcol[keep[i]] < 0) { h.zcol[keep[i]] = (int)kl.size(); kl.push_back(keep[i]); } }
  else for (int l = 0; l < L; ++l) { h.zcol[l] = l; kl.push_back(l); }
  h.zld = (int)kl.size();
  int64_t nfar = (int64_t)h.farR.size();
  std::vector<int64_t> list;
  if (blocks) list.assign(blocks, blocks + nblk); else { list.resize(nfar); for (int64_t b = 0; b < nfar; ++b) list[b] = b; }
  std::vector<AcaOut> res(list.size());
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t t = 0; t < (int64_t)list.size(); ++t) {
    int64_t b = list[t];
    AcaOut& o = res[t];
    aca_block(&h.xi[(size_t)h.farR[b] * 3 * h.m], &h.xi[(size_t)h.farC[b] * 3 * h.m], h.m, h.p, h.s, eps, o);
    if (h.zld != L) {  // keep only the requested columns
      const size_t r = o.k.size();
      std::vector<C2> zk(r * h.zld);
      for (size_t j = 0; j < r; ++j)
        for (int c = 0; c < h.zld; ++c) zk[j * h.zld + c] = o.Z[j * L + kl[c]];
      o.Z.swap(zk);
    }
  }
  h.rank.assign(nfar, 0); h.pivoff.assign(nfar, 0); h.zoff.assign(nfar, 0);
  h.pivk.clear(); h.pivq.clear(); h.Z.clear();
  std::vector<int64_t> where(nfar, -1);
  for (size_t t = 0; t < list.size(); ++t) where[list[t]] = (int64_t)t;
  int64_t tot = 0;
  for (int64_t b = 0; b < nfar; ++b) {
    h.pivoff[b] = (int64_t)h.pivk.size();
    h.zoff[b] = (int64_t)h.Z.size();
    if (where[b] < 0) continue;
    AcaOut& o = res[where[b]];
    h.rank[b] = (int)o.k.size();
    tot += h.rank[b];
    for (size_t t = 0; t < o.k.size(); ++t) { h.pivk.push_back(o.k[t]); h.pivq.push_back(o.q[t]); }
    h.Z.insert(h.Z.end(), o.Z.begin(), o.Z.end());
    std::vector<C2>().swap(o.Z);
  }
  if (ranks) for (int64_t t = 0; t < (int64_t)list.size(); ++t) ranks[t] = h.rank[list[t]];
  if (fragile) for (int64_t t = 0; t < (int64_t)list.size(); ++t) fragile[t] = res[t].fragile;
  h.aca_done = true;
  return tot;
}

int64_t orc_h2_aca(void* hp, const double* s_in, int32_t L, double eps, const int32_t* blocks, int64_t nblk,
                   int32_t* ranks, int32_t* fragile) {
  return orc_h2_aca_keep(hp, s_in, L, eps, blocks, nblk, nullptr, 0, ranks, fragile);
}

// Near-field MACA (Alg. 3 NEAR branch) over all
// near blocks, or the first nblk of `blocks`.  Same Alg. 2 and readings as
// the far blocks; entries from pentry.  Returns the sum of ranks.
int64_t orc_h2_aca_near(void* hp, const double* s_in, int32_t L, double eps, const int32_t* blocks, int64_t nblk,
                        int32_t* ranks, int32_t* fragile) {
  H2& h = *(H2*)hp;
  if (h.aca_done && h.L != L) return -1;
  h.tw_done = false;
  h.L = L;
  h.s.resize(L);
  for (int l = 0; l < L; ++l) h.s[l] = C2{s_in[2 * l], s_in[2 * l + 1]};
  int64_t nnear = (int64_t)h.nearR.size();
  std::vector<int64_t> list;
  if (blocks) list.assign(blocks, blocks + nblk); else { list.resize(nnear); for (int64_t b = 0; b < nnear; ++b) list[b] = b; }
  std::vector<AcaOut> res(list.size());
  std::vector<std::vector<C2>> slices(list.size());
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t t = 0; t < (int64_t)list.size(); ++t) {
    const int64_t b = list[t];
    const int pp = (h.cl[h.nearR[b]].end - h.cl[h.nearR[b]].begin) * (h.cl[h.nearC[b]].end - h.cl[h.nearC[b]].begin);
    aca_generic([&](int q, int l) { return near_aca_entry(h, (size_t)b, q, h.s, l); }, pp, L, eps, res[t]);
    for (size_t j = 0; j < res[t].k.size(); ++j)
      for (int q = 0; q < pp; ++q) slices[t].push_back(near_aca_entry(h, (size_t)b, q, h.s, res[t].k[j]));
  }
  h.nrank.assign(nnear, 0); h.npivoff.assign(nnear, 0); h.nzoff.assign(nnear, 0); h.nsoff.assign(nnear, 0);
  h.npivk.clear(); h.npivq.clear(); h.nZ.clear(); h.nS.clear();
  std::vector<int64_t> where(nnear, -1);
  for (size_t t = 0; t < list.size(); ++t) where[list[t]] = (int64_t)t;
  int64_t tot = 0;
  for (int64_t b = 0; b < nnear; ++b) {
    h.npivoff[b] = (int64_t)h.npivk.size();
    h.nzoff[b] = (int64_t)h.nZ.size();
    h.nsoff[b] = (int64_t)h.nS.size();
    if (where[b] < 0) continue;
    h.nS.insert(h.nS.end(), slices[where[b]].begin(), slices[where[b]].end());
    AcaOut& o = res[where[b]];
    h.nrank[b] = (int)o.k.size();
    tot += h.nrank[b];
    for (size_t t = 0; t < o.k.size(); ++t) { h.npivk.push_back(o.k[t]); h.npivq.push_back(o.q[t]); }
    h.nZ.insert(h.nZ.end(), o.Z.begin(), o.Z.end());
  }
  if (ranks) for (int64_t t = 0; t < (int64_t)list.size(); ++t) ranks[t] = h.nrank[list[t]];
  if (fragile) for (int64_t t = 0; t < (int64_t)list.size(); ++t) fragile[t] = res[t].fragile;
  h.near_done = true;
  return tot;
}

void orc_h2_aca_near_export(void* hp, const int32_t* blocks, int64_t nblk, int32_t* pivots, double* Z) {
  H2& h = *(H2*)hp;
  int64_t pz = 0, pp = 0;
  for (int64_t t = 0; t < nblk; ++t) {
    int64_t b = blocks ? blocks[t] : t;
    for (int j = 0; j < h.nrank[b]; ++j) {
      if (pivots) { pivots[2 * pp] = h.npivk[h.npivoff[b] + j]; pivots[2 * pp + 1] = h.npivq[h.npivoff[b] + j]; }
      ++pp;
    }
    if (Z) for (int64_t j = 0; j < (int64_t)h.nrank[b] * h.L; ++j) {
      Z[2 * pz] = h.nZ[h.nzoff[b] + j].re; Z[2 * pz + 1] = h.nZ[h.nzoff[b] + j].im; ++pz;
    }
  }
}

// Pinned collocation matrix (pentry) at one frequency, input order.
void orc_dense_matrix_pinned(const double* V, const int32_t* T, int64_t M, double sre, double sim, double* A) {
  Geometry g;
  make_geometry(V, T, M, g);
  C2 s{sre, sim};
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < M; ++i)
    for (int64_t j = 0; j < M; ++j) {
      C2 v = pentry(g, i, j, s);
      A[2 * (i * M + j)] = v.re;
      A[2 * (i * M + j) + 1] = v.im;
    }
}

double orc_pexpm1(double x) { return pexpm1(x); }

// pivots for the listed blocks (same order as the orc_h2_aca call), Z likewise.
void orc_h2_aca_export(void* hp, const int32_t* blocks, int64_t nblk, int32_t* pivots, double* Z) {
  H2& h = *(H2*)hp;
  int64_t pz = 0, pp = 0;
  for (int64_t t = 0; t < nblk; ++t) {
    int64_t b = blocks ? blocks[t] : t;
    for (int j = 0; j < h.rank[b]; ++j) {
      if (pivots) { pivots[2 * pp] = h.pivk[h.pivoff[b] + j]; pivots[2 * pp + 1] = h.pivq[h.pivoff[b] + j]; }
      ++pp;
    }
    if (Z) for (int64_t j = 0; j < (int64_t)h.rank[b] * h.zld; ++j) {
      Z[2 * pz] = h.Z[h.zoff[b] + j].re; Z[2 * pz + 1] = h.Z[h.zoff[b] + j].im; ++pz;
    }
  }
}

// y[t][:] = V(s_{lsel[t]}) x[t][:] (input order), for t < nsel.
int orc_h2_apply(void* hp, int32_t mode, const double* s_in, int32_t L, const int32_t* lsel, int32_t nsel,
                 const double* x, double* y) {
  H2& h = *(H2*)hp;
  if ((mode == MODE_H2ACA || mode == MODE_COMBINED) && (!h.aca_done || h.L != L)) return -1;
  if (mode == MODE_COMBINED && !h.near_done) return -1;
  std::vector<cplx> s(L);
  for (int l = 0; l < L; ++l) s[l] = cplx(s_in[2 * l], s_in[2 * l + 1]);
  if (mode == MODE_H2ACA || mode == MODE_COMBINED)
    for (int t = 0; t < nsel; ++t) if (h.zcol[lsel[t]] < 0) return -1;
  apply_multi(h, mode, s, lsel, nsel, (const cplx*)x, (cplx*)y, 0);
  return 0;
}

// The apply with only the listed far / near blocks contributing (timing sample).
int orc_h2_apply_sample(void* hp, int32_t mode, const double* s_in, int32_t L, const int32_t* lsel, int32_t nsel,
                        const double* x, double* y, const int32_t* far_blocks, int64_t nfs, const int32_t* near_blocks,
                        int64_t nns) {
  H2& h = *(H2*)hp;
  if (mode != MODE_H2ACA || !h.aca_done || h.L != L) return -1;
  std::vector<char> fo(h.farR.size(), 0), no(h.nearR.size(), 0);
  for (int64_t i = 0; i < nfs; ++i) {
    if (far_blocks[i] < 0 || far_blocks[i] >= (int64_t)fo.size()) return -1;
    fo[far_blocks[i]] = 1;
  }
  for (int64_t i = 0; i < nns; ++i) {
    if (near_blocks[i] < 0 || near_blocks[i] >= (int64_t)no.size()) return -1;
    no[near_blocks[i]] = 1;
  }
  for (int t = 0; t < nsel; ++t)
    for (size_t b = 0; b < fo.size(); ++b)
      if (fo[b] && (h.zcol[lsel[t]] < 0 || h.zoff[b] < 0)) return -1;
  std::vector<cplx> s(L);
  for (int l = 0; l < L; ++l) s[l] = cplx(s_in[2 * l], s_in[2 * l + 1]);
  apply_multi(h, mode, s, lsel, nsel, (const cplx*)x, (cplx*)y, 0, fo.data(), no.data());
  return 0;
}

// y[t][:] = (alpha I + K(s_{lsel[t]})) x[t][:] (double layer, NEXT-1)
int orc_h2_apply_dl(void* hp, int32_t mode, const double* s_in, int32_t L, const int32_t* lsel, int32_t nsel,
                    const double* x, double* y, double alpha) {
  H2& h = *(H2*)hp;
  if ((mode == MODE_H2ACA || mode == MODE_COMBINED) && (!h.aca_done || h.L != L)) return -1;
  if (mode == MODE_COMBINED && !h.near_done) return -1;
  std::vector<cplx> s(L);
  for (int l = 0; l < L; ++l) s[l] = cplx(s_in[2 * l], s_in[2 * l + 1]);
  int64_t M = h.g.M;
  if (mode == MODE_H2ACA || mode == MODE_COMBINED)
    for (int t = 0; t < nsel; ++t) if (h.zcol[lsel[t]] < 0) return -1;
  apply_multi(h, mode, s, lsel, nsel, (const cplx*)x, (cplx*)y, 1);
  for (int t = 0; t < nsel; ++t) {
    const cplx* xt = (const cplx*)(x + 2 * (int64_t)t * M);
    cplx* yt = (cplx*)(y + 2 * (int64_t)t * M);
    for (int64_t i = 0; i < M; ++i) yt[i] += alpha * xt[i];
  }
  return 0;
}

void orc_dense_matrix_dl(const double* V, const int32_t* T, int64_t M, double sre, double sim, double* A) {
  Geometry g;
  make_geometry(V, T, M, g);
  cplx s(sre, sim);
  for (int64_t i = 0; i < M; ++i)
    for (int64_t j = 0; j < M; ++j) {
      cplx v = entry_dl(g, i, j, s);
      A[2 * (i * M + j)] = v.real();
      A[2 * (i * M + j) + 1] = v.imag();
    }
}

void orc_normals(const double* V, const int32_t* T, int64_t M, double* nrm) {
  Geometry g;
  make_geometry(V, T, M, g);
  for (int64_t i = 0; i < 3 * M; ++i) nrm[i] = g.nrm[i];
}

void orc_forward(const double* xt, double* xf, int64_t M, int32_t N, double R) {
  forward((const cplx*)xt, (cplx*)xf, M, N, R);
}
void orc_inverse(const double* yf, double* yt, int64_t M, int32_t N, double R) {
  inverse((const cplx*)yf, (cplx*)yt, M, N, R);
}

// GMRES per selected frequency with the oracle's own operator in `mode`.
int orc_h2_gmres(void* hp, int32_t mode, const double* s_in, int32_t L, const int32_t* lsel, int32_t nsel,
                 const double* b, double* x, double tol, int32_t restart, int32_t maxit, int32_t* iters,
                 double* relres) {
  H2& h = *(H2*)hp;
  if ((mode == MODE_H2ACA || mode == MODE_COMBINED) && (!h.aca_done || h.L != L)) return -1;
  if (mode == MODE_COMBINED && !h.near_done) return -1;
  if (mode == MODE_H2ACA || mode == MODE_COMBINED)
    for (int t = 0; t < nsel; ++t) if (h.zcol[lsel[t]] < 0) return -1;
  std::vector<cplx> s(L);
  for (int l = 0; l < L; ++l) s[l] = cplx(s_in[2 * l], s_in[2 * l + 1]);
  int64_t M = h.g.M;
  if (mode == MODE_H2ACA || mode == MODE_H2ONLY) {  // one frequency at a time, parallel applies
    for (int t = 0; t < nsel; ++t) {
      int l = lsel[t];
      OneFreqCache k;
      build_cache(h, mode, s[l], l, s, k);
      auto op = [&](const cplx* in, cplx* out) { apply_cached(h, k, in, out); };
      iters[t] = gmres(op, M, (const cplx*)(b + 2 * (int64_t)t * M), (cplx*)(x + 2 * (int64_t)t * M), tol, restart,
                       maxit, &relres[t]);
    }
    return 0;
  }
#pragma omp parallel for schedule(dynamic, 1)
  for (int t = 0; t < nsel; ++t) {
    int l = lsel[t];
    auto op = [&](const cplx* in, cplx* out) { apply_one(h, mode, s[l], l, s, in, out); };
    iters[t] = gmres(op, M, (const cplx*)(b + 2 * (int64_t)t * M), (cplx*)(x + 2 * (int64_t)t * M), tol, restart,
                     maxit, &relres[t]);
  }
  return 0;
}

int32_t orc_admissible(const double* br, const double* bc, double eta) {
  Cluster r{}, c{};
  for (int a = 0; a < 3; ++a) { r.lo[a] = br[a]; r.hi[a] = br[3 + a]; c.lo[a] = bc[a]; c.hi[a] = bc[3 + a]; }
  return admissible(r, c, eta) ? 1 : 0;
}

// Generic MACA on a dense pp x L complex matrix A (row q = slice index, column l
// = frequency).  Returns the rank; pivots (k,q) r x 2, Z r x L, C r x pp,
// D r x L, Gram-norm history r (caller sizes with rmax = min(pp, L)).
int32_t orc_aca_matrix(const double* A, int32_t pp, int32_t L, double eps, int32_t* piv, double* Z, double* Cm,
                       double* Dm, double* nrm) {
  const C2* a = (const C2*)A;
  AcaOut out;
  std::vector<double> hist;
  std::vector<std::vector<C2>> Cs, Ds;
  aca_generic([&](int q, int l) { return a[(size_t)q * L + l]; }, pp, L, eps, out, &hist, &Cs, &Ds);
  int r = (int)out.k.size();
  for (int t = 0; t < r; ++t) {
    piv[2 * t] = out.k[t]; piv[2 * t + 1] = out.q[t];
    nrm[t] = hist[t];
    for (int l = 0; l < L; ++l) {
      Z[2 * ((size_t)t * L + l)] = out.Z[(size_t)t * L + l].re;
      Z[2 * ((size_t)t * L + l) + 1] = out.Z[(size_t)t * L + l].im;
      Dm[2 * ((size_t)t * L + l)] = Ds[t][l].re;
      Dm[2 * ((size_t)t * L + l) + 1] = Ds[t][l].im;
    }
    for (int q = 0; q < pp; ++q) {
      Cm[2 * ((size_t)t * pp + q)] = Cs[t][q].re;
      Cm[2 * ((size_t)t * pp + q) + 1] = Cs[t][q].im;
    }
  }
  return r;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// NEXT-2: time-domain weights from the compressed tensor and the
// fast right-hand-side convolution (eq:fastdft P:1542-1553, eq:fastrhs
// P:1566-1573), on the combined skeleton (every block b in P+ and P-):
//   V^_n[b] = sum_t C_{b,t} dhat_{b,t}[n],
//   dhat_{b,t}[n] = (R^{-n}/L) sum_l Z_b[t,l] e^{+2 pi i (n l mod L)/L}  (reading D2: L = N+1,
//                   the inverse transform of C5 applied to the coefficient row),
//   C_{b,t} = S_b(s_{k_t}) (far, with the bases U_r, W_c) or V_{k_t}[b] (near, stored).
// The MoT recursion itself (eq:cqmrhs P:652-680 and the LU of V^_0)
// is written in oracle/__init__.py on top of these.
// ---------------------------------------------------------------------------
static void up_pass(const H2& h, const std::vector<cplx>& x, std::vector<cplx>& xh) {
  const int p = h.p, C = (int)h.cl.size();
  xh.assign((size_t)C * p, cplx(0.0, 0.0));
  for (int c = C - 1; c >= 0; --c) {
    const Cluster& cc = h.cl[c];
    cplx* out = &xh[(size_t)c * p];
    if (cc.son0 < 0) {
      for (int nu = 0; nu < p; ++nu) {
        cplx acc(0.0, 0.0);
        for (int k = cc.begin; k < cc.end; ++k) acc += h.W[(size_t)k * p + nu] * x[k];
        out[nu] = acc;
      }
    } else {
      for (int son : {cc.son0, cc.son1}) {
        const double* Es = &h.E[(size_t)son * p * p];
        for (int mu = 0; mu < p; ++mu) {
          cplx acc(0.0, 0.0);
          for (int lam = 0; lam < p; ++lam) acc += Es[(size_t)lam * p + mu] * xh[(size_t)son * p + lam];
          out[mu] += acc;
        }
      }
    }
  }
}

static void down_pass(const H2& h, std::vector<cplx>& yh, std::vector<cplx>& y) {
  const int p = h.p, C = (int)h.cl.size();
  for (int c = 0; c < C; ++c) {
    const Cluster& cc = h.cl[c];
    if (cc.parent >= 0) {
      const double* Es = &h.E[(size_t)c * p * p];
      for (int lam = 0; lam < p; ++lam) {
        cplx acc(0.0, 0.0);
        for (int mu = 0; mu < p; ++mu) acc += Es[(size_t)lam * p + mu] * yh[(size_t)cc.parent * p + mu];
        yh[(size_t)c * p + lam] += acc;
      }
    }
    if (cc.son0 < 0)
      for (int k = cc.begin; k < cc.end; ++k) {
        cplx acc(0.0, 0.0);
        for (int mu = 0; mu < p; ++mu) acc += h.U[(size_t)k * p + mu] * yh[(size_t)c * p + mu];
        y[k] += acc;
      }
  }
}


static void dhat_rows(const std::vector<C2>& Z, int L, int N, double R, std::vector<cplx>& D) {
  const size_t rows = Z.size() / (size_t)L;
  D.assign(Z.size(), cplx(0.0, 0.0));
  std::vector<cplx> zf(L), dt(L);
  for (size_t r = 0; r < rows; ++r) {
    for (int l = 0; l < L; ++l) zf[l] = cplx(Z[r * L + l].re, Z[r * L + l].im);
    inverse(zf.data(), dt.data(), 1, N, R);
    for (int n = 0; n < L; ++n) D[r * L + n] = dt[n];
  }
}


// y_n = sum_{k = 0}^{min(n, kmax)} V^_{n-k} q_k for n = 0..N (cluster-basis form of
// eq:fastrhs: per block and term, u = sum_k dhat[n-k] Xc_k first, then C_t u).
static void conv_time(const H2& h, const cplx* q_in, cplx* y_out, int kmax) {
  const int L = h.L, p = h.p, m = h.m, C = (int)h.cl.size();
  const int64_t M = h.g.M;
  std::vector<std::vector<cplx>> q(L, std::vector<cplx>(M)), xh(L);
  for (int k = 0; k < L; ++k) {
    for (int64_t a = 0; a < M; ++a) q[k][a] = q_in[(int64_t)k * M + h.perm[a]];
    up_pass(h, q[k], xh[k]);
  }
  std::vector<cplx> S((size_t)p * p), u(std::max<int64_t>(p, 1)), un;
  for (int n = 0; n < L; ++n) {
    const int kend = std::min(n, kmax);
    std::vector<cplx> yh((size_t)C * p, cplx(0.0, 0.0)), y(M, cplx(0.0, 0.0));
    for (size_t b = 0; b < h.farR.size(); ++b) {
      const int r = h.farR[b], c = h.farC[b];
      const double* xr = &h.xi[(size_t)r * 3 * m];
      const double* xc = &h.xi[(size_t)c * 3 * m];
      for (int t = 0; t < h.rank[b]; ++t) {
        const cplx* d = &h.tDf[h.zoff[b] + (size_t)t * L];
        for (int nu = 0; nu < p; ++nu) {
          cplx acc(0.0, 0.0);
          for (int k = 0; k <= kend; ++k) acc += d[n - k] * xh[k][(size_t)c * p + nu];
          u[nu] = acc;
        }
        const int kk = h.pivk[h.pivoff[b] + t];
        const cplx sk(h.s[kk].re, h.s[kk].im);
        for (int mu = 0; mu < p; ++mu) {
          cplx acc(0.0, 0.0);
          for (int nu = 0; nu < p; ++nu) {
            double a3[3], b3[3];
            node_point(xr, m, mu, a3); node_point(xc, m, nu, b3);
            const double dx = b3[0] - a3[0], dy = b3[1] - a3[1], dz = b3[2] - a3[2];
            acc += kernel(std::sqrt((dx * dx + dy * dy) + dz * dz), sk) * u[nu];
          }
          yh[(size_t)r * p + mu] += acc;
        }
      }
    }
    down_pass(h, yh, y);
    for (size_t b = 0; b < h.nearR.size(); ++b) {
      const Cluster& R = h.cl[h.nearR[b]];
      const Cluster& Cc = h.cl[h.nearC[b]];
      const int nr = R.end - R.begin, nc = Cc.end - Cc.begin;
      un.assign(nc, cplx(0.0, 0.0));
      for (int t = 0; t < h.nrank[b]; ++t) {
        const cplx* d = &h.tDn[h.nzoff[b] + (size_t)t * L];
        for (int j = 0; j < nc; ++j) {
          cplx acc(0.0, 0.0);
          for (int k = 0; k <= kend; ++k) acc += d[n - k] * q[k][Cc.begin + j];
          un[j] = acc;
        }
        const C2* Sl = &h.nS[h.nsoff[b] + (size_t)t * nr * nc];
        for (int i = 0; i < nr; ++i) {
          cplx acc(0.0, 0.0);
          for (int j = 0; j < nc; ++j) acc += cplx(Sl[(size_t)i * nc + j].re, Sl[(size_t)i * nc + j].im) * un[j];
          y[R.begin + i] += acc;
        }
      }
    }
    for (int64_t a = 0; a < M; ++a) y_out[(int64_t)n * M + h.perm[a]] = y[a];
  }
}

// Dense V^_n (input order) assembled from the same compressed weights (for the
// oracle's LU-based MoT and the pins).
static void weight_dense(const H2& h, int n, cplx* A) {
  const int L = h.L, p = h.p, m = h.m;
  const int64_t M = h.g.M;
  std::fill(A, A + M * M, cplx(0.0, 0.0));
  std::vector<cplx> G((size_t)p * p);
  for (size_t b = 0; b < h.farR.size(); ++b) {
    const int r = h.farR[b], c = h.farC[b];
    const double* xr = &h.xi[(size_t)r * 3 * m];
    const double* xc = &h.xi[(size_t)c * 3 * m];
    std::fill(G.begin(), G.end(), cplx(0.0, 0.0));
    for (int t = 0; t < h.rank[b]; ++t) {
      const cplx d = h.tDf[h.zoff[b] + (size_t)t * L + n];
      const int kk = h.pivk[h.pivoff[b] + t];
      const cplx sk(h.s[kk].re, h.s[kk].im);
      for (int mu = 0; mu < p; ++mu)
        for (int nu = 0; nu < p; ++nu) {
          double a3[3], b3[3];
          node_point(xr, m, mu, a3); node_point(xc, m, nu, b3);
          const double dx = b3[0] - a3[0], dy = b3[1] - a3[1], dz = b3[2] - a3[2];
          G[(size_t)mu * p + nu] += d * kernel(std::sqrt((dx * dx + dy * dy) + dz * dz), sk);
        }
    }
    // V^_n[rows of r, cols of c] = U_r G W_c^T with the clusters' own Lagrange bases
    // (P:957-978): U_r[a,mu] = L_{r,mu}(c_a), W_c[k,nu] = |T_k| sum_q w_q L_{c,nu}(y_{k,q})
    const Cluster& R = h.cl[r];
    const Cluster& Cc = h.cl[c];
    std::vector<double> Wc((size_t)(Cc.end - Cc.begin) * p);
    for (int k = Cc.begin; k < Cc.end; ++k) {
      const int i = h.perm[k];
      for (int nu = 0; nu < p; ++nu) {
        double acc = 0.0;
        for (int q = 0; q < 7; ++q) acc += RULE.w[q] * lagrange3(xc, m, nu, &h.g.node[21 * i + 3 * q]);
        Wc[(size_t)(k - Cc.begin) * p + nu] = h.g.area[i] * acc;
      }
    }
    std::vector<cplx> GW((size_t)p * (Cc.end - Cc.begin));
    for (int mu = 0; mu < p; ++mu)
      for (int k = 0; k < Cc.end - Cc.begin; ++k) {
        cplx row(0.0, 0.0);
        for (int nu = 0; nu < p; ++nu) row += G[(size_t)mu * p + nu] * Wc[(size_t)k * p + nu];
        GW[(size_t)mu * (Cc.end - Cc.begin) + k] = row;
      }
    for (int a = R.begin; a < R.end; ++a) {
      double ur[512];
      for (int mu = 0; mu < p; ++mu) ur[mu] = lagrange3(xr, m, mu, &h.g.cen[3 * h.perm[a]]);
      for (int k = Cc.begin; k < Cc.end; ++k) {
        cplx acc(0.0, 0.0);
        for (int mu = 0; mu < p; ++mu) acc += ur[mu] * GW[(size_t)mu * (Cc.end - Cc.begin) + (k - Cc.begin)];
        A[(int64_t)h.perm[a] * M + h.perm[k]] += acc;
      }
    }
  }
  for (size_t b = 0; b < h.nearR.size(); ++b) {
    const Cluster& R = h.cl[h.nearR[b]];
    const Cluster& Cc = h.cl[h.nearC[b]];
    const int nr = R.end - R.begin, nc = Cc.end - Cc.begin;
    for (int t = 0; t < h.nrank[b]; ++t) {
      const cplx d = h.tDn[h.nzoff[b] + (size_t)t * L + n];
      const C2* Sl = &h.nS[h.nsoff[b] + (size_t)t * nr * nc];
      for (int i = 0; i < nr; ++i)
        for (int j = 0; j < nc; ++j)
          A[(int64_t)h.perm[R.begin + i] * M + h.perm[Cc.begin + j]] +=
              d * cplx(Sl[(size_t)i * nc + j].re, Sl[(size_t)i * nc + j].im);
    }
  }
}

extern "C" {
// dhat rows of every far and near block (requires orc_h2_aca and orc_h2_aca_near with
// the same L); R is the transform's scaling.
int orc_h2_time_weights(void* hp, double R) {
  H2& h = *(H2*)hp;
  if (!h.aca_done || !h.near_done || h.zld != h.L) return -1;
  dhat_rows(h.Z, h.L, h.L - 1, R, h.tDf);
  dhat_rows(h.nZ, h.L, h.L - 1, R, h.tDn);
  h.tw_done = true;
  return 0;
}

// y[n][:] = sum_{k <= min(n, kmax)} V^_{n-k} q[k][:], input order, complex [L][M].
int orc_h2_conv(void* hp, const double* q, double* y, int32_t kmax) {
  H2& h = *(H2*)hp;
  if (!h.tw_done) return -1;
  conv_time(h, (const cplx*)q, (cplx*)y, kmax);
  return 0;
}

int orc_h2_weight_dense(void* hp, int32_t n, double* A) {
  H2& h = *(H2*)hp;
  if (!h.tw_done || n < 0 || n >= h.L) return -1;
  weight_dense(h, n, (cplx*)A);
  return 0;
}
}  // extern "C"
