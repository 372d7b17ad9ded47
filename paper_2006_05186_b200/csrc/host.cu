// Host side of the library: error handling, CQM frequencies, panel geometry,
// cluster tree, block partition and Chebyshev cluster bases (bem_build_tree).
//
// The tree/partition rules are pinned for bit-exactness:
//   P:832-835  split the tight vertex box at the midpoint of its longest axis
//              (lowest axis on exact ties), centroids strictly below the
//              midpoint go left, stable order; one side empty -> stable sort by
//              centroid coordinate and split at floor(n/2);
//   P:826/882  leaves hold <= n_min panels (AM6);
//   P:843-865  block recursion from (root,root) in the order
//              (r0,c0),(r0,c1),(r1,c0),(r1,c1); one-sided if only one side has sons;
//   P:905-912  eq:qadm with squared norms, equality admissible; near <=> an
//              inadmissible leaf x leaf pair (AM9).
// Host code is compiled with -ffp-contract=off (bit-exact centroids/boxes).
#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <numeric>

#include "common.cuh"

namespace bem {

static thread_local std::string g_err;

void set_error(const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
}

static const double kPi = 3.14159265358979323846;
static const double kFourPi = 0x1.921fb54442d18p+3;

// 7-point degree-5 triangle rule (barycentric), north_star near-field rule.
struct TriRule {
  double b0[7], b1[7], b2[7], w[7];
  TriRule() {
    const double r15 = std::sqrt(15.0);
    const double a1 = (9.0 - 2.0 * r15) / 21.0, c1 = (6.0 + r15) / 21.0;
    const double a2 = (9.0 + 2.0 * r15) / 21.0, c2 = (6.0 - r15) / 21.0;
    const double w1 = (155.0 + r15) / 1200.0, w2 = (155.0 - r15) / 1200.0;
    const double B[7][3] = {{1.0 / 3.0, 1.0 / 3.0, 1.0 / 3.0}, {a1, c1, c1}, {c1, a1, c1}, {c1, c1, a1},
                            {a2, c2, c2}, {c2, a2, c2}, {c2, c2, a2}};
    const double W[7] = {9.0 / 40.0, w1, w1, w1, w2, w2, w2};
    for (int q = 0; q < 7; ++q) { b0[q] = B[q][0]; b1[q] = B[q][1]; b2[q] = B[q][2]; w[q] = W[q]; }
  }
};
static const TriRule kRule;

// int_T dS(y)/|y - c| for the in-plane centroid c: sum over edges of
// d (asinh(t_B/d) - asinh(t_A/d)) (polar integration around c).
static double panel_self_integral(const double* P0, const double* P1, const double* P2, const double* c) {
  const double* P[3] = {P0, P1, P2};
  double acc = 0.0;
  for (int e = 0; e < 3; ++e) {
    const double* A = P[e];
    const double* B = P[(e + 1) % 3];
    double ux = B[0] - A[0], uy = B[1] - A[1], uz = B[2] - A[2];
    double len = std::sqrt(ux * ux + uy * uy + uz * uz);
    ux /= len; uy /= len; uz /= len;
    double ax = A[0] - c[0], ay = A[1] - c[1], az = A[2] - c[2];
    double bx = B[0] - c[0], by = B[1] - c[1], bz = B[2] - c[2];
    double ta = ax * ux + ay * uy + az * uz;
    double tb = bx * ux + by * uy + bz * uz;
    // f = (A - t_A u) - c: the pinned operation order of DESIGN.md §5 (the near-field
    // MACA reads J bit-for-bit)
    double fx = (A[0] - ta * ux) - c[0], fy = (A[1] - ta * uy) - c[1], fz = (A[2] - ta * uz) - c[2];
    double d = std::sqrt(fx * fx + fy * fy + fz * fz);
    acc += d * (std::asinh(tb / d) - std::asinh(ta / d));
  }
  return acc;
}

}  // namespace bem

using namespace bem;

extern "C" const char* bem_last_error(void) { return g_err.c_str(); }

extern "C" bem_status cqm_frequencies(int32_t N, double T, double R, int32_t method, bem_c128* s_out) {
  BEM_REQ(N >= 1, "cqm_frequencies: N=%d < 1", N);
  BEM_REQ(T > 0.0, "cqm_frequencies: T must be > 0");
  BEM_REQ(R > 0.0 && R < 1.0, "cqm_frequencies: R must lie in (0,1)");
  BEM_REQ(method == 1 || method == 2, "cqm_frequencies: method must be 1 (BDF1) or 2 (BDF2)");
  BEM_REQ(s_out != nullptr, "cqm_frequencies: s_out is NULL");
  const int L = N + 1;
  const int half = L / 2;
  const double dt = T / (double)N;
  for (int l = 0; l <= half; ++l) {
    double zr, zi;
    if (l == 0) {
      zr = R; zi = 0.0;
    } else {
      double ang = (2.0 * kPi * (double)l) / (double)L;
      zr = R * std::cos(ang);
      zi = -(R * std::sin(ang));
    }
    double dr, di;
    if (method == 2) {
      double sqr = zr * zr - zi * zi, sqi = 2.0 * (zr * zi);
      dr = (1.5 - 2.0 * zr) + 0.5 * sqr;
      di = (-2.0 * zi) + 0.5 * sqi;
    } else {
      dr = 1.0 - zr;
      di = -zi;
    }
    s_out[l].re = dr / dt;
    s_out[l].im = (l == 0) ? 0.0 : di / dt;
  }
  for (int l = half + 1; l < L; ++l) {
    s_out[l].re = s_out[L - l].re;
    s_out[l].im = -s_out[L - l].im;
  }
  return BEM_OK;
}

namespace {

struct HostGeom {
  std::vector<double> cen, lo, hi, area, qn, J;  // input order
  std::vector<double> nrm;  // unit normals (b-a)x(c-a)/|.| in vertex order (double layer, NEXT-1)
};

// Tree construction with an explicit stack (pre-order ids, left son first).
struct Builder {
  const HostGeom& g;
  Tree& t;
  Builder(const HostGeom& gg, Tree& tt) : g(gg), t(tt) {}

  void run(int64_t M) {
    t.perm.resize(M);
    std::iota(t.perm.begin(), t.perm.end(), 0);
    struct Item { int b, e, level, parent, side; };
    std::vector<Item> stack{{0, (int)M, 0, -1, 0}};
    std::vector<int32_t> scratch;
    while (!stack.empty()) {
      Item it = stack.back();
      stack.pop_back();
      const int id = (int)t.begin.size();
      t.begin.push_back(it.b); t.end.push_back(it.e);
      t.son0.push_back(-1); t.son1.push_back(-1);
      t.level.push_back(it.level); t.parent.push_back(it.parent);
      if (it.parent >= 0) (it.side == 0 ? t.son0 : t.son1)[it.parent] = id;
      double lo[3] = {HUGE_VAL, HUGE_VAL, HUGE_VAL}, hi[3] = {-HUGE_VAL, -HUGE_VAL, -HUGE_VAL};
      for (int k = it.b; k < it.e; ++k) {
        const int i = t.perm[k];
        for (int a = 0; a < 3; ++a) {
          lo[a] = std::min(lo[a], g.lo[3 * i + a]);
          hi[a] = std::max(hi[a], g.hi[3 * i + a]);
        }
      }
      for (int a = 0; a < 3; ++a) { t.box.push_back(lo[a]); }
      for (int a = 0; a < 3; ++a) { t.box.push_back(hi[a]); }
      const int n = it.e - it.b;
      if (n <= t.nmin) continue;
      int ax = 0;
      double ext = hi[0] - lo[0];
      for (int a = 1; a < 3; ++a) {
        double ea = hi[a] - lo[a];
        if (ea > ext) { ext = ea; ax = a; }
      }
      const double mid = 0.5 * (lo[ax] + hi[ax]);
      scratch.assign(t.perm.begin() + it.b, t.perm.begin() + it.e);
      auto below = [&](int32_t i) { return g.cen[3 * i + ax] < mid; };
      int nl = 0;
      for (int32_t i : scratch) nl += below(i) ? 1 : 0;
      if (nl == 0 || nl == n) {
        std::stable_sort(scratch.begin(), scratch.end(),
                         [&](int32_t x, int32_t y) { return g.cen[3 * x + ax] < g.cen[3 * y + ax]; });
        nl = n / 2;
        std::copy(scratch.begin(), scratch.end(), t.perm.begin() + it.b);
      } else {
        int kl = it.b, kr = it.b + nl;
        for (int32_t i : scratch) {
          if (below(i)) t.perm[kl++] = i; else t.perm[kr++] = i;
        }
      }
      // push right first so that the left son is numbered next (pre-order)
      stack.push_back({it.b + nl, it.e, it.level + 1, id, 1});
      stack.push_back({it.b, it.b + nl, it.level + 1, id, 0});
    }
    t.C = (int)t.begin.size();
  }
};

bool admissible_boxes(const double* r, const double* c, double eta) {
  double dr2 = 0.0, dc2 = 0.0, dist2 = 0.0;
  double tr[3], tc[3], tg[3];
  for (int a = 0; a < 3; ++a) {
    tr[a] = r[3 + a] - r[a];
    tc[a] = c[3 + a] - c[a];
    double g = std::max(0.0, std::max(c[a] - r[3 + a], r[a] - c[3 + a]));
    tg[a] = g;
  }
  dr2 = (tr[0] * tr[0] + tr[1] * tr[1]) + tr[2] * tr[2];
  dc2 = (tc[0] * tc[0] + tc[1] * tc[1]) + tc[2] * tc[2];
  dist2 = (tg[0] * tg[0] + tg[1] * tg[1]) + tg[2] * tg[2];
  return std::max(dr2, dc2) <= (eta * eta) * dist2;
}

void build_partition(Tree& t) {
  std::vector<std::pair<int, int>> stack{{0, 0}};
  while (!stack.empty()) {
    auto [r, c] = stack.back();
    stack.pop_back();
    if (admissible_boxes(&t.box[6 * r], &t.box[6 * c], t.eta)) {
      t.far_r.push_back(r); t.far_c.push_back(c);
      continue;
    }
    const bool lr = t.son0[r] < 0, lc = t.son0[c] < 0;
    if (lr && lc) {
      t.near_r.push_back(r); t.near_c.push_back(c);
      t.nnz_near += (int64_t)(t.end[r] - t.begin[r]) * (t.end[c] - t.begin[c]);
      continue;
    }
    // push in reverse so that the pop order is (r0,c0),(r0,c1),(r1,c0),(r1,c1)
    if (!lr && !lc) {
      stack.push_back({t.son1[r], t.son1[c]});
      stack.push_back({t.son1[r], t.son0[c]});
      stack.push_back({t.son0[r], t.son1[c]});
      stack.push_back({t.son0[r], t.son0[c]});
    } else if (!lr) {
      stack.push_back({t.son1[r], c});
      stack.push_back({t.son0[r], c});
    } else {
      stack.push_back({r, t.son1[c]});
      stack.push_back({r, t.son0[c]});
    }
  }
}

// Chebyshev nodes of the first kind on the cluster box, axis-major.
void cheb_nodes(const double* box, int m, double* xi) {
  const double ex = box[3] - box[0], ey = box[4] - box[1], ez = box[5] - box[2];
  const double diag = std::sqrt((ex * ex + ey * ey) + ez * ez);
  for (int a = 0; a < 3; ++a) {
    double lo = box[a], hi = box[3 + a];
    if (hi - lo == 0.0) {  // degenerate axis (AM12)
      lo = lo - 1e-8 * diag;
      hi = hi + 1e-8 * diag;
    }
    const double mid = 0.5 * (lo + hi), half = 0.5 * (hi - lo);
    for (int k = 0; k < m; ++k) xi[a * m + k] = mid + half * std::cos(((double)(2 * k + 1) * kPi) / (double)(2 * m));
  }
}

// 1-D Lagrange basis values l_k(x), k < m, on nodes xs.
void lagrange_1d(const double* xs, int m, double x, double* out) {
  for (int k = 0; k < m; ++k) {
    double v = 1.0;
    for (int j = 0; j < m; ++j)
      if (j != k) v *= (x - xs[j]) / (xs[k] - xs[j]);
    out[k] = v;
  }
}

// values of all p = m^3 tensor Lagrange polynomials at point x (mu = kx + m ky + m^2 kz)
void lagrange_3d(const double* xi, int m, const double* x, double* out) {
  double lx[8], ly[8], lz[8];
  lagrange_1d(xi, m, x[0], lx);
  lagrange_1d(xi + m, m, x[1], ly);
  lagrange_1d(xi + 2 * m, m, x[2], lz);
  for (int kz = 0; kz < m; ++kz)
    for (int ky = 0; ky < m; ++ky)
      for (int kx = 0; kx < m; ++kx) out[kx + m * (ky + m * kz)] = lx[kx] * ly[ky] * lz[kz];
}

// n . grad of all p = m^3 tensor Lagrange polynomials at x (double-layer column basis)
void lagrange_grad_n_3d(const double* xi, int m, const double* x, const double* n, double* out) {
  double l[3][8], d[3][8];
  for (int a = 0; a < 3; ++a) {
    const double* xs = xi + a * m;
    lagrange_1d(xs, m, x[a], l[a]);
    for (int k = 0; k < m; ++k) {  // l_k'(t) = sum_{i != k} 1/(x_k - x_i) prod_{j != k,i} (t - x_j)/(x_k - x_j)
      double sum = 0.0;
      for (int i = 0; i < m; ++i) {
        if (i == k) continue;
        double v = 1.0 / (xs[k] - xs[i]);
        for (int j = 0; j < m; ++j)
          if (j != k && j != i) v *= (x[a] - xs[j]) / (xs[k] - xs[j]);
        sum += v;
      }
      d[a][k] = sum;
    }
  }
  for (int kz = 0; kz < m; ++kz)
    for (int ky = 0; ky < m; ++ky)
      for (int kx = 0; kx < m; ++kx)
        out[kx + m * (ky + m * kz)] = (n[0] * (d[0][kx] * l[1][ky] * l[2][kz]) + n[1] * (l[0][kx] * d[1][ky] * l[2][kz])) +
                                      n[2] * (l[0][kx] * l[1][ky] * d[2][kz]);
}

}  // namespace

extern "C" bem_status bem_build_tree(const double* V, int64_t nv, const int32_t* T, int64_t nt, int32_t leaf_size,
                                     double eta, int32_t m, int32_t device, bem_tree* out) {
  Nvtx nvtx_range("bem_build_tree");
  BEM_REQ(out != nullptr, "bem_build_tree: out is NULL");
  BEM_REQ(V != nullptr && T != nullptr, "bem_build_tree: NULL mesh arrays");
  BEM_REQ(nv >= 3 && nt >= 1, "bem_build_tree: need nv >= 3 and nt >= 1");
  BEM_REQ(nt < (int64_t)1 << 30, "bem_build_tree: too many panels");
  BEM_REQ(leaf_size > 1, "bem_build_tree: leaf_size (n_min) must be > 1");
  BEM_REQ(eta > 0.0, "bem_build_tree: eta must be > 0");
  BEM_REQ(m >= 1 && m <= 5, "bem_build_tree: cheb_order must be in [1,5]");
  int ndev = 0;
  if (device >= 0 && cudaGetDeviceCount(&ndev) != cudaSuccess) ndev = 0;
  BEM_REQ(device == -1 || (device >= 0 && device < ndev), "bem_build_tree: device %d not available (%d devices)",
          device, ndev);
  *out = nullptr;
  const int64_t M = nt;
  HostGeom g;
  g.cen.resize(3 * M); g.lo.resize(3 * M); g.hi.resize(3 * M); g.area.resize(M); g.qn.resize(21 * M); g.J.resize(M);
  g.nrm.resize(3 * M);
  for (int64_t i = 0; i < M; ++i) {
    const double* P[3];
    for (int v = 0; v < 3; ++v) {
      const int32_t idx = T[3 * i + v];
      BEM_REQ(idx >= 0 && idx < nv, "bem_build_tree: triangle %lld has vertex index %d out of range", (long long)i,
              idx);
      P[v] = V + 3 * (int64_t)idx;
    }
    for (int a = 0; a < 3; ++a) {
      g.cen[3 * i + a] = ((P[0][a] + P[1][a]) + P[2][a]) / 3.0;
      g.lo[3 * i + a] = std::min(std::min(P[0][a], P[1][a]), P[2][a]);
      g.hi[3 * i + a] = std::max(std::max(P[0][a], P[1][a]), P[2][a]);
    }
    const double ux = P[1][0] - P[0][0], uy = P[1][1] - P[0][1], uz = P[1][2] - P[0][2];
    const double vx = P[2][0] - P[0][0], vy = P[2][1] - P[0][1], vz = P[2][2] - P[0][2];
    const double cx = uy * vz - uz * vy, cy = uz * vx - ux * vz, cz = ux * vy - uy * vx;
    g.area[i] = 0.5 * std::sqrt((cx * cx + cy * cy) + cz * cz);
    BEM_REQ(g.area[i] > 0.0, "bem_build_tree: triangle %lld is degenerate (area <= 0)", (long long)i);
    g.nrm[3 * i] = cx / (2.0 * g.area[i]);
    g.nrm[3 * i + 1] = cy / (2.0 * g.area[i]);
    g.nrm[3 * i + 2] = cz / (2.0 * g.area[i]);
    for (int q = 0; q < 7; ++q)
      for (int a = 0; a < 3; ++a)
        g.qn[21 * i + 3 * q + a] =
            q == 0 ? g.cen[3 * i + a] : (kRule.b0[q] * P[0][a] + kRule.b1[q] * P[1][a]) + kRule.b2[q] * P[2][a];
    g.J[i] = panel_self_integral(P[0], P[1], P[2], &g.cen[3 * i]);
  }

  bem_tree_s* h = new bem_tree_s();
  Tree& t = h->t;
  t.device = device; t.M = M; t.nmin = leaf_size; t.eta = eta; t.m = m; t.p = m * m * m;
  Builder(g, t).run(M);
  build_partition(t);
  const int C = t.C, p = t.p;
  for (int c = 0; c < C; ++c) {
    t.depth = std::max(t.depth, (int)t.level[c]);
    if (t.son0[c] < 0) t.leaves.push_back(c);
  }
  t.n_leaves = (int)t.leaves.size();
  t.level_nonleaf.assign(t.depth + 1, {});
  for (int c = 0; c < C; ++c)
    if (t.son0[c] >= 0) t.level_nonleaf[t.level[c]].push_back(c);
  // bases
  t.xi.resize((size_t)C * 3 * m);
  for (int c = 0; c < C; ++c) cheb_nodes(&t.box[6 * c], m, &t.xi[(size_t)c * 3 * m]);
  std::vector<double> U((size_t)M * p), W((size_t)M * p, 0.0), WK((size_t)M * p, 0.0), E((size_t)C * p * p, 0.0), tmp(p);
  std::vector<int32_t> leaf_of(M);
  for (int li = 0; li < t.n_leaves; ++li) {
    const int c = t.leaves[li];
    const double* xi = &t.xi[(size_t)c * 3 * m];
    for (int k = t.begin[c]; k < t.end[c]; ++k) {
      const int i = t.perm[k];
      leaf_of[k] = li;
      lagrange_3d(xi, m, &g.cen[3 * i], &U[(size_t)k * p]);
      for (int q = 0; q < 7; ++q) {
        lagrange_3d(xi, m, &g.qn[21 * i + 3 * q], tmp.data());
        for (int nu = 0; nu < p; ++nu) W[(size_t)k * p + nu] += kRule.w[q] * tmp[nu];
      }
      for (int nu = 0; nu < p; ++nu) W[(size_t)k * p + nu] *= g.area[i];
      for (int q = 0; q < 7; ++q) {  // double layer: |T_j| sum_q w_q n_j . grad L_nu(y_q)
        lagrange_grad_n_3d(xi, m, &g.qn[21 * i + 3 * q], &g.nrm[3 * i], tmp.data());
        for (int nu = 0; nu < p; ++nu) WK[(size_t)k * p + nu] += kRule.w[q] * tmp[nu];
      }
      for (int nu = 0; nu < p; ++nu) WK[(size_t)k * p + nu] *= g.area[i];
    }
  }
  for (int c = 0; c < C; ++c) {
    const int par = t.parent[c];
    if (par < 0) continue;
    const double* xs = &t.xi[(size_t)c * 3 * m];
    const double* xp = &t.xi[(size_t)par * 3 * m];
    for (int lam = 0; lam < p; ++lam) {
      const double pt[3] = {xs[lam % m], xs[m + (lam / m) % m], xs[2 * m + lam / (m * m)]};
      lagrange_3d(xp, m, pt, &E[(size_t)c * p * p + (size_t)lam * p]);
    }
  }
  // cluster-ordered panel data
  std::vector<double> cen((size_t)3 * M), qn((size_t)21 * M), qw((size_t)7 * M), sj(M), area(M), nrm((size_t)3 * M),
      rawJ(M);
  for (int64_t k = 0; k < M; ++k) {
    const int i = t.perm[k];
    for (int a = 0; a < 3; ++a) cen[3 * k + a] = g.cen[3 * i + a];
    for (int j = 0; j < 21; ++j) qn[21 * k + j] = g.qn[21 * i + j];
    for (int q = 0; q < 7; ++q) qw[7 * k + q] = (kRule.w[q] * g.area[i]) / kFourPi;
    sj[k] = g.J[i] / kFourPi;
    rawJ[k] = g.J[i];
    area[k] = g.area[i];
    for (int a = 0; a < 3; ++a) nrm[3 * k + a] = g.nrm[3 * i + a];
  }
  // near field: per leaf, the flat list of near source panels (cluster order),
  // concatenated column-leaf ranges in partition order
  std::vector<int32_t> leaf_pos(C, -1);
  for (int li = 0; li < t.n_leaves; ++li) leaf_pos[t.leaves[li]] = li;
  // The source leaves of a target leaf are listed by increasing box distance from it (a warp
  // step of 32 consecutive sources is then compact), and every step carries gsuf = the smallest
  // squared distance of the target leaf's box to the centroid of any source from that step on:
  // K1's underflow cutoff leaves the loop once gsuf > (tau / Re s + hmax)^2 (near_common.cuh;
  // every later source is then out of reach too).
  std::vector<std::vector<int32_t>> per_leaf(t.n_leaves);
  {
    auto box_dist = [&](int a, int b) {
      double d2 = 0.0;
      for (int k = 0; k < 3; ++k) {
        const double gp = std::max(0.0, std::max(t.box[6 * a + k] - t.box[6 * b + 3 + k], t.box[6 * b + k] - t.box[6 * a + 3 + k]));
        d2 += gp * gp;
      }
      return d2;
    };
    std::vector<std::vector<std::pair<double, int32_t>>> cols(t.n_leaves);
    for (size_t b = 0; b < t.near_r.size(); ++b)
      cols[leaf_pos[t.near_r[b]]].push_back({box_dist(t.near_r[b], t.near_c[b]), t.near_c[b]});
    for (int li = 0; li < t.n_leaves; ++li) {
      std::stable_sort(cols[li].begin(), cols[li].end(),
                       [](const std::pair<double, int32_t>& x, const std::pair<double, int32_t>& y) { return x.first < y.first; });
      for (auto& e : cols[li])
        for (int j = t.begin[e.second]; j < t.end[e.second]; ++j) per_leaf[li].push_back(j);
    }
  }
  std::vector<int32_t> njb(t.n_leaves), nje(t.n_leaves), nj, ngb(t.n_leaves);
  std::vector<unsigned> gsuf;  // float bits of the squared distances, rounded down
  for (int li = 0; li < t.n_leaves; ++li) {
    njb[li] = (int32_t)nj.size();
    nj.insert(nj.end(), per_leaf[li].begin(), per_leaf[li].end());
    nje[li] = (int32_t)nj.size();
    ngb[li] = (int32_t)gsuf.size();
    const int n = (int)per_leaf[li].size(), ng = (n + 31) / 32;
    const double* bx = &t.box[6 * (size_t)t.leaves[li]];
    gsuf.resize(gsuf.size() + ng);
    double run = 1e300;
    for (int g = ng - 1; g >= 0; --g) {
      for (int i = 32 * g; i < std::min(n, 32 * g + 32); ++i) {
        const int64_t j = per_leaf[li][i];
        double d2 = 0.0;
        for (int k = 0; k < 3; ++k) {
          const double gp = std::max(0.0, std::max(bx[k] - cen[3 * j + k], cen[3 * j + k] - bx[3 + k]));
          d2 += gp * gp;
        }
        run = std::min(run, d2);
      }
      float fr = (float)std::min(run, 1e30);
      if ((double)fr > run) fr = std::nextafterf(fr, 0.0f);
      unsigned ub;
      std::memcpy(&ub, &fr, sizeof ub);
      gsuf[ngb[li] + g] = ub;
    }
  }
  // near blocks grouped by row leaf (partition order within a row): the combined
  // mode's near-field MACA apply walks a row leaf's blocks
  std::vector<int32_t> nb_ptr(t.n_leaves + 1, 0), nb_sorted(t.near_r.size());
  for (size_t b = 0; b < t.near_r.size(); ++b) nb_ptr[leaf_pos[t.near_r[b]] + 1]++;
  for (int li = 0; li < t.n_leaves; ++li) nb_ptr[li + 1] += nb_ptr[li];
  {
    std::vector<int32_t> f(nb_ptr.begin(), nb_ptr.end() - 1);
    for (size_t b = 0; b < t.near_r.size(); ++b) nb_sorted[f[leaf_pos[t.near_r[b]]]++] = (int32_t)b;
  }
  for (int li = 0; li < t.n_leaves; ++li)
    t.max_leaf = std::max(t.max_leaf, t.end[t.leaves[li]] - t.begin[t.leaves[li]]);
  t.nb_ptr = nb_ptr;
  t.nb_sorted = nb_sorted;
  // far CSR by row cluster
  t.far_ptr.assign(C + 1, 0);
  for (size_t b = 0; b < t.far_r.size(); ++b) t.far_ptr[t.far_r[b] + 1]++;
  for (int c = 0; c < C; ++c) t.far_ptr[c + 1] += t.far_ptr[c];
  t.far_sorted.resize(t.far_r.size());
  {
    std::vector<int32_t> f(t.far_ptr.begin(), t.far_ptr.end() - 1);
    for (size_t b = 0; b < t.far_r.size(); ++b) t.far_sorted[f[t.far_r[b]]++] = (int32_t)b;
  }
  if (device == -1) {  // host-only structure (export / inspection; no operator can be built on it)
    *out = h;
    return BEM_OK;
  }
  DeviceGuard dg(device);
  auto fail = [&](bem_status st) { delete h; return st; };
#define UP(buf, vec)                             \
  do {                                           \
    cudaError_t e_ = t.buf.upload(vec);          \
    if (e_ != cudaSuccess) {                     \
      set_error("bem_build_tree: upload %s: %s", #buf, cudaGetErrorString(e_)); \
      return fail(e_ == cudaErrorMemoryAllocation ? BEM_ENOMEM : BEM_ECUDA); \
    }                                            \
  } while (0)
  UP(d_perm, t.perm); UP(d_begin, t.begin); UP(d_end, t.end); UP(d_son0, t.son0); UP(d_son1, t.son1);
  UP(d_parent, t.parent); UP(d_leaf_of, leaf_of);
  t.hmax = 0.0;  // K1's underflow cutoff: r >= |c_i - c_j| - hmax for every quadrature node of panel j
  for (int64_t k = 0; k < t.M; ++k)
    for (int q = 0; q < 7; ++q) {
      const double dx = qn[21 * k + 3 * q] - cen[3 * k], dy = qn[21 * k + 3 * q + 1] - cen[3 * k + 1],
                   dz = qn[21 * k + 3 * q + 2] - cen[3 * k + 2];
      t.hmax = std::max(t.hmax, std::sqrt(dx * dx + dy * dy + dz * dz));
    }
  t.hmax *= 1.0 + 0x1p-40;
  UP(d_cen, cen); UP(d_qn, qn); UP(d_qw, qw); UP(d_selfJ, sj); UP(d_area, area); UP(d_nrm, nrm); UP(d_WK, WK);
  // transposed copies for the downward pass (K2): lanes run over lambda / panel k, so
  // E^T[c][mu][lambda] and U^T[mu][k] make its loads coalesced
  std::vector<double> ET(E.size()), UT(U.size());
  {
    const size_t pp = (size_t)t.p * t.p;
    for (size_t c = 0; c < E.size() / pp; ++c)
      for (int l = 0; l < t.p; ++l)
        for (int mu = 0; mu < t.p; ++mu) ET[c * pp + (size_t)mu * t.p + l] = E[c * pp + (size_t)l * t.p + mu];
    for (int64_t k = 0; k < t.M; ++k)
      for (int mu = 0; mu < t.p; ++mu) UT[(size_t)mu * t.M + k] = U[(size_t)k * t.p + mu];
  }
  // 1-D factors of the transfer matrices (tensor Chebyshev interpolation):
  // E[c][lam][mu] = prod_a E1[c][a][lam_a][mu_a] with E1[c][a] = the parent's axis-a Lagrange
  // polynomials at the son's axis-a nodes (K2 applies E as three m x m mode products)
  std::vector<double> E1((size_t)t.C * 3 * t.m * t.m, 0.0);
  for (int c = 0; c < t.C; ++c) {
    const int par = t.parent[c];
    if (par < 0) continue;
    for (int a = 0; a < 3; ++a) {
      const double* xs = &t.xi[(size_t)c * 3 * t.m + (size_t)a * t.m];
      const double* xp = &t.xi[(size_t)par * 3 * t.m + (size_t)a * t.m];
      for (int lam = 0; lam < t.m; ++lam)
        lagrange_1d(xp, t.m, xs[lam], &E1[(((size_t)c * 3 + a) * t.m + lam) * t.m]);
    }
  }
  UP(d_E1, E1);
  UP(d_U, U); UP(d_W, W); UP(d_E, E); UP(d_ET, ET); UP(d_UT, UT); UP(d_xi, t.xi); UP(d_leaves, t.leaves);
  UP(d_near_jb, njb); UP(d_near_je, nje); UP(d_near_j, nj); UP(d_near_gb, ngb); UP(d_near_gsuf, gsuf);
  UP(d_J, rawJ); UP(d_near_r, t.near_r); UP(d_near_c, t.near_c); UP(d_nb_ptr, nb_ptr); UP(d_nb_sorted, nb_sorted);
  UP(d_far_ptr, t.far_ptr); UP(d_far_sorted, t.far_sorted); UP(d_far_r, t.far_r); UP(d_far_c, t.far_c);
  t.d_level_nonleaf.resize(t.depth + 1);
  for (int lv = 0; lv <= t.depth; ++lv) UP(d_level_nonleaf[lv], t.level_nonleaf[lv]);
#undef UP
  *out = h;
  return BEM_OK;
}

extern "C" bem_status bem_tree_get_stats(bem_tree h, bem_tree_stats* out) {
  BEM_REQ(h && out, "bem_tree_get_stats: NULL argument");
  const Tree& t = h->t;
  out->M = t.M; out->clusters = t.C; out->leaves = t.n_leaves;
  out->near_blocks = (int64_t)t.near_r.size(); out->far_blocks = (int64_t)t.far_r.size();
  out->nnz_near = t.nnz_near; out->depth = t.depth; out->p = t.p;
  return BEM_OK;
}

extern "C" bem_status bem_tree_export(bem_tree h, int32_t* perm, int32_t* clusters, double* boxes,
                                      int32_t* near_pairs, int32_t* far_pairs) {
  BEM_REQ(h, "bem_tree_export: NULL tree");
  const Tree& t = h->t;
  if (perm) std::copy(t.perm.begin(), t.perm.end(), perm);
  if (clusters)
    for (int c = 0; c < t.C; ++c) {
      clusters[5 * c] = t.begin[c]; clusters[5 * c + 1] = t.end[c];
      clusters[5 * c + 2] = t.son0[c]; clusters[5 * c + 3] = t.son1[c]; clusters[5 * c + 4] = t.level[c];
    }
  if (boxes) std::copy(t.box.begin(), t.box.end(), boxes);
  if (near_pairs)
    for (size_t b = 0; b < t.near_r.size(); ++b) { near_pairs[2 * b] = t.near_r[b]; near_pairs[2 * b + 1] = t.near_c[b]; }
  if (far_pairs)
    for (size_t b = 0; b < t.far_r.size(); ++b) { far_pairs[2 * b] = t.far_r[b]; far_pairs[2 * b + 1] = t.far_c[b]; }
  return BEM_OK;
}

extern "C" bem_status bem_tree_destroy(bem_tree h) {
  if (!h) return BEM_OK;
  if (h->t.refcount > 0) {
    set_error("bem_tree_destroy: %d operator(s) still reference this tree", h->t.refcount);
    return BEM_ESTATE;
  }
  DeviceGuard dg(h->t.device);
  delete h;
  return BEM_OK;
}
