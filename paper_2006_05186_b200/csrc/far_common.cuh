// Helpers shared by the K3 coupling kernels (far.cu: far7 / far8 / h2o / generic;
// farq.cu: far10 on the INT8 tensor cores): Chebyshev node coordinates, the slice
// entry from a precomputed (r, 1/(4 pi r)) pair, and where the MACA coefficients
// Z_b[j, t] live (stored pool or the factors-only tile buffer).
#pragma once
#include "common.cuh"
#include "near_common.cuh"
#include "fastmath.cuh"

namespace bem {

// Where the coefficients Z_b[j, t] come from: the stored pool ([r_b][nl] at zoff[b]) or
// the current frequency tile's buffer ([r_b][ZW] at ztoff[b]: leftover columns [0, tb)
// then the tile's DMMA columns; factors-only skeleton).
struct ZSrc {
  const int64_t* zoff;
  const double2* Z;
  int tiled, ZW;  // tiled: Z = tile buffer, zoff = per-block offsets in it
  int64_t zn;     // elements of Z (bounds checks)
};

// far10 (farq.cu): K3 on the INT8 tensor cores, FP64 products emulated by byte slices
struct Far10Args {
  int nl, m, p, rcap, tb, nd;
  int tile0 = 0;  // first frequency tile of this launch (grid y offset)
  int nch = 1;    // mu chunks of 32 rows (grid x = segment * nch + chunk)
  int gmax = 1;   // ACA terms per readout group (int32 level sums stay below 2^31)
  int gx = 0, nitems = 0;  // set by launch_far10: grid x (segments x mu chunks), work items (x tiles)
  int* ctr = nullptr;      // non-null: persistent CTAs taking work items from this counter
  int64_t part_n = 0;
  const int4* segs;
  const int32_t* far_sorted;
  const int32_t* far_c;
  const double* xi;
  const double2* s;
  const int32_t* rank;
  const int32_t* pivk;
  ZSrc z;
  const double2* xhat;
  const double* xmax;  // [C][nl]: max_nu |xhat_c(nu, t)|
  double2* part;
  const int32_t* mask;
  // (block, tile) underflow mask (bit `tile` of skip[b] set: the block's compressed fibres of that
  // frequency tile are below the rounding of the result and are not computed); nullable
  const uint32_t* skip = nullptr;
  const int32_t* colmap = nullptr;  // [tiles][128]: local frequency of every tile column (-1: padding)
  int nfar = 0, ncm = 0;            // entries of skip / colmap (bounds checks)
  // K1 fused into the launch (nctr != nullptr): near-field warps take (target, class tile)
  // items from *nctr (F = 4 classes per item) while the CTA's coupling work runs
  NearArgs na;
  unsigned* nctr = nullptr;
  unsigned n_items = 0;
};
constexpr int kFar10Tile = 128;  // frequency columns per CTA (the MMA's M)
// far10's (block, frequency tile) underflow mask, see far10_skip_kernel (farq.cu)
struct Far10SkipArgs {
  int nfar, nl, m, rcap, tb, nd;
  int tile_lo, tile_hi;  // tiles whose bits are (re)computed
  double delta;
  double sref;  // lower bound of the 1 / diagonal scale: max(1, 1 / (4 hmax))
  const int32_t* far_r;
  const int32_t* far_c;
  const double* xi;
  const double2* s;
  const int32_t* local_l;
  const int32_t* rank;
  const int32_t* pivk;
  ZSrc z;
  const int32_t* colmap;
  uint32_t* skip;
};
cudaError_t launch_far10_skip(const Far10SkipArgs& a, cudaStream_t st);
cudaError_t launch_far10(const Far10Args& a, int nseg, int ntile, cudaStream_t st, int nearw = 0);
cudaError_t launch_xmax(const double2* xhat, int64_t rows, int p, double* out, cudaStream_t st);

namespace {

__device__ __forceinline__ void node(const double* xi, int m, int mu, double* out) {
  out[0] = xi[mu % m];
  out[1] = xi[m + (mu / m) % m];
  out[2] = xi[2 * m + mu / (m * m)];
}

// the same value from a precomputed (r, 1/(4 pi r)) pair (kern_rs' own intermediates:
// bit-identical slice entries)
__device__ __forceinline__ double2 kern_tab(double2 rw, double2 s, const double* etab, const double2* sctab) {
  const double e = fast::exp_neg_tab(-s.x * rw.x, etab) * rw.y;
  double sn, cs;
  fast::sincos_tab(s.y * rw.x, sctab, &sn, &cs);
  return make_double2(e * cs, -e * sn);
}

__device__ __forceinline__ double2 dist_pair(double d2) {
  const double ir = rsqrt(d2);
  return make_double2(d2 * ir, ir * 0.079577471545947667884);  // (r, 1/(4 pi r)) as kern_rs
}

// Z_b[j, t] = zD[j * stride + t] for the tile's DMMA columns t, zL[j * stride + t] for the
// leftover columns t < tb.
__device__ __forceinline__ void zrows(const ZSrc& z, int b, int nl, int tb, int tc0, const double2*& zD,
                                      const double2*& zL, int& stride) {
  zL = z.Z + z.zoff[b];
  if (z.tiled) {
    zD = zL + (tb - tc0);
    stride = z.ZW;
  } else {
    zD = zL;
    stride = nl;
  }
}

}  // namespace
}  // namespace bem
