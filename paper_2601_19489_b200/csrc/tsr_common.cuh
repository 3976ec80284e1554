// Shared device code for the sm_100a tile rasterizer.
//
// Numerics contract:
//   * tile decisions (SnugBox, column walk, min-q test) are evaluated in FP64
//     on the FP32 SplatBatch values upcast to FP64, with exactly the operation
//     order NumPy uses in binning.py:74-222, one rounding per binary op and NO
//     fused multiply-add (explicit __dmul_rn/__dadd_rn/... intrinsics), so the
//     (tile, splat) pairs are bit-identical to the float64 reference;
//   * everything else is FP32.  The alpha of a (pixel, splat) evaluation is
//     computed by ONE inline function with explicit rounding intrinsics so the
//     forward and the backward see bit-identical alphas (forward.py:71-84).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/tilesplat_b200.h"

namespace tsr {

constexpr int kTile = 16;
constexpr int kTilePixels = kTile * kTile;
constexpr int kGroup = 32;  // CHECKPOINT_INTERVAL (forward.py:28)
// region-culled backward segments: list positions per work unit (a multiple
// of 2 kGroup; K3 writes a checkpoint record at every segment start)
#ifndef TSR_SEG_SHIFT
#define TSR_SEG_SHIFT 10
#endif
constexpr int kSegShift = TSR_SEG_SHIFT;
constexpr int kSeg = 1 << kSegShift;
// Region-culled K4 work: one STREAM per (tile, segment, region) -- the
// region's list entries in that 1024-position segment.  K3 files each
// stream with entries (and every tile's (segment 0, region 0) stream, which
// also counts the tile's merges) under its length's bucket once the tile's
// lists are complete: width 4 below 256 entries (64 buckets), width 128
// above (8 more, the last open-ended).  K4r's warps take kGPW streams at a
// time in descending bucket order, one per lane group, so the groups that
// run in lockstep have near-equal lengths and the longest run first.
// Bucket b holds up to tsr_stream_bucket_cap(P, tiles) stream ids at
// units[b * cap ...], its count at ctl[b]; ctl[kStreamBuckets] is the
// backward's grab counter, ctl[kStreamBuckets + 1] the id counter.  Stream
// record id (two uint4 after the buckets, units + kStreamBuckets * cap):
// {tile << 16 | segment << 3 | region, tile list start, tile list length,
// first region-list entry of the segment}, {entries, -, -, -}.
#ifndef TSR_STREAM_BUCKETS_W8
#define TSR_STREAM_BUCKETS_W8 0
#endif
// 0: width 4 below 256 entries (72 buckets); 1: width 8 below 1024 (129);
// 2: width 2 below 256, then 64 (144)
constexpr int kStreamBuckets = TSR_STREAM_BUCKETS_W8 == 1 ? 129 : (TSR_STREAM_BUCKETS_W8 == 2 ? 144 : 72);
constexpr int kUnitCtl = 192;  // ints in the control block (zeroed by K3's launch)
__host__ __device__ inline long long tsr_stream_bucket_cap(long long pairs, int n_tiles) {
  return 8 * (pairs / kSeg + n_tiles + 1);
}
__host__ __device__ inline int tsr_stream_bucket(int length) {
  if (TSR_STREAM_BUCKETS_W8 == 1) return length < 1024 ? length >> 3 : 128;  // width 8
  if (TSR_STREAM_BUCKETS_W8 == 2) {
    if (length < 256) return length >> 1;
    const int b2 = 128 + ((length - 256) >> 6);
    return b2 < kStreamBuckets - 1 ? b2 : kStreamBuckets - 1;
  }
  if (length < 256) return length >> 2;
  const int b = 64 + ((length - 256) >> 7);
  return b < kStreamBuckets - 1 ? b : kStreamBuckets - 1;
}
constexpr float kAlphaCap = 0.99f;                 // forward.py:25
constexpr float kMinAlpha = 1.0f / 255.0f;         // forward.py:26
constexpr float kTTerminate = 1e-4f;               // forward.py:27
constexpr float kCovDilation = 0.3f;               // projection.py:26
constexpr float kMinOpacity = 1.0f / 255.0f;       // projection.py:27
// conic prescale: exp(-q/2) == exp2(q * kQScale) (the cross term carries 2b)
constexpr float kQScale = -0.72134752044448170368f;  // -0.5 * log2(e)

// ------------------------------------------------------------------ FP64 --
// Explicitly rounded FP64 helpers: the compiler may not contract these.
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double ddiv(double a, double b) { return __ddiv_rn(a, b); }
__device__ __forceinline__ double dsqrt(double a) { return __dsqrt_rn(a); }
// numpy.minimum / maximum propagate NaN; inputs here are finite for valid
// batches, and we keep NaN-propagation anyway.
__device__ __forceinline__ double npmin(double a, double b) {
  return (a != a || b != b) ? (a + b) : (a < b ? a : b);
}
__device__ __forceinline__ double npmax(double a, double b) {
  return (a != a || b != b) ? (a + b) : (a > b ? a : b);
}

// Splat parameters upcast to FP64 (rows of the FP32 batch).
struct SplatF64 {
  double mx, my, a, b, c, t;
};

__device__ __forceinline__ SplatF64 load_splat_f64(const float* rec) {
  SplatF64 s;
  s.mx = (double)rec[0];
  s.my = (double)rec[1];
  s.a = (double)rec[2];
  s.b = (double)rec[3];
  s.c = (double)rec[4];
  s.t = (double)rec[7];
  return s;
}

// _tile_span (binning.py:74-84): inclusive tile ids of the closed interval.
// x / 16 == x * 0.0625 exactly in IEEE (power-of-two scaling rounds the same
// exact value), so the FP64 division is replaced by a multiply.
__device__ __forceinline__ void tile_span(double lo, double hi, int n_tiles,
                                          long long& t0, long long& t1) {
  double c0 = ceil(dsub(dmul(lo, 0.0625), 1.0));
  double f1 = floor(dmul(hi, 0.0625));
  long long i0 = (long long)c0;
  long long i1 = (long long)f1;
  t0 = i0 > 0 ? i0 : 0;
  t1 = i1 < (long long)(n_tiles - 1) ? i1 : (long long)(n_tiles - 1);
}

// compute_snugboxes (binning.py:87-104).  Also carries the per-splat
// invariants of the column walk (binning.py:189, 205-206): det, ymax_rel
// (== ey), dx_up.
struct SnugRect {
  double x_min, x_max, y_min, y_max;
  long long tx0, tx1, ty0, ty1;
  double det, ymax_rel, dx_up;
};

__device__ __forceinline__ SnugRect snugbox(const SplatF64& s, int tiles_x, int tiles_y) {
  SnugRect r;
  double det = dsub(dmul(s.a, s.c), dmul(s.b, s.b));
  double ex = dsqrt(ddiv(dmul(s.c, s.t), det));
  double ey = dsqrt(ddiv(dmul(s.a, s.t), det));
  r.x_min = dsub(s.mx, ex);
  r.x_max = dadd(s.mx, ex);
  r.y_min = dsub(s.my, ey);
  r.y_max = dadd(s.my, ey);
  tile_span(r.x_min, r.x_max, tiles_x, r.tx0, r.tx1);
  tile_span(r.y_min, r.y_max, tiles_y, r.ty0, r.ty1);
  r.det = det;
  r.ymax_rel = ey;  // sqrt((a*t)/det), the same expression as binning.py:205
  r.dx_up = dmul(-ddiv(s.b, s.a), ey);
  return r;
}

// Row span [ty0, ty1] of column tx from the column walk of bin_sequential
// (binning.py:186-215).  Returns the number of rows (>= 0).
__device__ __forceinline__ int column_rows(const SplatF64& s, const SnugRect& r,
                                           long long tx, int tiles_y,
                                           long long& ty0, long long& ty1) {
  double xl = dsub(npmax((double)(16 * tx), r.x_min), s.mx);
  double xr = dsub(npmin((double)(16 * tx + 16), r.x_max), s.mx);
  // y_bounds(dx): rad = sqrt(max(0, (b*b - a*c)*dx*dx + t*c))
  double bbac = dsub(dmul(s.b, s.b), dmul(s.a, s.c));
  double tc = dmul(s.t, s.c);
  double negb = -s.b;
  double rad_l = dsqrt(npmax(0.0, dadd(dmul(dmul(bbac, xl), xl), tc)));
  double rad_r = dsqrt(npmax(0.0, dadd(dmul(dmul(bbac, xr), xr), tc)));
  double lo_l = ddiv(dsub(dmul(negb, xl), rad_l), s.c);
  double hi_l = ddiv(dadd(dmul(negb, xl), rad_l), s.c);
  double lo_r = ddiv(dsub(dmul(negb, xr), rad_r), s.c);
  double hi_r = ddiv(dadd(dmul(negb, xr), rad_r), s.c);
  double ylo = npmin(lo_l, lo_r);
  double yhi = npmax(hi_l, hi_r);
  // global y tangent points (per-splat invariants hoisted into SnugRect)
  const double ymax_rel = r.ymax_rel, dx_up = r.dx_up;
  const double dx_dn = -dx_up;
  if (dx_up >= xl && dx_up <= xr) yhi = npmax(yhi, ymax_rel);
  if (dx_dn >= xl && dx_dn <= xr) ylo = npmin(ylo, -ymax_rel);
  long long a0, a1;
  tile_span(dadd(ylo, s.my), dadd(yhi, s.my), tiles_y, a0, a1);
  ty0 = a0 > r.ty0 ? a0 : r.ty0;
  ty1 = a1 < r.ty1 ? a1 : r.ty1;
  long long n = ty1 - ty0 + 1;
  return n > 0 ? (int)n : 0;
}

// bin_aabb's rectangle (binning.py:301-325): the square of half-side
// sqrt(t / lambda_min(conic)) around the mean, in the reference's NumPy
// operation order; every tile of the rectangle is emitted (column-major).
__device__ __forceinline__ void aabb_rect(const SplatF64& s, int tiles_x, int tiles_y,
                                          long long& tx0, long long& tx1, long long& ty0,
                                          long long& ty1) {
  const double half_sum = dmul(dadd(s.a, s.c), 0.5);   // (a + c) / 2.0 (exact halving)
  const double half_diff = dmul(dsub(s.a, s.c), 0.5);  // (a - c) / 2.0
  const double lam_min = dsub(half_sum, dsqrt(dadd(dmul(half_diff, half_diff), dmul(s.b, s.b))));
  const double radius = dsqrt(ddiv(s.t, lam_min));
  tile_span(dsub(s.mx, radius), dadd(s.mx, radius), tiles_x, tx0, tx1);
  tile_span(dsub(s.my, radius), dadd(s.my, radius), tiles_y, ty0, ty1);
}

// Total pairs of one splat under bin_sequential.
__device__ __forceinline__ long long count_sequential(const SplatF64& s, int tiles_x,
                                                      int tiles_y) {
  SnugRect r = snugbox(s, tiles_x, tiles_y);
  long long total = 0;
  if (r.tx0 > r.tx1 || r.ty0 > r.ty1) return 0;
  for (long long tx = r.tx0; tx <= r.tx1; ++tx) {
    long long ty0, ty1;
    total += column_rows(s, r, tx, tiles_y, ty0, ty1);
  }
  return total;
}

// min_q_box (binning.py:241-259): exact min of the quadratic over a box given
// relative to the mean; used by the load-balanced strategy.
__device__ __forceinline__ double min_q_box(const SplatF64& s, double rx0, double rx1,
                                            double ry0, double ry1) {
  bool inside = (rx0 <= 0.0) && (0.0 <= rx1) && (ry0 <= 0.0) && (0.0 <= ry1);
  if (inside) return 0.0;
  auto q = [&](double dx, double dy) {
    // a*dx*dx + 2.0*b*dx*dy + c*dy*dy, left to right
    double t0 = dmul(dmul(s.a, dx), dx);
    double t1 = dmul(dmul(dmul(2.0, s.b), dx), dy);
    double t2 = dmul(dmul(s.c, dy), dy);
    return dadd(dadd(t0, t1), t2);
  };
  auto clip = [](double v, double lo, double hi) {
    // np.clip(v, lo, hi) == minimum(maximum(v, lo), hi)
    return npmin(npmax(v, lo), hi);
  };
  double bc = -ddiv(s.b, s.c);
  double ba = -ddiv(s.b, s.a);
  double y_at_x0 = clip(dmul(bc, rx0), ry0, ry1);
  double y_at_x1 = clip(dmul(bc, rx1), ry0, ry1);
  double x_at_y0 = clip(dmul(ba, ry0), rx0, rx1);
  double x_at_y1 = clip(dmul(ba, ry1), rx0, rx1);
  return npmin(npmin(q(rx0, y_at_x0), q(rx1, y_at_x1)),
               npmin(q(x_at_y0, ry0), q(x_at_y1, ry1)));
}

// ---- load-balanced writing, warp-cooperative (bin_load_balanced,
// binning.py:262-298; lane_test_counts :289-298) ------------
// The 32 lanes of a warp each own one splat.  The candidate tiles of the 32
// SnugBox rectangles (column-major) are flattened into one list and the
// lanes test it round-robin, 32 candidates per round, each with the FP64
// min-q box test (min_q_box <= t).  So a warp spends rounds in proportion to
// its splats' total candidate count, not to the largest rectangle (the
// per-thread loop's divergence).  Per (splat, column) the passing rows are a
// run (the level set is convex); the owner gets its exact count plus the
// same compact span record the sequential walk writes, so the emission in
// sort.cu needs no FP64 re-walk for this strategy either (a span that does
// not fit, or a non-contiguous column, keeps the overflow bit: re-walk).
struct LbSplat {
  double mx, my, a, b, c, t, bc, ba;  // bc = -(b / c), ba = -(b / a): per-splat constants
  int tx0, ty0, ncols, nrows;
  float inv_rows;  // 1 / nrows (FP32)
  float fmx, fmy, fa, fb2, fc, ft, fbc, fba;  // FP32 copies for the filter below
};

__device__ __forceinline__ LbSplat make_lb_splat(const SplatF64& s, const SnugRect& r, int ncols,
                                                 int nrows) {
  LbSplat L;
  L.mx = s.mx; L.my = s.my; L.a = s.a; L.b = s.b; L.c = s.c; L.t = s.t;
  L.bc = ncols ? -ddiv(s.b, s.c) : 0.0;
  L.ba = ncols ? -ddiv(s.b, s.a) : 0.0;
  L.tx0 = ncols ? (int)r.tx0 : 0;
  L.ty0 = ncols ? (int)r.ty0 : 0;
  L.ncols = ncols;
  L.nrows = nrows;
  L.inv_rows = nrows ? 1.0f / (float)nrows : 0.f;
  L.fmx = (float)s.mx; L.fmy = (float)s.my; L.fa = (float)s.a; L.fb2 = (float)(2.0 * s.b);
  L.fc = (float)s.c; L.ft = (float)s.t; L.fbc = (float)L.bc; L.fba = (float)L.ba;
  return L;
}

// FP32 pre-decision of min_q_box <= t for tile (tx, ty): +1 certainly
// passes, -1 certainly fails, 0 too close to call (then the exact FP64 test
// decides).  The batch values, t and the tile edges are FP32-exact, so the
// FP32 evaluation differs from the FP64 one only by rounding: a few units of
// 2^-24 relative on the box coordinates, the hoisted divides and every
// product, i.e. |q32 - q64| <= ~10 eps Q with Q = |a| X^2 + 2|b| X Y + |c| Y^2
// over the box (X, Y its largest |coordinates|; the clipped candidates move
// continuously with their inputs).  The band is 64 eps Q: most candidates
// are decided in FP32 and the decisions are exactly the FP64 ones.
__device__ __forceinline__ int min_q_box_lb32(const LbSplat& S, int tx, int ty) {
  const float rx0 = (float)(16 * tx) - S.fmx, rx1 = rx0 + 16.f;
  const float ry0 = (float)(16 * ty) - S.fmy, ry1 = ry0 + 16.f;
  float qm = 0.f;
  if (!((rx0 <= 0.f) && (0.f <= rx1) && (ry0 <= 0.f) && (0.f <= ry1))) {
    auto q = [&](float dx, float dy) {
      return fmaf(S.fa * dx, dx, fmaf(S.fb2 * dx, dy, S.fc * dy * dy));
    };
    auto clip = [](float v, float lo, float hi) { return fminf(fmaxf(v, lo), hi); };
    const float y0 = clip(S.fbc * rx0, ry0, ry1), y1 = clip(S.fbc * rx1, ry0, ry1);
    const float x0 = clip(S.fba * ry0, rx0, rx1), x1 = clip(S.fba * ry1, rx0, rx1);
    qm = fminf(fminf(q(rx0, y0), q(rx1, y1)), fminf(q(x0, ry0), q(x1, ry1)));
  }
  const float X = fmaxf(fabsf(rx0), fabsf(rx1)), Y = fmaxf(fabsf(ry0), fabsf(ry1));
  const float Q = fabsf(S.fa) * X * X + fabsf(S.fb2) * X * Y + fabsf(S.fc) * Y * Y;
  const float band = 64.f * 5.9604645e-8f * Q + 1e-30f;
  if (qm + band < S.ft) return 1;
  if (qm - band > S.ft) return -1;
  return 0;
}

// column-major candidate j of a rectangle with nrows rows -> (column, row).
// (j + 1/2) / nrows is at least 1 / (2 nrows) from an integer; the FP32
// product's error is below 2.4e-7 x column, so truncation equals j / nrows
// whenever ncols x nrows <= 2^16 (every rectangle: there are < 2^16 tiles).
__device__ __forceinline__ void lb_cell(const LbSplat& S, int j, int& c, int& rr) {
  c = __float2int_rz(((float)j + 0.5f) * S.inv_rows);
  rr = j - c * S.nrows;
}

// min_q_box (binning.py:241-259) with the splat's two divides and 2 b hoisted
// (the same FP64 values the per-box form computes -- 2.0 * b is exact -- so
// decisions are identical).  The batch is finite here (projected splats), so
// the clips use plain min/max (NumPy's NaN propagation never triggers).
__device__ __forceinline__ double min_q_box_lb(const LbSplat& S, double rx0, double rx1,
                                               double ry0, double ry1) {
  if ((rx0 <= 0.0) && (0.0 <= rx1) && (ry0 <= 0.0) && (0.0 <= ry1)) return 0.0;
  const double b2 = dmul(2.0, S.b);
  auto q = [&](double dx, double dy) {
    const double t0 = dmul(dmul(S.a, dx), dx);
    const double t1 = dmul(dmul(b2, dx), dy);
    const double t2 = dmul(dmul(S.c, dy), dy);
    return dadd(dadd(t0, t1), t2);
  };
  auto clip = [](double v, double lo, double hi) { return fmin(fmax(v, lo), hi); };
  const double y0 = clip(dmul(S.bc, rx0), ry0, ry1), y1 = clip(dmul(S.bc, rx1), ry0, ry1);
  const double x0 = clip(dmul(S.ba, ry0), rx0, rx1), x1 = clip(dmul(S.ba, ry1), rx0, rx1);
  return fmin(fmin(q(rx0, y0), q(rx1, y1)), fmin(q(x0, ry0), q(x1, ry1)));
}
struct LbWarp {
  LbSplat sp[32];
  unsigned cnt[32];
  unsigned char ccnt[32][8];    // passing rows per (splat, column < 8)
  unsigned char cstart[32][8];  // first passing row (255: none yet)
  unsigned bad;                 // splats whose span cannot be encoded
};

__device__ __forceinline__ long long warp_count_lb(const SplatF64& s, bool valid, int tiles_x,
                                                   int tiles_y, uint4& span, LbWarp& w) {
  const int lane = threadIdx.x & 31;
  SnugRect r;
  int ncols = 0, nrows = 0;
  if (valid) {
    r = snugbox(s, tiles_x, tiles_y);
    if (r.tx0 <= r.tx1 && r.ty0 <= r.ty1) {
      ncols = (int)(r.tx1 - r.tx0 + 1);
      nrows = (int)(r.ty1 - r.ty0 + 1);
    }
  }
  w.sp[lane] = make_lb_splat(s, r, ncols, nrows);
  w.cnt[lane] = 0;
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    w.ccnt[lane][c] = 0;
    w.cstart[lane][c] = 255;
  }
  if (lane == 0) w.bad = 0;
  const int area = ncols * nrows;
  int incl = area;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, incl, d);
    if (lane >= d) incl += v;
  }
  const int offs = incl - area;
  const int total = __shfl_sync(0xffffffffu, incl, 31);
  __syncwarp();
  bool carry = false;  // pass of the previous candidate (last lane of the last round)
  for (int base = 0; base < total; base += 32) {
    const int k = base + lane;
    const bool active = k < total;
    // owner = the last lane whose offset is <= k (offsets are non-decreasing)
    int o = 0;
#pragma unroll
    for (int st = 16; st > 0; st >>= 1) {
      const int v = __shfl_sync(0xffffffffu, offs, (o + st) & 31);
      if (o + st < 32 && v <= k) o += st;
    }
    const int ob = __shfl_sync(0xffffffffu, offs, o);
    bool pass = false;
    int c = 0, rr = 0;
    if (active) {
      const LbSplat& S = w.sp[o];
      const int j = k - ob;
      lb_cell(S, j, c, rr);
      const int d = min_q_box_lb32(S, S.tx0 + c, S.ty0 + rr);
      if (d == 0) {  // within the FP32 error band: the exact FP64 test
        const double rx0 = dsub((double)(16 * (S.tx0 + c)), S.mx);
        const double ry0 = dsub((double)(16 * (S.ty0 + rr)), S.my);
        pass = min_q_box_lb(S, rx0, dadd(rx0, 16.0), ry0, dadd(ry0, 16.0)) <= S.t;
      } else {
        pass = d > 0;
      }
    }
    bool prev = __shfl_up_sync(0xffffffffu, pass, 1);
    if (lane == 0) prev = carry;
    const bool start = pass && (rr == 0 || !prev);
    const bool head = active && (lane == 0 || rr == 0);  // a new (splat, column) run
    const unsigned pb = __ballot_sync(0xffffffffu, pass);
    const unsigned sb = __ballot_sync(0xffffffffu, start);
    const unsigned hb = __ballot_sync(0xffffffffu, head);
    carry = __shfl_sync(0xffffffffu, pass, 31);
    if (head) {
      const unsigned above = hb & ~((2u << lane) - 1u);  // (2 << 31) wraps to 0: all bits
      const int next = lane == 31 ? 32 : (above ? __ffs(above) - 1 : 32);
      const unsigned seg = (next == 32 ? 0xffffffffu : ((1u << next) - 1u)) & ~((1u << lane) - 1u);
      const unsigned np = __popc(pb & seg), ns = __popc(sb & seg);
      atomicAdd(&w.cnt[o], np);  // one head per (splat, column): several per splat
      if (c < 8) {
        w.ccnt[o][c] += (unsigned char)np;
        if (ns) {
          if (ns > 1 || w.cstart[o][c] != 255) {
            atomicOr(&w.bad, 1u << o);
          } else {
            w.cstart[o][c] = (unsigned char)(rr + (__ffs(sb & seg) - 1 - lane));
          }
        }
      }
    }
    __syncwarp();
  }
  const long long count = w.cnt[lane];
  span = make_uint4(0u, 0u, 0u, 0u);
  if (ncols) {
    span.x = (uint32_t)(r.tx0 & 0xffff) | ((uint32_t)(ncols < 255 ? ncols : 255) << 16);
    span.y = (uint32_t)(r.ty0 & 0xffff);
    bool fits = ncols <= 8 && !((w.bad >> lane) & 1u);
    for (int c = 0; fits && c < ncols; ++c) {
      const unsigned nr = w.ccnt[lane][c];
      const unsigned off = nr ? w.cstart[lane][c] : 0u;
      if (nr > 15 || off > 15) {
        fits = false;
        break;
      }
      const uint32_t code = (off & 15u) | (nr << 4);
      if (c < 4) span.z |= code << (8 * c);
      else span.w |= code << (8 * (c - 4));
    }
    if (!fits) span = make_uint4(span.x, span.y | (1u << 31), 0u, 0u);
  }
  __syncwarp();  // w is reused by the next call
  return count;
}


// The same round-robin walk, emitting: every passing candidate of splat o is
// written as (tile, row[o]) at out_base[o] + (passing
// candidates of o before it, column-major) -- the rank-major emission's
// FP64 re-walk for rows whose span record overflowed (sort.cu).  All 32
// lanes call; `valid` lanes own a splat.
__device__ __forceinline__ void warp_emit_lb(const SplatF64& s, bool valid, int tiles_x,
                                             int tiles_y, uint32_t row, long long out_base,
                                             long long p_cap, uint32_t* __restrict__ pairs,
                                             uint32_t* __restrict__ pair_rows, LbWarp& w) {
  const int lane = threadIdx.x & 31;
  SnugRect r;
  int ncols = 0, nrows = 0;
  if (valid) {
    r = snugbox(s, tiles_x, tiles_y);
    if (r.tx0 <= r.tx1 && r.ty0 <= r.ty1) {
      ncols = (int)(r.tx1 - r.tx0 + 1);
      nrows = (int)(r.ty1 - r.ty0 + 1);
    }
  }
  w.sp[lane] = make_lb_splat(s, r, ncols, nrows);
  w.cnt[lane] = 0;  // passing candidates written so far
  const int area = ncols * nrows;
  int incl = area;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, incl, d);
    if (lane >= d) incl += v;
  }
  const int offs = incl - area;
  const int total = __shfl_sync(0xffffffffu, incl, 31);
  __syncwarp();
  for (int base = 0; base < total; base += 32) {
    const int k = base + lane;
    const bool active = k < total;
    int o = 0;
#pragma unroll
    for (int st = 16; st > 0; st >>= 1) {
      const int v = __shfl_sync(0xffffffffu, offs, (o + st) & 31);
      if (o + st < 32 && v <= k) o += st;
    }
    const int ob = __shfl_sync(0xffffffffu, offs, o);
    const long long ob_out = __shfl_sync(0xffffffffu, out_base, o);
    const uint32_t orow = __shfl_sync(0xffffffffu, row, o);
    bool pass = false;
    int tile = 0;
    if (active) {
      const LbSplat& S = w.sp[o];
      const int j = k - ob;
      int c, rr;
      lb_cell(S, j, c, rr);
      const int d = min_q_box_lb32(S, S.tx0 + c, S.ty0 + rr);
      if (d == 0) {  // within the FP32 error band: the exact FP64 test
        const double rx0 = dsub((double)(16 * (S.tx0 + c)), S.mx);
        const double ry0 = dsub((double)(16 * (S.ty0 + rr)), S.my);
        pass = min_q_box_lb(S, rx0, dadd(rx0, 16.0), ry0, dadd(ry0, 16.0)) <= S.t;
      } else {
        pass = d > 0;
      }
      tile = (S.ty0 + rr) * tiles_x + S.tx0 + c;
    }
    const unsigned pb = __ballot_sync(0xffffffffu, pass);
    // lanes of o's segment in this round: [max(ob - base, 0), lane)
    const int seg0 = ob - base > 0 ? ob - base : 0;
    const unsigned below = ((1u << lane) - 1u) & ~((1u << seg0) - 1u);
    if (pass) {
      const long long g = ob_out + w.cnt[o] + __popc(pb & below);
      if (g < p_cap) {
        pairs[g] = (uint32_t)tile;
        pair_rows[g] = orow;
      }
    }
    __syncwarp();
    // per-splat running counts: every passing lane's owner gains one; the
    // lowest lane of each owner segment adds its segment's total
    {
      const bool first = active && (lane == 0 || k == ob);
      const unsigned fb = __ballot_sync(0xffffffffu, first);
      if (first) {
        const unsigned above = fb & ~((2u << lane) - 1u);
        const int next = lane == 31 ? 32 : (above ? __ffs(above) - 1 : 32);
        const unsigned seg = (next == 32 ? 0xffffffffu : ((1u << next) - 1u)) &
                             ~((1u << lane) - 1u);
        w.cnt[o] += __popc(pb & seg);
      }
    }
    __syncwarp();
  }
  __syncwarp();  // w is reused by the next call
}

// ------------------------------------------------------------------ FP32 --
// Alpha of one (pixel, splat) evaluation (splat_alpha, forward.py:71-84) on
// the prescaled conic (a', b2', c') = kQScale * (a, 2b, c) (b2' = 2 b' is
// exact):
//   dxx = dx dx, dxy = dx dy, dyy = dy dy,
//   q' = a' dxx + (b2' dxy + c' dyy) = kQScale * q,
//   gauss = 2^q' = exp(-q/2), raw = o * gauss, alpha = min(0.99, raw).
// K3 and K4 run exactly this sequence (packed FP32x2 instructions round each
// half like the scalar ones), so their alphas agree bit for bit; K4 reuses
// dxx, dxy, dyy for the conic gradient.
__device__ __forceinline__ float fast_exp2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

struct AlphaEval {
  float dx, dy, gauss, raw, alpha;
};

__device__ __forceinline__ AlphaEval eval_alpha(float px, float py, float mx, float my,
                                                float a, float b2, float c, float o) {
  AlphaEval e;
  e.dx = __fsub_rn(px, mx);
  e.dy = __fsub_rn(py, my);
  const float qs = __fmaf_rn(a, __fmul_rn(e.dx, e.dx),
                             __fmaf_rn(b2, __fmul_rn(e.dx, e.dy),
                                       __fmul_rn(c, __fmul_rn(e.dy, e.dy))));
  e.gauss = fast_exp2(qs);
  e.raw = __fmul_rn(o, e.gauss);
  e.alpha = fminf(kAlphaCap, e.raw);
  return e;
}

// ------------------------------------------------------------------- SH ---
// Real SH basis (scene.py:186-221); l=0 term is 1 (degree 0 == raw RGB).
__device__ __forceinline__ void sh_basis(int deg, float x, float y, float z, float* out) {
  const float C1 = 0.4886025119029199f;
  const float C2[5] = {1.0925484305920792f, -1.0925484305920792f, 0.31539156525252005f,
                       -1.0925484305920792f, 0.5462742152960396f};
  const float C3[7] = {-0.5900435899266435f, 2.890611442640554f, -0.4570457994644658f,
                       0.3731763325901154f, -0.4570457994644658f, 1.445305721320277f,
                       -0.5900435899266435f};
  out[0] = 1.0f;
  if (deg >= 1) {
    out[1] = -C1 * y;
    out[2] = C1 * z;
    out[3] = -C1 * x;
  }
  if (deg >= 2) {
    float xx = x * x, yy = y * y, zz = z * z;
    out[4] = C2[0] * x * y;
    out[5] = C2[1] * y * z;
    out[6] = C2[2] * (2.f * zz - xx - yy);
    out[7] = C2[3] * x * z;
    out[8] = C2[4] * (xx - yy);
    if (deg >= 3) {
      out[9] = C3[0] * y * (3.f * xx - yy);
      out[10] = C3[1] * x * y * z;
      out[11] = C3[2] * y * (4.f * zz - xx - yy);
      out[12] = C3[3] * z * (2.f * zz - 3.f * xx - 3.f * yy);
      out[13] = C3[4] * x * (4.f * zz - xx - yy);
      out[14] = C3[5] * z * (xx - yy);
      out[15] = C3[6] * x * (xx - 3.f * yy);
    }
  }
}

// d basis_k / d dir (sh_basis_grad, scene.py:233-276), accumulated against a
// per-coefficient weight wk: returns sum_k wk * d basis_k / d dir.
__device__ __forceinline__ void sh_basis_vjp(int deg, float x, float y, float z,
                                             const float* wk, float* gdir) {
  const float C1 = 0.4886025119029199f;
  const float C2[5] = {1.0925484305920792f, -1.0925484305920792f, 0.31539156525252005f,
                       -1.0925484305920792f, 0.5462742152960396f};
  const float C3[7] = {-0.5900435899266435f, 2.890611442640554f, -0.4570457994644658f,
                       0.3731763325901154f, -0.4570457994644658f, 1.445305721320277f,
                       -0.5900435899266435f};
  float gx = 0.f, gy = 0.f, gz = 0.f;
  if (deg >= 1) {
    gy += -C1 * wk[1];
    gz += C1 * wk[2];
    gx += -C1 * wk[3];
  }
  if (deg >= 2) {
    gx += C2[0] * y * wk[4];
    gy += C2[0] * x * wk[4];
    gy += C2[1] * z * wk[5];
    gz += C2[1] * y * wk[5];
    gx += C2[2] * (-2.f * x) * wk[6];
    gy += C2[2] * (-2.f * y) * wk[6];
    gz += C2[2] * (4.f * z) * wk[6];
    gx += C2[3] * z * wk[7];
    gz += C2[3] * x * wk[7];
    gx += C2[4] * (2.f * x) * wk[8];
    gy += C2[4] * (-2.f * y) * wk[8];
  }
  if (deg >= 3) {
    float xx = x * x, yy = y * y, zz = z * z;
    gx += C3[0] * 6.f * x * y * wk[9];
    gy += C3[0] * 3.f * (xx - yy) * wk[9];
    gx += C3[1] * y * z * wk[10];
    gy += C3[1] * x * z * wk[10];
    gz += C3[1] * x * y * wk[10];
    gx += C3[2] * (-2.f * x * y) * wk[11];
    gy += C3[2] * (4.f * zz - xx - 3.f * yy) * wk[11];
    gz += C3[2] * 8.f * y * z * wk[11];
    gx += C3[3] * (-6.f * x * z) * wk[12];
    gy += C3[3] * (-6.f * y * z) * wk[12];
    gz += C3[3] * (6.f * zz - 3.f * xx - 3.f * yy) * wk[12];
    gx += C3[4] * (4.f * zz - 3.f * xx - yy) * wk[13];
    gy += C3[4] * (-2.f * x * y) * wk[13];
    gz += C3[4] * 8.f * x * z * wk[13];
    gx += C3[5] * 2.f * x * z * wk[14];
    gy += C3[5] * (-2.f * y * z) * wk[14];
    gz += C3[5] * (xx - yy) * wk[14];
    gx += C3[6] * 3.f * (xx - yy) * wk[15];
    gy += C3[6] * (-6.f * x * y) * wk[15];
  }
  gdir[0] = gx;
  gdir[1] = gy;
  gdir[2] = gz;
}

__host__ __device__ inline int sh_degree_of(int coeffs) {
  return coeffs >= 16 ? 3 : coeffs >= 9 ? 2 : coeffs >= 4 ? 1 : 0;
}

// ------------------------------------------------------- look-back scan ---
// Decoupled look-back status word: [63:62] flag (0 none, 1 aggregate,
// 2 inclusive prefix), [61:0] value.  Called by ALL 32 lanes of one warp;
// returns the exclusive prefix of block `bid` (lanes read 32 predecessors at
// a time, so the walk costs one L2 round trip per 32 blocks).
__device__ __forceinline__ void lb_store(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long lb_load(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ unsigned long long warp_lookback(unsigned long long* status, int bid,
                                                            unsigned long long aggregate) {
  constexpr unsigned long long kAgg = 1ull << 62, kPre = 2ull << 62, kVal = (1ull << 62) - 1;
  const int lane = threadIdx.x & 31;
  if (bid == 0) {
    if (lane == 0) lb_store(&status[0], kPre | aggregate);
    return 0ull;
  }
  if (lane == 0) lb_store(&status[bid], kAgg | aggregate);
  unsigned long long excl = 0;
  int j = bid - 1;
  while (true) {
    const int idx = j - lane;
    unsigned long long s = kPre;  // lanes before block 0 act as a zero prefix
    if (idx >= 0) {
      do {
        s = lb_load(&status[idx]);
      } while ((s >> 62) == 0);
    }
    const unsigned pre = __ballot_sync(0xffffffffu, (s >> 62) == 2);
    const int stop = pre ? __ffs(pre) - 1 : 32;  // nearest predecessor with a prefix
    unsigned long long v = (lane <= stop && idx >= 0) ? (s & kVal) : 0ull;
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
    excl += v;
    if (pre) break;
    j -= 32;
  }
  if (lane == 0) lb_store(&status[bid], kPre | (excl + aggregate));
  return excl;
}

// --------------------------------------------------------------- errors ---
#define TSR_CHECK_LAUNCH()                                   \
  do {                                                       \
    cudaError_t _e = cudaGetLastError();                     \
    if (_e != cudaSuccess) return TSR_E_CUDA;                \
  } while (0)

__host__ __device__ inline int tiles_of(int px) { return (px + kTile - 1) / kTile; }

}  // namespace tsr
