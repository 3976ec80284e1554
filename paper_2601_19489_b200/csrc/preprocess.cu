// K1: preprocess -- projection, SH colour, SnugBox and exact pair count.
// Two kernels: (a) cull + compaction of the surviving rows in source order
// (cheap per-CTA work, so the decoupled look-back chain is short), then
// (b) the heavy projection + FP64 tile walk, fully parallel, writing straight
// into the compacted row (pair total by block reduction + one atomic).
//
// Reference semantics:
//   _geometry / project      projection.py:77-136  (cull z <= near or o < 1/255,
//                                                   EWA Sigma2 + 0.3 I, conic, t)
//   _splat_colors / eval_sh  trainer.py:170-178, scene.py:224-230
//   compute_snugboxes        binning.py:87-104
//   bin_sequential count     binning.py:166-215  (exact FP64 column walk)
//   bin_load_balanced count  binning.py:225-286  (FP64 min-q test per tile)
// Rows stay in source order (projection.py:133), pairs are splat-major
// (binning.py:217-221), so the later stable sort reproduces the reference's
// tie order.
#include <cuda_runtime.h>

#include "tsr_common.cuh"

namespace tsr {

constexpr int kScanBlock = 256;
// Look-back values pack (rows, pairs): [61:36] rows (26 bits), [35:0] pairs.
__device__ __forceinline__ unsigned long long pack_rp(unsigned long long rows,
                                                      unsigned long long pairs) {
  return (rows << 36) | pairs;
}

// Block-wide exclusive scan of a packed (rows, pairs) value, then a
// decoupled look-back for the block's global prefix.  Returns the global
// exclusive prefix of this thread; *block_total receives the block aggregate.
__device__ __forceinline__ unsigned long long scan_lookback(
    unsigned long long v, int dyn_bid, unsigned long long* status,
    unsigned long long* s_warp, unsigned long long* s_prefix) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int kWarps = kScanBlock / 32;
  unsigned long long incl = v;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    unsigned long long t = __shfl_up_sync(0xffffffffu, incl, d);
    if (lane >= d) incl += t;
  }
  if (lane == 31) s_warp[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    unsigned long long w = lane < kWarps ? s_warp[lane] : 0ull;
    unsigned long long wi = w;
#pragma unroll
    for (int d = 1; d < kWarps; d <<= 1) {
      unsigned long long t = __shfl_up_sync(0xffffffffu, wi, d);
      if (lane >= d) wi += t;
    }
    unsigned long long agg = __shfl_sync(0xffffffffu, wi, kWarps - 1);
    if (lane < kWarps) s_warp[lane] = wi - w;  // exclusive warp offsets
    const unsigned long long excl = warp_lookback(status, dyn_bid, agg);
    if (lane == 0) {
      s_prefix[0] = excl;
      s_prefix[1] = agg;
    }
  }
  __syncthreads();
  return s_prefix[0] + s_warp[warp] + (incl - v);
}

__device__ __forceinline__ long long count_load_balanced(const SplatF64& s, int tiles_x,
                                                         int tiles_y) {
  SnugRect r = snugbox(s, tiles_x, tiles_y);
  if (r.tx0 > r.tx1 || r.ty0 > r.ty1) return 0;
  long long total = 0;
  for (long long tx = r.tx0; tx <= r.tx1; ++tx) {
    double rx0 = dsub((double)(16 * tx), s.mx);
    double rx1 = dadd(rx0, 16.0);
    for (long long ty = r.ty0; ty <= r.ty1; ++ty) {
      double ry0 = dsub((double)(16 * ty), s.my);
      double ry1 = dadd(ry0, 16.0);
      total += (min_q_box(s, rx0, rx1, ry0, ry1) <= s.t) ? 1 : 0;
    }
  }
  return total;
}

// Exact pair count of one splat plus its compact column-span record (read by
// the rank-major emission in sort.cu, which then needs no FP64 re-walk):
//   x = tx0 | ncols << 16, y = ty_base | overflow << 31,
//   z, w = columns 0..7 as (row offset 4 bits | nrows 4 bits) bytes.
// overflow is set when the span does not fit (the emission then re-walks).
template <int kStrategy = -1>  // -1: runtime `strategy`; 0 / 2: that strategy only
__device__ __forceinline__ long long count_pairs_of(const float* rp, int strategy, int tiles_x,
                                                    int tiles_y, uint4& span) {
  if (kStrategy >= 0) strategy = kStrategy;
  SplatF64 s = load_splat_f64(rp);
  span = make_uint4(0u, 0u, 0u, 0u);
  if (strategy == 1) {
    span.y = 1u << 31;
    return count_load_balanced(s, tiles_x, tiles_y);
  }
  if (strategy == 2) {  // bin_aabb: the whole rectangle, one span code per column
    long long tx0, tx1, ty0, ty1;
    aabb_rect(s, tiles_x, tiles_y, tx0, tx1, ty0, ty1);
    if (tx0 > tx1 || ty0 > ty1) return 0;
    const long long ncols = tx1 - tx0 + 1, nrows = ty1 - ty0 + 1;
    span.x = (uint32_t)(tx0 & 0xffff) | ((uint32_t)(ncols < 255 ? ncols : 255) << 16);
    span.y = (uint32_t)(ty0 & 0xffff);
    if (ncols <= 8 && nrows <= 15) {
      for (long long c = 0; c < ncols; ++c) {
        const uint32_t code = (uint32_t)nrows << 4;
        if (c < 4) span.z |= code << (8 * c);
        else span.w |= code << (8 * (c - 4));
      }
    } else {
      span.y |= 1u << 31;
    }
    return ncols * nrows;
  }
  SnugRect r = snugbox(s, tiles_x, tiles_y);
  if (r.tx0 > r.tx1 || r.ty0 > r.ty1) return 0;
  const long long ncols = r.tx1 - r.tx0 + 1;
  bool fits = ncols <= 8;
  span.x = (uint32_t)(r.tx0 & 0xffff) | ((uint32_t)(ncols < 255 ? ncols : 255) << 16);
  span.y = (uint32_t)(r.ty0 & 0xffff);
  long long total = 0;
  // The column walk of binning.py:186-215 evaluates the y-bounds quadratic
  // at both x edges of every column.  Inside the SnugBox the right edge of
  // column tx (min(16 tx + 16, x_max) - mx with 16 tx + 16 <= x_max) and the
  // left edge of column tx + 1 (max(16 tx + 16, x_min) - mx with
  // 16 tx + 16 >= x_min) are the same FP64 expression on the same operands,
  // so each interior edge is evaluated once (bit-identical to re-evaluating
  // it): ncols + 1 edges instead of 2 ncols (one FP64 sqrt + two divides each).
  const double bbac = dsub(dmul(s.b, s.b), dmul(s.a, s.c));
  const double tc = dmul(s.t, s.c);
  const double negb = -s.b;
  auto edge = [&](double x, double& lo, double& hi) {
    const double rad = dsqrt(npmax(0.0, dadd(dmul(dmul(bbac, x), x), tc)));
    lo = ddiv(dsub(dmul(negb, x), rad), s.c);
    hi = ddiv(dadd(dmul(negb, x), rad), s.c);
  };
  double xl = dsub(npmax((double)(16 * r.tx0), r.x_min), s.mx), lo_l, hi_l;
  edge(xl, lo_l, hi_l);
  const double dx_up = r.dx_up, dx_dn = -r.dx_up, ymax_rel = r.ymax_rel;
  for (long long tx = r.tx0; tx <= r.tx1; ++tx) {
    const double xr = dsub(npmin((double)(16 * tx + 16), r.x_max), s.mx);
    double lo_r, hi_r;
    edge(xr, lo_r, hi_r);
    double ylo = npmin(lo_l, lo_r), yhi = npmax(hi_l, hi_r);
    if (dx_up >= xl && dx_up <= xr) yhi = npmax(yhi, ymax_rel);
    if (dx_dn >= xl && dx_dn <= xr) ylo = npmin(ylo, -ymax_rel);
    long long a0, a1;
    tile_span(dadd(ylo, s.my), dadd(yhi, s.my), tiles_y, a0, a1);
    const long long ty0 = a0 > r.ty0 ? a0 : r.ty0;
    const long long ty1 = a1 < r.ty1 ? a1 : r.ty1;
    const int nr = ty1 - ty0 + 1 > 0 ? (int)(ty1 - ty0 + 1) : 0;
    xl = xr;
    lo_l = lo_r;
    hi_l = hi_r;
    total += nr;
    const long long c = tx - r.tx0;
    const long long off = nr > 0 ? ty0 - r.ty0 : 0;
    if (nr > 15 || off > 15) fits = false;
    if (fits && c < 8) {
      const uint32_t code = ((uint32_t)off & 15u) | ((uint32_t)nr << 4);
      if (c < 4) span.z |= code << (8 * c);
      else span.w |= code << (8 * (c - 4));
    }
  }
  if (!fits) span.y |= 1u << 31;
  return total;
}

// Culling test (projection.py:80-83); shared by both K1 kernels so they agree.
__device__ __forceinline__ bool keep_one(const tsr_gaussians_t& g, const tsr_camera_t& cam,
                                         long long i, float& X, float& Y, float& Z, float& o) {
  const float px = g.positions[3 * i], py = g.positions[3 * i + 1],
              pz = g.positions[3 * i + 2];
  const float* R = cam.R;
  X = fmaf(R[0], px, fmaf(R[1], py, fmaf(R[2], pz, cam.t[0])));
  Y = fmaf(R[3], px, fmaf(R[4], py, fmaf(R[5], pz, cam.t[1])));
  Z = fmaf(R[6], px, fmaf(R[7], py, fmaf(R[8], pz, cam.t[2])));
  o = 1.0f / (1.0f + expf(-g.opacity_logits[i]));
  return (Z > cam.near_plane) && (o >= kMinOpacity);
}

// Projection of one Gaussian into the 12-float raster record.  Returns false
// when culled (projection.py:82).
__device__ __forceinline__ bool project_one(const tsr_gaussians_t& g, const tsr_camera_t& cam,
                                            long long i, float* rec) {
  float X, Y, Z, o;
  if (!keep_one(g, cam, i, X, Y, Z, o)) return false;
  const float px = g.positions[3 * i], py = g.positions[3 * i + 1],
              pz = g.positions[3 * i + 2];
  const float* R = cam.R;

  // R_q from the normalised quaternion (scene.py:33-47)
  float qw = g.rotations[4 * i], qx = g.rotations[4 * i + 1], qy = g.rotations[4 * i + 2],
        qz = g.rotations[4 * i + 3];
  const float qn = rsqrtf(qw * qw + qx * qx + qy * qy + qz * qz);
  qw *= qn; qx *= qn; qy *= qn; qz *= qn;
  float Rq[9];
  Rq[0] = 1.f - 2.f * (qy * qy + qz * qz);
  Rq[1] = 2.f * (qx * qy - qw * qz);
  Rq[2] = 2.f * (qx * qz + qw * qy);
  Rq[3] = 2.f * (qx * qy + qw * qz);
  Rq[4] = 1.f - 2.f * (qx * qx + qz * qz);
  Rq[5] = 2.f * (qy * qz - qw * qx);
  Rq[6] = 2.f * (qx * qz - qw * qy);
  Rq[7] = 2.f * (qy * qz + qw * qx);
  Rq[8] = 1.f - 2.f * (qx * qx + qy * qy);
  const float s0 = expf(g.log_scales[3 * i]), s1 = expf(g.log_scales[3 * i + 1]),
              s2 = expf(g.log_scales[3 * i + 2]);
  // M = R_q diag(s);  Sigma3 = M M^T
  float M[9] = {Rq[0] * s0, Rq[1] * s1, Rq[2] * s2, Rq[3] * s0, Rq[4] * s1,
                Rq[5] * s2, Rq[6] * s0, Rq[7] * s1, Rq[8] * s2};
  const float iz = 1.0f / Z;
  const float j00 = cam.fx * iz, j02 = -cam.fx * X * iz * iz;
  const float j11 = cam.fy * iz, j12 = -cam.fy * Y * iz * iz;
  // A = J R_eff (2x3)
  float A0[3], A1[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    A0[k] = j00 * R[k] + j02 * R[6 + k];
    A1[k] = j11 * R[3 + k] + j12 * R[6 + k];
  }
  // Sigma2 = (A M)(A M)^T + 0.3 I
  float T0[3], T1[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    T0[k] = A0[0] * M[k] + A0[1] * M[3 + k] + A0[2] * M[6 + k];
    T1[k] = A1[0] * M[k] + A1[1] * M[3 + k] + A1[2] * M[6 + k];
  }
  const float s11 = T0[0] * T0[0] + T0[1] * T0[1] + T0[2] * T0[2] + kCovDilation;
  const float s12 = T0[0] * T1[0] + T0[1] * T1[1] + T0[2] * T1[2];
  const float s22 = T1[0] * T1[0] + T1[1] * T1[1] + T1[2] * T1[2] + kCovDilation;
  const float det = s11 * s22 - s12 * s12;
  rec[0] = cam.fx * X * iz + cam.cx;
  rec[1] = cam.fy * Y * iz + cam.cy;
  rec[2] = s22 / det;
  rec[3] = -s12 / det;
  rec[4] = s11 / det;
  rec[5] = o;
  rec[6] = Z;
  rec[7] = fmaxf(0.0f, 2.0f * logf(255.0f * o));
  // colour: SH degree 0 is the raw coefficient (scene.py:227-228)
  const int C = g.sh_coeffs;
  const float* coef = g.colors + (long long)i * C * 3;
  if (C == 1) {
    rec[8] = coef[0];
    rec[9] = coef[1];
    rec[10] = coef[2];
  } else {
    float dx = px - cam.center[0], dy = py - cam.center[1], dz = pz - cam.center[2];
    float inv = rsqrtf(dx * dx + dy * dy + dz * dz);
    dx *= inv; dy *= inv; dz *= inv;
    float basis[16];
    sh_basis(sh_degree_of(C), dx, dy, dz, basis);
    float cr = 0.f, cg = 0.f, cb = 0.f;
    for (int k = 0; k < C; ++k) {
      cr = fmaf(basis[k], coef[3 * k], cr);
      cg = fmaf(basis[k], coef[3 * k + 1], cg);
      cb = fmaf(basis[k], coef[3 * k + 2], cb);
    }
    rec[8] = cr;
    rec[9] = cg;
    rec[10] = cb;
  }
  rec[11] = 0.f;
  return true;
}

// (a) cull + compaction: row_of_source, source_ids and M.  4 consecutive
// Gaussians per thread (N / 1024 blocks: more CTAs in flight beat a shorter
// look-back chain here, measured).
#ifndef TSR_CULL_ITEMS
#define TSR_CULL_ITEMS 4
#endif
constexpr int kCullItems = TSR_CULL_ITEMS;
__global__ void __launch_bounds__(kScanBlock) cull_compact_kernel(
    tsr_gaussians_t g, tsr_camera_t cam, int32_t* __restrict__ source_ids,
    int32_t* __restrict__ row_of_source, int64_t* __restrict__ totals,
    unsigned long long* __restrict__ status, unsigned int* __restrict__ ticket, int n_blocks) {
  __shared__ unsigned long long s_warp[kScanBlock / 32];
  __shared__ unsigned long long s_prefix[2];
  __shared__ int s_bid;
  if (threadIdx.x == 0) s_bid = (int)atomicAdd(ticket, 1u);
  __syncthreads();
  const int bid = s_bid;
  const long long i0 = ((long long)bid * kScanBlock + threadIdx.x) * kCullItems;
  unsigned keep_mask = 0;
#pragma unroll
  for (int k = 0; k < kCullItems; ++k) {
    float X, Y, Z, o;
    if (i0 + k < g.n && keep_one(g, cam, i0 + k, X, Y, Z, o)) keep_mask |= 1u << k;
  }
  unsigned long long excl =
      scan_lookback((unsigned long long)__popc(keep_mask), bid, status, s_warp, s_prefix);
#pragma unroll
  for (int k = 0; k < kCullItems; ++k) {
    const long long i = i0 + k;
    if (i >= g.n) break;
    const bool keep = (keep_mask >> k) & 1u;
    if (keep) source_ids[excl] = (int32_t)i;
    row_of_source[i] = keep ? (int32_t)excl : -1;
    excl += keep ? 1 : 0;
  }
  if (bid == n_blocks - 1 && threadIdx.x == 0) totals[0] = (long long)(s_prefix[0] + s_prefix[1]);
}

// (b) projection + colour + exact pair count into the compacted rows.
// kS: the binning strategy (0 sequential walk, 1 warp-cooperative
// load-balanced, 2 AABB), a template parameter so each instantiation holds
// only its own count code (registers)
#ifndef TSR_K1_MINB
#define TSR_K1_MINB 4
#endif
template <int kS>
__global__ void __launch_bounds__(kScanBlock, kS == 1 ? 3 : TSR_K1_MINB) preprocess_kernel(
    tsr_gaussians_t g, tsr_camera_t cam, int strategy, float4* __restrict__ rec_out,
    const int32_t* __restrict__ row_of_source, int32_t* __restrict__ counts,
    uint32_t* __restrict__ depth_bits, uint4* __restrict__ spans,
    unsigned long long* __restrict__ total_pairs) {
  __shared__ unsigned long long s_sum[kScanBlock / 32];
  constexpr bool kLB = kS == 1;
  __shared__ LbWarp s_lb[kLB ? kScanBlock / 32 : 1];
  const long long i = (long long)blockIdx.x * kScanBlock + threadIdx.x;
  const int tiles_x = tiles_of(cam.width), tiles_y = tiles_of(cam.height);
  long long cnt = 0;
  const int row = i < g.n ? row_of_source[i] : -1;
  if (kLB) {
    float rec[12] = {};
    uint4 span;
    if (row >= 0) project_one(g, cam, i, rec);
    // warp-cooperative: every lane of the warp takes part
    cnt = warp_count_lb(load_splat_f64(rec), row >= 0, tiles_x, tiles_y, span,
                        s_lb[threadIdx.x >> 5]);
    if (row >= 0) {
      float4* dst = rec_out + (long long)row * 3;
      dst[0] = make_float4(rec[0], rec[1], rec[2], rec[3]);
      dst[1] = make_float4(rec[4], rec[5], rec[6], rec[7]);
      dst[2] = make_float4(rec[8], rec[9], rec[10], rec[11]);
      counts[row] = (int32_t)cnt;
      depth_bits[row] = __float_as_uint(rec[6]);
      spans[row] = span;
    }
  } else if (row >= 0) {
    float rec[12];
    project_one(g, cam, i, rec);
    uint4 span;
    cnt = count_pairs_of<kS>(rec, strategy, tiles_x, tiles_y, span);
    float4* dst = rec_out + (long long)row * 3;
    dst[0] = make_float4(rec[0], rec[1], rec[2], rec[3]);
    dst[1] = make_float4(rec[4], rec[5], rec[6], rec[7]);
    dst[2] = make_float4(rec[8], rec[9], rec[10], rec[11]);
    counts[row] = (int32_t)cnt;
    depth_bits[row] = __float_as_uint(rec[6]);
    spans[row] = span;
  }
  unsigned long long v = (unsigned long long)cnt;
  for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
  if ((threadIdx.x & 31) == 0) s_sum[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long t = 0;
    for (int w = 0; w < kScanBlock / 32; ++w) t += s_sum[w];
    if (t) atomicAdd(total_pairs, t);
  }
}

// Pair count + span + depth bits of a caller-built batch; P total by a block
// reduction + one atomic per CTA.
__global__ void __launch_bounds__(kScanBlock) count_kernel(
    const float* __restrict__ rec, long long m, int width, int height, int strategy,
    int32_t* __restrict__ counts, uint32_t* __restrict__ depth_bits, uint4* __restrict__ spans,
    unsigned long long* __restrict__ total_pairs) {
  __shared__ unsigned long long s_sum[kScanBlock / 32];
  __shared__ LbWarp s_lb[kScanBlock / 32];
  const long long i = (long long)blockIdx.x * kScanBlock + threadIdx.x;
  long long cnt = 0;
  uint4 span;
  if (strategy == 1) {
    SplatF64 sf{};
    if (i < m) sf = load_splat_f64(rec + i * 12);
    cnt = warp_count_lb(sf, i < m, tiles_of(width), tiles_of(height), span,
                        s_lb[threadIdx.x >> 5]);
  }
  if (i < m) {
    if (strategy != 1)
      cnt = count_pairs_of(rec + i * 12, strategy, tiles_of(width), tiles_of(height), span);
    counts[i] = (int32_t)cnt;
    depth_bits[i] = __float_as_uint(rec[i * 12 + 6]);
    spans[i] = span;
  }
  unsigned long long v = (unsigned long long)cnt;
  for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
  if ((threadIdx.x & 31) == 0) s_sum[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long t = 0;
    for (int w = 0; w < kScanBlock / 32; ++w) t += s_sum[w];
    if (t) atomicAdd(total_pairs, t);
  }
}

__global__ void snugbox_kernel(const float* __restrict__ rec, long long m, int width,
                               int height, double* x_min, double* x_max, double* y_min,
                               double* y_max, int32_t* tile_rect) {
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  SplatF64 s = load_splat_f64(rec + i * 12);
  SnugRect r = snugbox(s, tiles_of(width), tiles_of(height));
  x_min[i] = r.x_min;
  x_max[i] = r.x_max;
  y_min[i] = r.y_min;
  y_max[i] = r.y_max;
  tile_rect[4 * i] = (int32_t)r.tx0;
  tile_rect[4 * i + 1] = (int32_t)r.tx1;
  tile_rect[4 * i + 2] = (int32_t)r.ty0;
  tile_rect[4 * i + 3] = (int32_t)r.ty1;
}

static size_t scan_workspace(long long n) {
  long long blocks = (n + kScanBlock - 1) / kScanBlock;
  return 256 + (size_t)blocks * sizeof(unsigned long long);
}

}  // namespace tsr

using namespace tsr;

extern "C" size_t tsr_preprocess_workspace(int64_t n) { return scan_workspace(n); }

extern "C" int tsr_preprocess_fwd(const tsr_gaussians_t* g, const tsr_camera_t* cam,
                                  int32_t strategy, float* rec, int32_t* source_ids,
                                  int32_t* row_of_source, int32_t* counts, uint32_t* depth_bits,
                                  void* spans, int64_t* totals, void* workspace,
                                  size_t workspace_bytes, void* stream) {
  if (!g || !cam || g->n < 0 || g->n >= TSR_MAX_GAUSSIANS) return TSR_E_INVALID;
  if (g->sh_coeffs != 1 && g->sh_coeffs != 4 && g->sh_coeffs != 9 && g->sh_coeffs != 16)
    return TSR_E_INVALID;
  if (workspace_bytes < scan_workspace(g->n)) return TSR_E_WORKSPACE;
  cudaStream_t s = (cudaStream_t)stream;
  if (cudaMemsetAsync(totals, 0, 2 * sizeof(int64_t), s) != cudaSuccess) return TSR_E_CUDA;
  if (g->n == 0) return TSR_OK;
  int blocks = (int)((g->n + kScanBlock - 1) / kScanBlock);
  if (cudaMemsetAsync(workspace, 0, scan_workspace(g->n), s) != cudaSuccess) return TSR_E_CUDA;
  unsigned int* ticket = (unsigned int*)workspace;
  unsigned long long* status = (unsigned long long*)((char*)workspace + 256);
  const int cull_blocks = (int)((g->n + kScanBlock * kCullItems - 1) / (kScanBlock * kCullItems));
  cull_compact_kernel<<<cull_blocks, kScanBlock, 0, s>>>(*g, *cam, source_ids, row_of_source,
                                                         totals, status, ticket, cull_blocks);
  TSR_CHECK_LAUNCH();
  auto* pk = strategy == 1   ? preprocess_kernel<1>
             : strategy == 2 ? preprocess_kernel<2>
                             : preprocess_kernel<0>;
  pk<<<blocks, kScanBlock, 0, s>>>(*g, *cam, strategy, (float4*)rec,
                                                  row_of_source, counts, depth_bits,
                                                  (uint4*)spans,
                                                  (unsigned long long*)(totals + 1));
  TSR_CHECK_LAUNCH();
  return TSR_OK;
}

extern "C" int tsr_count_pairs(const float* rec, int64_t m, int32_t width, int32_t height,
                               int32_t strategy, int32_t* counts, uint32_t* depth_bits,
                               void* spans, int64_t* totals, void* stream) {
  if (m < 0 || m >= TSR_MAX_GAUSSIANS || width <= 0 || height <= 0 || !totals)
    return TSR_E_INVALID;
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t host_totals[2] = {m, 0};
  if (cudaMemcpyAsync(totals, host_totals, sizeof(host_totals), cudaMemcpyHostToDevice, s) !=
      cudaSuccess)
    return TSR_E_CUDA;
  if (m == 0) return TSR_OK;
  int blocks = (int)((m + kScanBlock - 1) / kScanBlock);
  count_kernel<<<blocks, kScanBlock, 0, s>>>(rec, m, width, height, strategy, counts, depth_bits,
                                             (uint4*)spans,
                                             (unsigned long long*)(totals + 1));
  TSR_CHECK_LAUNCH();
  return TSR_OK;
}

extern "C" int tsr_snugboxes(const float* rec, int64_t m, int32_t width, int32_t height,
                             double* x_min, double* x_max, double* y_min, double* y_max,
                             int32_t* tile_rect, void* stream) {
  if (m < 0 || width <= 0 || height <= 0) return TSR_E_INVALID;
  if (m == 0) return TSR_OK;
  int blocks = (int)((m + 255) / 256);
  snugbox_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(rec, m, width, height, x_min, x_max,
                                                           y_min, y_max, tile_rect);
  TSR_CHECK_LAUNCH();
  return TSR_OK;
}
