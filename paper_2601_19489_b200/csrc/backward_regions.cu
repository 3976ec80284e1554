// K4r: region-culled per-Gaussian raster backward (backward_per_gaussian,
// backward.py:137-223) -- the training step's backward.
//
// Same arithmetic as K4 (backward.cu): per pixel and list position p, with
// gc_p = <g_color, c_p> + g_depth d_p,
//   T_p = T_seg * prod_{i<p, part_i} (1 - alpha_i)
//   R_p = Ktot + g_T T_f - K_seg - sum_{i<=p} w_i gc_i
//   dL/dalpha_p = T_p gc_p - R_p / (1 - alpha_p)
// and per splat the ten Grad2D sums (backward.py:195-222), merged into
// grad2d with atomics.  Alphas are K3's bit for bit (same operation
// sequence), so participation (p < n_considered, alpha >= 1/255) agrees.
//
// What differs is the schedule.  K4 keeps splats in lanes and streams every
// active pixel of the tile past them, so each (pixel, splat) pair of the
// tile's list costs a full evaluation.  K4r keeps PIXELS in lanes and
// streams the splats past them, and only the splats that blend at >= 1 pixel
// of the lanes' 8x8 region: K3 sees every blend and writes, per (tile, 8x8
// block), the list positions with a blending pixel as the region's list
// (render.cu, RegionArgs) -- exactly the entries with a participating pixel
// (p < n_considered, alpha >= 1/255) here, since K4r evaluates K3's alphas
// bit for bit.  Every other entry contributes exact zeros to every pixel of
// the region, so skipping it changes nothing.
//
// Layout.  A warp's lanes form kGPW groups of kGL lanes; each group runs one
// STREAM -- the entries of one region's list inside one 1024-position
// segment of its tile -- as a kGL-stage systolic pipeline: at step t lane j
// processes stream entry e = t - j for its pixels; the ten per-splat
// partial sums flow lane to lane (one shuffle each), so lane kGL - 1 holds
// entry t - kGL + 1's complete region sums.  The pixel state (T, R) never
// leaves its lane.  Default 8x8 regions: 8-lane groups of 8 pixels per
// lane, four per warp, lane j owning columns x0 = 8 bx + (j & 3), x0 + 4 and
// rows y0 + 2k (k < 4), y0 = 8 by + (j >> 2); 16-lane groups of 4 pixels
// (TSR_K4R_PX=4) and 8x4 regions (TSR_K4R_REGION=4) follow the same pattern
// (rows kGL / 4 apart).  Vertical pixel pairs share dy, so the alpha and
// chain arithmetic is packed FP32x2.  Splat records are staged per group in
// a shared-memory ring of 4 kGL entries (cp.async straight from rec, one
// block of kGL entries a round ahead; the list position and row two and
// three rounds ahead); finished sums go to a kGL-entry buffer and are merged
// kGL at a time, one lane per entry.
//
// Segments and scheduling.  K3 writes a checkpoint record at every segment
// start and the region list offsets at every segment boundary, so a heavy
// tile's work spreads over many streams and warps (the paper's
// redistribution across heavy tiles).  K3 files each
// stream under its length's bucket; a warp's groups take kGPW streams of
// near-equal length at a time, longest first, so the groups that run in
// lockstep rarely idle and the tail holds the short streams.  The tile's
// (segment 0, region 0) stream also counts the tile's merges.
#include <climits>
#include <cstdlib>

#include <cuda_runtime.h>

#include "tsr_common.cuh"

namespace tsr {
namespace {

constexpr int kRWarps = 4;
// 8 pixels per lane: 3 CTAs/SM (167 registers, no spill) measured faster
// than 4 (128 registers with a spill): 345 vs 353 us
#ifndef TSR_K4R_SETUP_FLAT
#define TSR_K4R_SETUP_FLAT 1
#endif
#ifndef TSR_K4R_CTAS_PX8
#define TSR_K4R_CTAS_PX8 3
#endif
#ifndef TSR_K4R_CTAS
#define TSR_K4R_CTAS 4
#endif
constexpr int kRThreads = 32 * kRWarps;

__device__ __forceinline__ float2 f2(float x, float y) { return make_float2(x, y); }
__device__ __forceinline__ float2 bc(float x) { return make_float2(x, x); }

__device__ __forceinline__ float rcp_approx(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(s), "l"(gmem) : "memory");
}
// 8-byte vector atomic add (relaxed, device scope): one L2 request for two fields
__device__ __forceinline__ void red_add2(float* p, float a, float b) {
  asm volatile("red.relaxed.gpu.global.add.v2.f32 [%0], {%1, %2};" ::"l"(p), "f"(a), "f"(b)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

// a = (p < nc && alpha >= 1/255) ? alpha : 0 as one chained compare + select
__device__ __forceinline__ float participate(int p, int nc, float alpha) {
  float a;
  asm("{\n\t.reg .pred q;\n\t"
      "setp.lt.s32 q, %1, %2;\n\t"
      "setp.ge.and.f32 q, %3, %4, q;\n\t"
      "selp.f32 %0, %3, 0f00000000, q;\n\t}"
      : "=f"(a)
      : "r"(p), "r"(nc), "f"(alpha), "f"(kMinAlpha));
  return a;
}

// upstream of a lane's kPX pixels (columns X0, X0 + 4; rows Y0 + k dy) is
// not all zero
template <int kPX>
__device__ __forceinline__ bool lane_nz(const float* __restrict__ grad_color,
                                        const float* __restrict__ grad_depth,
                                        const float* __restrict__ grad_final_T, int width,
                                        int height, int X0, int Y0, int dy) {
  bool nz = false;
#pragma unroll
  for (int q = 0; q < kPX; ++q) {
    const int x = X0 + (q & 1) * 4, y = Y0 + (q >> 1) * dy;
    if (x < width && y < height) {
      const long long pix = (long long)y * width + x;
      nz |= grad_color[3 * pix] != 0.f || grad_color[3 * pix + 1] != 0.f ||
            grad_color[3 * pix + 2] != 0.f || (grad_depth && grad_depth[pix] != 0.f) ||
            (grad_final_T && grad_final_T[pix] != 0.f);
    }
  }
  return nz;
}

// kGL lanes per region pipeline, kPX pixels per lane (two columns x kPX/2
// rows; rows of a lane are kGL/4 apart): kGL x kPX = the region's pixels.
//   (16, 4): 8x8 regions, 4 per tile, 2 per warp
//   ( 8, 4): 8x4 regions, 8 per tile, 4 per warp
//   ( 8, 8): 8x8 regions, 4 per tile, 4 per warp (half the fill and half
//            the per-step shuffles / loads per pixel)
//   ( 4, 8): 8x4 regions, 8 per tile, 8 per warp
template <bool kDepth, int kGL, int kPX>
__global__ void __launch_bounds__(kRThreads, kPX == 8 ? TSR_K4R_CTAS_PX8 : TSR_K4R_CTAS)
    render_bwd_regions_kernel(
    const float4* __restrict__ rec, const int32_t* __restrict__ values,
    const int64_t* __restrict__ offsets, int width, int height, int tiles_x,
    const float* __restrict__ color, const float* __restrict__ depth,
    const float* __restrict__ final_T, const int32_t* __restrict__ n_considered,
    const float* __restrict__ ckpt, const int64_t* __restrict__ ckpt_base,
    const uint32_t* __restrict__ rlist, const int32_t* __restrict__ rseg,
    const float* __restrict__ grad_color, const float* __restrict__ grad_depth,
    const float* __restrict__ grad_final_T, float* __restrict__ grad2d,
    unsigned long long* __restrict__ merges, const uint32_t* __restrict__ units,
    const int32_t* __restrict__ bucket_counts, int32_t* __restrict__ counter) {
  constexpr int kGPW = 32 / kGL;               // regions (lane groups) per warp
  constexpr int kRS = kGL / 4;                 // row stride of a lane's pixels
  constexpr int kRH = kRS * (kPX / 2);         // region height
  constexpr int kNR = kTilePixels / (kGL * kPX);  // regions per tile
  constexpr int kUPS = kNR / kGPW;             // units per (tile, segment): 1 or 2
  constexpr int kNRG = kPX / 4;                // row pairs (packed FP32x2) of a lane
  constexpr int kNQ = 2 * kNRG;                // pixel pairs of a lane: (column, row pair)
  constexpr int kRing = 4 * kGL;               // staged list entries per group (4 blocks of kGL)
  constexpr int kOut = kGL;                    // finished-entry sums per group (one round)
  constexpr int kPR = 2 * kRing;               // position / row ring depth (8 blocks)
  static_assert(kNR * kGL * kPX == kTilePixels && kUPS >= 1, "region shape");
  // one group's ring: a slot's three records share one address register
  struct GroupRing {
    float4 a[kRing];   // mx, my, a, b
    float4 b[kRing];   // c, opacity, depth, level t
    float4 c[kRing];   // r, g, b, -
  };
  __shared__ GroupRing s_ring[kRWarps][kGPW];
  // finished sums, group-minor so the warp's last-lane stores share a line
  __shared__ float4 s_oa[kRWarps][kOut][kGPW];   // sums: gq dx, gq dy, gq dxx, gq dxy
  __shared__ float4 s_ob[kRWarps][kOut][kGPW];   //       gq dyy, ld alpha, w g_r, w g_g
  __shared__ float2 s_oc[kRWarps][kOut][kGPW];   //       w g_b, w g_d
  // list positions (staged 3 rounds ahead, read by the steps) and rows (2
  // rounds ahead, read by the staging and the merge); block b's slots are
  // reused by block b + 8, whose position is fetched at round b + 5, after
  // block b's last step (round b + 1) and merge (end of round b + 1)
  __shared__ int2 s_pr[kRWarps][kGPW][kPR];  // (list position, batch row)
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, h = lane / kGL, j = lane % kGL;
  float4* ra = s_ring[warp][h].a;
  float4* rb = s_ring[warp][h].b;
  float4* rc = s_ring[warp][h].c;
  float4(*oa)[kGPW] = s_oa[warp];
  float4(*ob)[kGPW] = s_ob[warp];
  float2(*oc)[kGPW] = s_oc[warp];
  int2* spr = s_pr[warp][h];
  // sentinel splat: alpha = gauss = 0 at every pixel, finite products
  const float4 sent_a = make_float4(-65536.f, -65536.f, 1.f, 0.f);
  const float4 sent_b = make_float4(1.f, 1.f, 0.f, 0.f);
  const float4 zero4 = make_float4(0.f, 0.f, 0.f, 0.f);
  const float keep = j != 0 ? 1.f : 0.f;  // lane 0 of a group starts each entry's sums
  // streams (tsr_common.cuh) are drawn longest first: kGPW at a time per
  // warp, one per lane group, in descending bucket order; s_spre[b] = the
  // streams in buckets above b (bucket kStreamBuckets - 1 first)
  __shared__ int s_spre[kStreamBuckets + 1];
  const int n_tiles_all = tiles_x * ((height + kTile - 1) / kTile);
  const long long cap = tsr_stream_bucket_cap(offsets[n_tiles_all], n_tiles_all);
  const uint4* __restrict__ recs = reinterpret_cast<const uint4*>(units + kStreamBuckets * cap);
  if (threadIdx.x == 0) {
    int acc = 0;
    for (int bk = kStreamBuckets - 1; bk >= 0; --bk) {
      s_spre[bk] = acc;
      acc += bucket_counts[bk];
    }
    s_spre[kStreamBuckets] = acc;  // all streams
  }
  __syncthreads();
  const int n_streams = s_spre[kStreamBuckets];

  for (;;) {
    int u = 0;
    if (lane == 0) u = atomicAdd(counter, 1);
    u = __shfl_sync(0xffffffffu, u, 0);
    if (u * kGPW >= n_streams) break;
    // this group's stream: index u kGPW + h in descending bucket order
    const int si = u * kGPW + h;
    int tile = 0, seg = 0, r = 0, s_n = 0, s_e0 = 0, s_L = 0;
    uint32_t s_start = 0;
    const bool has = si < n_streams;
    if (has) {
      // s_spre is non-increasing in b; si lies in the smallest bucket b with
      // s_spre[b] <= si (si < s_spre[b - 1] = s_spre[b] + count[b])
      int lo = 0, hi = kStreamBuckets - 1;
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (s_spre[mid] <= si) hi = mid;
        else lo = mid + 1;
      }
      const uint32_t id = units[lo * cap + (si - s_spre[lo])];
      const uint4 ra0 = recs[2 * id], ra1 = recs[2 * id + 1];
      tile = (int)(ra0.x >> 16);
      seg = (int)((ra0.x >> 3) & 0x1fffu);
      r = (int)(ra0.x & 7u);
      s_start = ra0.y;
      s_n = (int)ra0.z;
      s_e0 = (int)ra0.w;
      s_L = (int)ra1.x;
    }
    const long long start = s_start;
    const int n = s_n;
    const int e0 = s_e0;
    int L = s_L;
    const bool counts_merges = has && seg == 0 && r == 0;  // the tile's merge count
    const int tyi = tile / tiles_x, txi = tile - tyi * tiles_x;
    const int X0 = txi * kTile + 8 * (r & 1) + (j & 3), Y0 = tyi * kTile + kRH * (r >> 1) + (j >> 2);
    const int p0 = seg << kSegShift;
    if (!__any_sync(0xffffffffu, L > 0 || counts_merges)) continue;  // nothing to stream

    // ---- pixel state: pair q = (column c = q / kNRG, row pair g = q % kNRG):
    // pixels (X0 + 4c, Y0 + 2g kRS) and (X0 + 4c, Y0 + (2g + 1) kRS)
    float2 T[kNQ], R[kNQ], gr[kNQ], gg[kNQ], gb[kNQ], gd[kNQ];
    int nc[kNQ][2];
    bool nzl = false;
    // ckpt_base[tile] == offsets[tile] >> 5 (the index's record base)
    const float* ck = seg > 0 ? ckpt + ((start >> 5) + ((long long)seg << (kSegShift - 5)) - 1) *
                                           (5 * kTilePixels)
                              : nullptr;
#if TSR_K4R_SETUP_FLAT
    // every load of the lane's pixels first (one round trip instead of a
    // load -> test -> load chain per pixel); out-of-frame pixels read pixel 0
    // and are masked below -- the arithmetic of the active ones is unchanged
    float l_gr[kPX], l_gg[kPX], l_gb[kPX], l_gd[kPX], l_gt[kPX], l_cr[kPX], l_cg[kPX], l_cb[kPX],
        l_ft[kPX], l_dp[kPX], l_kt[kPX], l_kr[kPX], l_kg[kPX], l_kb[kPX], l_kd[kPX];
    int l_nc[kPX];
    bool l_in[kPX];
#pragma unroll
    for (int pp = 0; pp < kPX; ++pp) {
      const int q = pp >> 1, e = pp & 1;
      const int x = X0 + 4 * (q / kNRG), y = Y0 + (2 * (q % kNRG) + e) * kRS;
      l_in[pp] = x < width && y < height;
      const long long pix = l_in[pp] ? (long long)y * width + x : 0;
      l_gr[pp] = grad_color[3 * pix];
      l_gg[pp] = grad_color[3 * pix + 1];
      l_gb[pp] = grad_color[3 * pix + 2];
      l_gd[pp] = (kDepth && grad_depth) ? grad_depth[pix] : 0.f;
      l_gt[pp] = grad_final_T ? grad_final_T[pix] : 0.f;
      l_nc[pp] = n_considered[pix];
      l_cr[pp] = color[3 * pix];
      l_cg[pp] = color[3 * pix + 1];
      l_cb[pp] = color[3 * pix + 2];
      l_ft[pp] = final_T[pix];
      l_dp[pp] = kDepth ? depth[pix] : 0.f;
      l_kt[pp] = l_kr[pp] = l_kg[pp] = l_kb[pp] = l_kd[pp] = 0.f;
      if (ck) {
        const int lp = l_in[pp] ? (y - tyi * kTile) * kTile + (x - txi * kTile) : 0;
        l_kt[pp] = ck[lp];
        l_kr[pp] = ck[kTilePixels + lp];
        l_kg[pp] = ck[2 * kTilePixels + lp];
        l_kb[pp] = ck[3 * kTilePixels + lp];
        if (kDepth) l_kd[pp] = ck[4 * kTilePixels + lp];
      }
    }
#pragma unroll
    for (int q = 0; q < kNQ; ++q) {
      float v[2][6];
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int pp = 2 * q + e;
        float t0 = 0.f, r0 = 0.f, g_r = 0.f, g_g = 0.f, g_b = 0.f, g_d = 0.f;
        int ncv = 0;
        if (l_in[pp]) {
          g_r = l_gr[pp];
          g_g = l_gg[pp];
          g_b = l_gb[pp];
          g_d = l_gd[pp];
          const float gt = l_gt[pp];
          nzl |= (g_r != 0.f) || (g_g != 0.f) || (g_b != 0.f) || (g_d != 0.f) || (gt != 0.f);
          ncv = l_nc[pp];
          if (ncv > p0) {  // active in this segment
            float k = g_r * l_cr[pp] + g_g * l_cg[pp] + g_b * l_cb[pp] + gt * l_ft[pp];
            if (kDepth) k += g_d * l_dp[pp];
            float T0 = 1.f, K0 = 0.f;
            if (ck) {
              T0 = l_kt[pp];
              K0 = g_r * l_kr[pp] + g_g * l_kg[pp] + g_b * l_kb[pp];
              if (kDepth) K0 += g_d * l_kd[pp];
            }
            t0 = T0;
            r0 = k - K0;
          }
        }
        v[e][0] = t0; v[e][1] = r0; v[e][2] = g_r; v[e][3] = g_g; v[e][4] = g_b; v[e][5] = g_d;
        nc[q][e] = ncv;
      }
      T[q] = f2(v[0][0], v[1][0]);
      R[q] = f2(v[0][1], v[1][1]);
      gr[q] = f2(v[0][2], v[1][2]);
      gg[q] = f2(v[0][3], v[1][3]);
      gb[q] = f2(v[0][4], v[1][4]);
      gd[q] = f2(v[0][5], v[1][5]);
    }
#else
#pragma unroll
    for (int q = 0; q < kNQ; ++q) {
      float v[2][6];
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int x = X0 + 4 * (q / kNRG), y = Y0 + (2 * (q % kNRG) + e) * kRS;
        float t0 = 0.f, r0 = 0.f, g_r = 0.f, g_g = 0.f, g_b = 0.f, g_d = 0.f;
        int ncv = 0;
        if (x < width && y < height) {
          const long long pix = (long long)y * width + x;
          g_r = grad_color[3 * pix];
          g_g = grad_color[3 * pix + 1];
          g_b = grad_color[3 * pix + 2];
          if (kDepth && grad_depth) g_d = grad_depth[pix];
          const float gt = grad_final_T ? grad_final_T[pix] : 0.f;
          nzl |= (g_r != 0.f) || (g_g != 0.f) || (g_b != 0.f) || (g_d != 0.f) || (gt != 0.f);
          ncv = n_considered[pix];
          if (ncv > p0) {  // active in this segment
            float k = g_r * color[3 * pix] + g_g * color[3 * pix + 1] + g_b * color[3 * pix + 2] +
                      gt * final_T[pix];
            if (kDepth) k += g_d * depth[pix];
            float T0 = 1.f, K0 = 0.f;
            if (ck) {
              const int lp = (y - tyi * kTile) * kTile + (x - txi * kTile);
              T0 = ck[lp];
              K0 = g_r * ck[kTilePixels + lp] + g_g * ck[2 * kTilePixels + lp] +
                   g_b * ck[3 * kTilePixels + lp];
              if (kDepth) K0 += g_d * ck[4 * kTilePixels + lp];
            }
            t0 = T0;
            r0 = k - K0;
          }
        }
        v[e][0] = t0; v[e][1] = r0; v[e][2] = g_r; v[e][3] = g_g; v[e][4] = g_b; v[e][5] = g_d;
        nc[q][e] = ncv;
      }
      T[q] = f2(v[0][0], v[1][0]);
      R[q] = f2(v[0][1], v[1][1]);
      gr[q] = f2(v[0][2], v[1][2]);
      gg[q] = f2(v[0][3], v[1][3]);
      gb[q] = f2(v[0][4], v[1][4]);
      gd[q] = f2(v[0][5], v[1][5]);
    }
#endif
    // merges follow the reference's count: every pair of a tile whose
    // upstream is not all zero (backward.py:156-158, 214-222); the tile's
    // (segment 0, region 0) stream checks all of its regions
    const unsigned gmask = (kGL == 32 ? 0xffffffffu : ((1u << kGL) - 1u)) << (h * kGL);
    if (__any_sync(0xffffffffu, counts_merges)) {
      bool tnz = false;
      if (counts_merges) {
#pragma unroll 1
        for (int q = 0; q < kNR; ++q)
          tnz |= lane_nz<kPX>(grad_color, kDepth ? grad_depth : nullptr, grad_final_T, width, height,
                         txi * kTile + 8 * (q & 1) + (j & 3), tyi * kTile + kRH * (q >> 1) + (j >> 2),
                         kRS);
      }
      const unsigned any_nz = __ballot_sync(0xffffffffu, tnz) & gmask;
      if (counts_merges && j == 0 && any_nz) atomicAdd(merges, (unsigned long long)n);
    }
    // a group whose pixels have no upstream streams exact zeros: skip it
    const bool gnz = (__ballot_sync(0xffffffffu, nzl) & gmask) != 0u;
    if (!gnz) L = 0;
    int Lmax = L;
#pragma unroll
    for (int m = kGL; m < 32; m <<= 1) Lmax = max(Lmax, __shfl_xor_sync(0xffffffffu, Lmax, m));
    if (Lmax == 0) continue;  // exact zeros

    // the region list holds (position, row) pairs (render.cu)
    const uint2* lst = reinterpret_cast<const uint2*>(rlist) + kNR * start + (long long)r * n + e0;
    // Every list access is asynchronous (cp.async into shared memory, waited
    // once per round), three stages per entry e of this lane's group:
    //   (position, row) lst[e]    -> spr   (3 rounds ahead; K3 wrote the rows)
    //   record    rec[row] x 3    -> ring  (1 round ahead)
    auto fetch_pos = [&](int e) {
      if (e < L) cp_async8(&spr[e & (kPR - 1)], lst + e);
      else spr[e & (kPR - 1)] = make_int2(INT_MAX, -1);
    };
    auto stage = [&](int e) {
      const int slot = e & (kRing - 1);
      const int row = spr[e & (kPR - 1)].y;
      if (row >= 0) {
        cp_async16(&ra[slot], rec + 3 * (long long)row);
        cp_async16(&rb[slot], rec + 3 * (long long)row + 1);
        cp_async16(&rc[slot], rec + 3 * (long long)row + 2);
      } else {
        ra[slot] = sent_a;
        rb[slot] = sent_b;
        rc[slot] = zero4;
      }
    };
    __syncwarp();  // the previous unit's merge has read the ring
    // block -1 (the pipeline fill reads entries -kGL..-1): sentinels
    ra[kRing - kGL + j] = sent_a;
    rb[kRing - kGL + j] = sent_b;
    rc[kRing - kGL + j] = zero4;
    spr[kPR - kGL + j] = make_int2(INT_MAX, -1);
    fetch_pos(j);
    fetch_pos(kGL + j);
    fetch_pos(2 * kGL + j);
    cp_async_commit();
    cp_async_wait_all();
    __syncwarp();
    stage(j);
    cp_async_commit();

    float xf[2];
    xf[0] = (float)X0 + 0.5f;
    xf[1] = (float)(X0 + 4) + 0.5f;
    float2 yf[kNRG];
#pragma unroll
    for (int g = 0; g < kNRG; ++g)
      yf[g] = f2((float)(Y0 + 2 * g * kRS) + 0.5f, (float)(Y0 + (2 * g + 1) * kRS) + 0.5f);
    float s_mx = 0.f, s_my = 0.f, s_a = 0.f, s_b = 0.f, s_c = 0.f, s_o = 0.f, s_r = 0.f,
          s_g = 0.f, s_bl = 0.f, s_d = 0.f;
    const float2 one = bc(1.f);

    // one systolic step: entry t - j of this group for the lane's kPX pixels
    // (A, B, pos of a step are loaded one step ahead; the colour record C in
    // the step, first used after the alpha chain)
    auto step = [&](const float4& A, const float4& B, int pos, int t) {
      const float4 C = rc[(t - j) & (kRing - 1)];
      float i_mx = __shfl_up_sync(0xffffffffu, s_mx, 1, kGL);
      float i_my = __shfl_up_sync(0xffffffffu, s_my, 1, kGL);
      float i_a = __shfl_up_sync(0xffffffffu, s_a, 1, kGL);
      float i_b = __shfl_up_sync(0xffffffffu, s_b, 1, kGL);
      float i_c = __shfl_up_sync(0xffffffffu, s_c, 1, kGL);
      float i_o = __shfl_up_sync(0xffffffffu, s_o, 1, kGL);
      float i_r = __shfl_up_sync(0xffffffffu, s_r, 1, kGL);
      float i_g = __shfl_up_sync(0xffffffffu, s_g, 1, kGL);
      float i_bl = __shfl_up_sync(0xffffffffu, s_bl, 1, kGL);
      float i_d = kDepth ? __shfl_up_sync(0xffffffffu, s_d, 1, kGL) : 0.f;
      // alpha: K3's operation sequence (eval_alpha) per pixel
      const float ca = __fmul_rn(A.z, kQScale), cb = __fmul_rn(A.w, 2.0f * kQScale),
                  cc = __fmul_rn(B.x, kQScale);
      float dx[2], dxx[2];
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        dx[c] = __fsub_rn(xf[c], A.x);
        dxx[c] = __fmul_rn(dx[c], dx[c]);
      }
      float2 dy[kNRG], dyy[kNRG], cyy[kNRG];
#pragma unroll
      for (int g = 0; g < kNRG; ++g) {
        dy[g] = __fadd2_rn(yf[g], bc(-A.y));
        dyy[g] = __fmul2_rn(dy[g], dy[g]);
        cyy[g] = __fmul2_rn(bc(cc), dyy[g]);
      }
      // accumulators start from their first term (no adds of zero)
      float2 G[kNRG], H[kNRG];  // per row pair: sum gq, sum gq dx (over the two columns)
      float Sq[2];              // per column: sum gq
      float2 wr, wg, wbl, wd = bc(0.f);
#pragma unroll
      for (int q = 0; q < kNQ; ++q) {
        const int c = q / kNRG, g = q % kNRG;
        const float2 dxy = __fmul2_rn(bc(dx[c]), dy[g]);
        const float2 qs = __ffma2_rn(bc(ca), bc(dxx[c]), __ffma2_rn(bc(cb), dxy, cyy[g]));
        const float2 ga = f2(fast_exp2(qs.x), fast_exp2(qs.y));
        const float2 raw = __fmul2_rn(bc(B.y), ga);
        const float2 al = f2(fminf(kAlphaCap, raw.x), fminf(kAlphaCap, raw.y));
        // non-participants get a = 0: w = 0, T and R unchanged exactly
        const float2 a = f2(participate(pos, nc[q][0], al.x), participate(pos, nc[q][1], al.y));
        const float2 om = __fadd2_rn(one, f2(-a.x, -a.y));
        float2 gc = __ffma2_rn(gr[q], bc(C.x), __ffma2_rn(gg[q], bc(C.y), __fmul2_rn(gb[q], bc(C.z))));
        if (kDepth) gc = __ffma2_rn(gd[q], bc(B.z), gc);
        const float2 w = __fmul2_rn(T[q], a);
        const float2 num = __ffma2_rn(f2(-w.x, -w.y), gc, R[q]);
        const float2 rcp = f2(rcp_approx(om.x), rcp_approx(om.y));
        const float2 dL = __ffma2_rn(f2(-num.x, -num.y), rcp, __fmul2_rn(T[q], gc));
        T[q] = __fmul2_rn(T[q], om);
        R[q] = num;
        // uncapped participants only (backward.py:64,72): a == raw exactly
        // for them; a non-participant with raw == 0 has gauss == 0
        const float2 ld = f2(a.x == raw.x ? dL.x : 0.f, a.y == raw.y ? dL.y : 0.f);
        const float2 gq = __fmul2_rn(ld, al);
        if (c == 0) {
          G[g] = gq;
          H[g] = __fmul2_rn(gq, bc(dx[c]));
        } else {
          G[g] = __fadd2_rn(G[g], gq);
          H[g] = __ffma2_rn(gq, bc(dx[c]), H[g]);
        }
        if (g == 0)
          Sq[c] = gq.x + gq.y;
        else
          Sq[c] += gq.x + gq.y;
        if (q == 0) {
          wr = __fmul2_rn(w, gr[q]);
          wg = __fmul2_rn(w, gg[q]);
          wbl = __fmul2_rn(w, gb[q]);
          if (kDepth) wd = __fmul2_rn(w, gd[q]);
        } else {
          wr = __ffma2_rn(w, gr[q], wr);
          wg = __ffma2_rn(w, gg[q], wg);
          wbl = __ffma2_rn(w, gb[q], wbl);
          if (kDepth) wd = __ffma2_rn(w, gd[q], wd);
        }
      }
      // region sums of this lane's pixels, added to the incoming sums
      float t_mx = H[0].x + H[0].y, t_o = G[0].x + G[0].y;
      float t_b = fmaf(H[0].x, dy[0].x, __fmul_rn(H[0].y, dy[0].y));
      float t_my = fmaf(G[0].x, dy[0].x, __fmul_rn(G[0].y, dy[0].y));
      float t_c = fmaf(G[0].x, dyy[0].x, __fmul_rn(G[0].y, dyy[0].y));
#pragma unroll
      for (int g = 1; g < kNRG; ++g) {
        t_mx += H[g].x + H[g].y;
        t_b = fmaf(H[g].x, dy[g].x, fmaf(H[g].y, dy[g].y, t_b));
        t_my = fmaf(G[g].x, dy[g].x, fmaf(G[g].y, dy[g].y, t_my));
        t_c = fmaf(G[g].x, dyy[g].x, fmaf(G[g].y, dyy[g].y, t_c));
        t_o += G[g].x + G[g].y;
      }
      s_mx = fmaf(i_mx, keep, t_mx);
      s_b = fmaf(i_b, keep, t_b);
      s_my = fmaf(i_my, keep, t_my);
      s_c = fmaf(i_c, keep, t_c);
      s_a = fmaf(dxx[0], Sq[0], fmaf(dxx[1], Sq[1], i_a * keep));
      // sum ld gauss = (sum ld alpha) / o for uncapped participants (alpha =
      // o gauss): the sum of gq holds it; the merge divides by o
      s_o = fmaf(i_o, keep, t_o);
      s_r = fmaf(i_r, keep, wr.x + wr.y);
      s_g = fmaf(i_g, keep, wg.x + wg.y);
      s_bl = fmaf(i_bl, keep, wbl.x + wbl.y);
      if (kDepth) s_d = fmaf(i_d, keep, wd.x + wd.y);
      if (j == kGL - 1) {  // entry t - (kGL - 1) is complete: park its sums
        const int o = (t - (kGL - 1)) & (kOut - 1);
        oa[o][h] = make_float4(s_mx, s_my, s_a, s_b);
        ob[o][h] = make_float4(s_c, s_o, s_r, s_g);
        oc[o][h] = make_float2(s_bl, s_d);
      }
    };
    // merge entry e's region sums (one lane per entry; backward.py:214-222)
    const float ms = 2.0f / kQScale;
    auto flush = [&](int e) {
      if (e < 0 || e >= L) return;
      const float4 A = oa[e & (kOut - 1)][h], B = ob[e & (kOut - 1)][h];
      const float2 Cc = oc[e & (kOut - 1)][h];
      if (!((B.y != 0.f) | (B.z != 0.f) | (B.w != 0.f) | (Cc.x != 0.f) | (Cc.y != 0.f) |
            (A.z != 0.f)))
        return;
      const int slot = e & (kRing - 1);
      const float4 sa = ra[slot];
      const float4 sbr = rb[slot];
      const float cc = __fmul_rn(sbr.x, kQScale);
      const float ca = __fmul_rn(sa.z, kQScale), hb = __fmul_rn(sa.w, kQScale);  // (2b') / 2
      const int row = spr[e & (kPR - 1)].y;
      // sum gq u = a' sum gq dx + b' sum gq dy, likewise v (the conic's rows)
      const float uu = fmaf(ca, A.x, hb * A.y), vv = fmaf(hb, A.x, cc * A.y);
      // five 8-byte vector atomics per row (rows are 40 B: 8-B aligned)
      float* dst = grad2d + (long long)row * TSR_GRAD2D_FLOATS;
      red_add2(dst + 0, ms * 0.5f * uu, ms * 0.5f * vv);
      red_add2(dst + 2, -0.5f * A.z, -A.w);
      red_add2(dst + 4, -0.5f * B.x, __fdiv_rn(B.y, sbr.y));  // sum ld gauss (see the step)
      red_add2(dst + 6, B.z, B.w);
      red_add2(dst + 8, Cc.x, kDepth ? Cc.y : 0.f);
    };

    auto load = [&](float4& A, float4& B, int& pos, int t) {
      const int slot = (t - j) & (kRing - 1);
      A = ra[slot];
      B = rb[slot];
      pos = spr[(t - j) & (kPR - 1)].x;
    };
    const int steps = Lmax + kGL - 1;  // entry Lmax - 1 leaves the last lane at step Lmax + kGL - 2
    const int rounds = (steps + kGL - 1) / kGL;
    cp_async_wait_all();
    __syncwarp();  // block 0 staged
    float4 A0, B0, A1, B1;
    int q0, q1;
    load(A0, B0, q0, 0);
    for (int k = 0; k < rounds; ++k) {
      // block k's records and k + 1, k + 2's (position, row) pairs landed
      // (waited at the previous round's second-to-last step)
      stage(kGL * (k + 1) + j);
      fetch_pos(kGL * (k + 3) + j);
      cp_async_commit();
#pragma unroll 1
      for (int i = 0; i < kGL; i += 2) {
        const int t = kGL * k + i;
        if (t >= steps) break;  // the last round stops at its last step
        if (i == kGL - 2) {  // block k + 1 (the next step's lane 0 entry) has landed
          cp_async_wait_all();
          __syncwarp();
        }
        load(A1, B1, q1, t + 1);
        step(A0, B0, q0, t);
        load(A0, B0, q0, t + 2);
        step(A1, B1, q1, t + 1);
      }
      __syncwarp();
      flush(kGL * k - (kGL - 1) + j);
    }
    cp_async_wait_all();  // the last staged block lands before the ring is reused
  }
}

}  // namespace
}  // namespace tsr

using namespace tsr;

extern "C" size_t tsr_region_list_entries(int32_t width, int32_t height, int64_t p_bound) {
  (void)width;
  (void)height;
  // up to 8 regions per tile, (position, row) pairs of uint32
  return 2 * (8 * (size_t)(p_bound > 0 ? p_bound : 0) + 1);
}

extern "C" size_t tsr_region_unit_entries(int32_t width, int32_t height, int64_t p_bound) {
  if (width <= 0 || height <= 0) return 0;
  // kStreamBuckets buckets, each able to hold every stream id of a P <= p_bound
  // list, then the stream records (8 uint32 each)
  return (size_t)(kStreamBuckets + 8) *
         (size_t)tsr_stream_bucket_cap(p_bound > 0 ? p_bound : 0, tiles_of(width) * tiles_of(height));
}

extern "C" size_t tsr_region_ctl_entries(void) { return kUnitCtl; }

extern "C" size_t tsr_region_seg_entries(int32_t width, int32_t height, int64_t p_bound) {
  if (width <= 0 || height <= 0) return 0;
  return 8 * ((size_t)(p_bound > 0 ? p_bound : 0) / kSeg + (size_t)tiles_of(width) * tiles_of(height) + 1);
}

extern "C" int tsr_render_bwd_regions(const float* rec, const int32_t* values,
                                      const int64_t* offsets, int32_t width, int32_t height,
                                      const float* color, const float* depth,
                                      const float* final_T, const int32_t* n_considered,
                                      const float* ckpt, const int64_t* ckpt_base,
                                      const uint32_t* region_list, const int32_t* region_seg,
                                      const uint32_t* region_units, int32_t* region_ctl,
                                      const float* grad_color, const float* grad_depth,
                                      const float* grad_final_T, float* grad2d,
                                      unsigned long long* merges, int32_t region_height,
                                      void* stream) {
  if (width <= 0 || height <= 0 || !grad_color || !merges || !grad2d || !ckpt || !ckpt_base ||
      !region_list || !region_seg || !region_units || !region_ctl || !offsets ||
      (region_height != 8 && region_height != 4))
    return TSR_E_INVALID;
  const int tx = tiles_of(width), ty = tiles_of(height), n_tiles = tx * ty;
  if (n_tiles >= (1 << 16)) return TSR_E_INVALID;
  cudaStream_t s = (cudaStream_t)stream;
  // 8x8 regions: 16 lanes x 4 pixels (TSR_K4R_PX=4) or 8 lanes x 8 pixels
  // (TSR_K4R_PX=8); 8x4 regions: 8 lanes x 4 pixels or 4 lanes x 8 pixels
  static const int px = getenv("TSR_K4R_PX") ? atoi(getenv("TSR_K4R_PX")) : 8;
  const int shape = region_height == 4 ? (px == 8 ? 3 : 2) : (px == 8 ? 1 : 0);
  using KFn = decltype(&render_bwd_regions_kernel<false, 16, 4>);
  KFn table[4][2] = {
      {render_bwd_regions_kernel<false, 16, 4>, render_bwd_regions_kernel<true, 16, 4>},
      {render_bwd_regions_kernel<false, 8, 8>, render_bwd_regions_kernel<true, 8, 8>},
      {render_bwd_regions_kernel<false, 8, 4>, render_bwd_regions_kernel<true, 8, 4>},
      {render_bwd_regions_kernel<false, 4, 8>, render_bwd_regions_kernel<true, 4, 8>}};
  KFn k = table[shape][grad_depth ? 1 : 0];
  static int per_sm[8] = {0, 0, 0, 0, 0, 0, 0, 0}, sms = 0;
  int& ps = per_sm[2 * shape + (grad_depth ? 1 : 0)];
  if (ps == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ps, k, kRThreads, 0);
    if (ps < 1) ps = 1;
  }
  // region_ctl = (stream bucket counts filed by K3, grab counter; zeroed by K3's launch)
  k<<<sms * ps, kRThreads, 0, s>>>((const float4*)rec, values, offsets, width, height, tx, color,
                                   depth, final_T, n_considered, ckpt, ckpt_base, region_list,
                                   region_seg, grad_color, grad_depth, grad_final_T, grad2d, merges,
                                   region_units, region_ctl, region_ctl + kStreamBuckets);
  TSR_CHECK_LAUNCH();
  return TSR_OK;
}
