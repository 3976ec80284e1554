// K3: forward rasterizer (render, forward.py:87-161).
//
// One CTA per 16x16 tile, 4 warps; warp w owns an 8x8 pixel block and each
// lane a vertical pixel PAIR (rows y, y + 4), so every per-pixel operation of
// the blend is one packed FP32x2 instruction (FFMA2/FMUL2/FADD2: one issue
// slot for two pixels; dx is shared by the pair).  The tile's depth-sorted
// list is consumed in batches of 256 splats staged in shared memory.  Per
// pixel:
//   alpha = min(0.99, o exp(-q/2)); blend iff alive && alpha >= 1/255;
//   C += T alpha c; D += T alpha d; T *= 1 - alpha; n_considered = k+1 while
//   alive; alive &= T >= 1e-4 AFTER blending (forward.py:125-138).
// Termination: a warp stops scanning once its 64 pixels are dead (warp-level
// early exit) and the CTA stops at the next batch boundary once all 256 are
// dead (forward.py:141-145).
// Culling: for each chunk of 32 staged splats every lane tests one splat
// against the warp's 8x8 block with the exact minimum of its quadratic over
// the block's pixel-centre rectangle (min_q_box, binning.py:241-259, in FP32
// with a safety margin); only splats that can reach alpha >= 1/255 somewhere
// in the block are evaluated.  A skipped splat provably leaves T, C, D
// unchanged, so the outputs are identical; n_considered is restored from the
// termination position.
// Checkpoints (forward.py:139-140): after every 32nd list position the state
// (T, C, D) is stored for each pixel that consumed that position -- exactly
// the records the per-Gaussian backward reads (it enters group g of a pixel
// only when n_considered > 32 g).  Padding records of dead pixels are never
// written (they are never read).
// Scoring (forward.py:132-137; density.py:36-76): a blend whose weight
// w = T alpha >= 1/255 is a "strong" contribution.  kScore selects what is
// done with them, per warp and list position with ballots (deterministic):
//   1  count them per (tile, warp)              -> Contributions sizes
//   2  write (pixel, row) pairs at a scanned (tile, warp) base
//   3  mask-weighted score per row: += weight for every strong contribution
//      to a pixel whose error mask is set (one atomic per warp and splat);
//      the density pass of the trainer uses this form and never materialises
//      the contribution lists.
#include <cstdlib>

#include <cuda_runtime.h>

#include "tsr_common.cuh"

namespace tsr {


// Conservative strip test: can the splat reach alpha >= 1/255 (q <= t) at any
// pixel centre of [x0, x1] x [y0, y1]?  FP32 min of the quadratic over the
// box; the margin (1e-3 relative + 1e-3) dwarfs the FP32 rounding of both
// this test and the alpha evaluation, so a blending splat is never skipped.
__device__ __forceinline__ bool strip_hit(float mx, float my, float a, float b, float c,
                                          float t, float x0, float x1, float y0, float y1) {
  const float rx0 = x0 - mx, rx1 = x1 - mx, ry0 = y0 - my, ry1 = y1 - my;
  float qmin = 0.f;
  if (!(rx0 <= 0.f && rx1 >= 0.f && ry0 <= 0.f && ry1 >= 0.f)) {
    auto q = [&](float dx, float dy) { return fmaf(a * dx, dx, fmaf(2.f * b * dx, dy, c * dy * dy)); };
    // approximate divides: a slightly-off edge argmin only raises the
    // candidate q by a second-order amount, far inside the margin below
    const float bc = __fdividef(-b, c), ba = __fdividef(-b, a);
    const float yx0 = fminf(fmaxf(bc * rx0, ry0), ry1), yx1 = fminf(fmaxf(bc * rx1, ry0), ry1);
    const float xy0 = fminf(fmaxf(ba * ry0, rx0), rx1), xy1 = fminf(fmaxf(ba * ry1, rx0), rx1);
    qmin = fminf(fminf(q(rx0, yx0), q(rx1, yx1)), fminf(q(xy0, ry0), q(xy1, ry1)));
  }
  return qmin <= fmaf(t, 1.001f, 1e-3f);
}

__device__ __forceinline__ float2 bc2(float x) { return make_float2(x, x); }

// One list entry for a vertical pixel pair (same x, rows y and y + 4) of one
// lane, branch-free (predicated): the warp executes it in lockstep.  dx is
// shared; every other per-pixel operation is one packed FP32x2 instruction.
// The alpha sequence is eval_alpha's, so K4 reproduces these alphas bitwise.
// Liveness is T itself: a pixel is alive iff T >= 1e-4.  T starts at 1 and
// only changes by blending, blending needs a live pixel, and the pixel dies
// at the first blend that takes T below 1e-4 (forward.py:138), after which T
// is frozen below the threshold -- so (T >= 1e-4) is exactly the reference's
// alive flag.  Pixels outside the image start at T = 0 (never written).
struct PixPair {
  float2 T, Cr, Cg, Cb, D;
  int nc0, nc1;  // blends so far (popcounts of the per-chunk participation masks)
  int ncons0, ncons1;
  bool strong0, strong1;  // last blend was a strong contribution (w >= 1/255)
  bool part0, part1;      // last entry blended (the backward's participation)
  __device__ __forceinline__ bool alive0() const { return T.x >= kTTerminate; }
  __device__ __forceinline__ bool alive1() const { return T.y >= kTTerminate; }
};

struct ScoreArgs {
  const uint8_t* mask;         // kScore 3: (H, W) error mask
  float weight;                // kScore 3
  float* row_score;            // kScore 3: (M,) += weight per masked strong contribution
  long long* warp_counts;      // kScore 1: (T * 4,)
  const long long* warp_base;  // kScore 2: (T * 4,) exclusive scan of warp_counts
  long long* out_pixel;        // kScore 2
  long long* out_row;          // kScore 2
};

__device__ __forceinline__ void blend_pair(const float4 g, const float4 c, const float4 col,
                                           float pxf, float2 pyf, int pos, PixPair& s) {
  const float dx = __fsub_rn(pxf, g.x);
  const float2 dy = __fadd2_rn(pyf, bc2(-g.y));
  const float dxx = __fmul_rn(dx, dx);
  const float2 dxy = __fmul2_rn(bc2(dx), dy), dyy = __fmul2_rn(dy, dy);
  const float2 qs = __ffma2_rn(bc2(c.x), bc2(dxx),
                               __ffma2_rn(bc2(c.y), dxy, __fmul2_rn(bc2(c.z), dyy)));
  const float2 raw = __fmul2_rn(bc2(g.z), make_float2(fast_exp2(qs.x), fast_exp2(qs.y)));
  const float2 alpha = make_float2(fminf(kAlphaCap, raw.x), fminf(kAlphaCap, raw.y));
  const bool live0 = s.alive0(), live1 = s.alive1();
  const bool b0 = live0 & (alpha.x >= kMinAlpha);
  const bool b1 = live1 & (alpha.y >= kMinAlpha);
  // the non-blending pixel of a pair gets a = 0: w = T * 0 = 0 and
  // T * (1 - 0) = T exactly, so no selects on w and T are needed
  const float2 a = make_float2(b0 ? alpha.x : 0.f, b1 ? alpha.y : 0.f);
  const float2 w = __fmul2_rn(s.T, a);
  s.strong0 = b0 && (w.x >= kMinAlpha);
  s.strong1 = b1 && (w.y >= kMinAlpha);
  s.part0 = b0;
  s.part1 = b1;
  s.Cr = __ffma2_rn(w, bc2(col.x), s.Cr);
  s.Cg = __ffma2_rn(w, bc2(col.y), s.Cg);
  s.Cb = __ffma2_rn(w, bc2(col.z), s.Cb);
  s.D = __ffma2_rn(w, bc2(col.w), s.D);
  s.T = __fmul2_rn(s.T, __fadd2_rn(bc2(1.f), make_float2(-a.x, -a.y)));
}

// Region lists for the region-culled backward (kCkpt 3/4, backward_regions.cu):
// warp w's 8x8 block is region w of the tile (or its two 8x4 halves); every
// list position that blends at >= 1 pixel of the region is appended to the
// region's list, in list order -- exactly the entries with a participating
// pixel (p < n_considered, alpha >= 1/255) in the backward; the others
// contribute exact zeros there.  With kNR regions per tile (4: 8x8, 8: 8x4
// halves) region r of tile t stores its positions at
// list[kNR start_t + r n_t ...] (entries: (list position, batch row) pairs);
// seg[kNR (segbase_t + s - 1) + r]
// holds the number of entries with position < kSeg s for s = 1..ceil(n/kSeg)
// (segbase_t = (start_t >> 10) + t: floor((O + n) / kSeg) - floor(O / kSeg)
// + 1 >= ceil(n / kSeg), so the tiles' segment slots never overlap).
// It also files the tile's streams for the region-culled K4 (one per
// (segment, region) with entries, tsr_common.cuh) under their length's
// bucket once the tile's lists are complete; the control block (bucket
// counts, grab counter) is zeroed before K3 by the launch.
struct RegionArgs {
  uint32_t* list;
  int32_t* seg;
  uint32_t* units;
  int32_t* ctl;
};

// 4 warps; warp w owns the 8x8 block (bx, by) = (w & 1, w >> 1) of the tile;
// lane l owns pixels (8 bx + (l & 7), 8 by + (l >> 3)) and the one 4 rows below.
constexpr int kFwdThreads = 128;
constexpr int kBatch = 256;

// kCkpt: 0 no checkpoints, 1 every record (the reference's checkpoints), 2
// only the odd records -- the ones K4 reads (supergroup starts, 64 positions
// apart): half the checkpoint traffic in the training step; 3 only the
// records at segment starts (every kSeg positions) plus the region lists the
// region-culled backward reads.
template <int kCkpt, int kScore>
__global__ void __launch_bounds__(kFwdThreads) render_fwd_kernel(
    const float4* __restrict__ rec, const int32_t* __restrict__ values,
    const int64_t* __restrict__ offsets, int width, int height, int tiles_x, float bg_r,
    float bg_g, float bg_b, float* __restrict__ out_color, float* __restrict__ out_depth,
    float* __restrict__ out_T, int32_t* __restrict__ out_ncontrib,
    int32_t* __restrict__ out_ncons, float* __restrict__ ckpt,
    const int64_t* __restrict__ ckpt_base, ScoreArgs sc, const int32_t* __restrict__ order,
    RegionArgs rg = RegionArgs{}) {
  // per staged splat: [0] mx, my, opacity, depth  [1] prescaled conic a',
  // 2b', c'  [2] r, g, b, depth -- one base address per list entry
  __shared__ float4 s_spl[kBatch][3];
  __shared__ float4 s_raw[kBatch];  // a, b, c (unscaled), level t
  __shared__ int s_row[(kScore || kCkpt >= 3) ? kBatch : 1];

  // heavy tiles first when an order is given (tile_order_kernel; its last
  // entry flags whether it differs from raster order)
  const int tile = (order && order[gridDim.x]) ? order[blockIdx.x] : (int)blockIdx.x;
  const int tyi = tile / tiles_x, txi = tile - tyi * tiles_x;
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int bx = warp & 1, by = warp >> 1;
  const int lx = 8 * bx + (lane & 7), ly0 = 8 * by + (lane >> 3), ly1 = ly0 + 4;
  const int x = txi * kTile + lx, y0 = tyi * kTile + ly0, y1 = tyi * kTile + ly1;
  const bool in0 = x < width && y0 < height, in1 = x < width && y1 < height;
  const float pxf = (float)x + 0.5f;
  const float2 pyf = make_float2((float)y0 + 0.5f, (float)y1 + 0.5f);
  // this warp's block of pixel centres
  const float sx0 = (float)(txi * kTile + 8 * bx) + 0.5f, sy0 = (float)(tyi * kTile + 8 * by) + 0.5f;
  const long long start = offsets[tile], end = offsets[tile + 1];
  const int n = (int)(end - start);
  float* ck0 = nullptr;
  if (kCkpt) ck0 = ckpt + ckpt_base[tile] * (5 * kTilePixels) + ly0 * kTile + lx;

  PixPair s;
  s.T = make_float2(in0 ? 1.f : 0.f, in1 ? 1.f : 0.f);
  s.Cr = s.Cg = s.Cb = s.D = bc2(0.f);
  s.nc0 = s.nc1 = 0;
  s.ncons0 = s.ncons1 = 0;
  s.strong0 = s.strong1 = false;
  const unsigned lt_mask = (1u << lane) - 1u;
  long long sc_cursor = 0;  // kScore 1/2: this warp's contributions so far
  if (kScore == 2) sc_cursor = sc.warp_base[tile * 4 + warp];
  const long long pix0 = (long long)y0 * width + x, pix1 = (long long)y1 * width + x;
  // region mode: kCkpt 3 = the warp's 8x8 block is one region (4 per tile);
  // kCkpt 4 = its top / bottom 8x4 halves (rows of the lanes' first / second
  // pixels) are two regions, (2 by + half) * 2 + bx (8 per tile)
  constexpr bool kRegions = kCkpt >= 3;
  constexpr int kNR = kCkpt == 4 ? 8 : 4;
  // region list entries are (list position, batch row) pairs
  uint2* rl = nullptr;
  uint2* rl2 = nullptr;
  int r_count = 0, r_count2 = 0, s_next = 1;
  const int reg0 = kCkpt == 4 ? (2 * by) * 2 + bx : warp, reg1 = (2 * by + 1) * 2 + bx;
  const long long segbase = (start >> kSegShift) + tile;
  if (kRegions) rl = reinterpret_cast<uint2*>(rg.list) + kNR * start + (long long)reg0 * n;
  if (kCkpt == 4) rl2 = reinterpret_cast<uint2*>(rg.list) + kNR * start + (long long)reg1 * n;
  bool m0 = false, m1 = false;
  if (kScore == 3) {
    m0 = in0 && sc.mask[pix0];
    m1 = in1 && sc.mask[pix1];
  }

  for (int b0 = 0; b0 < n; b0 += kBatch) {
    if (!__syncthreads_or(s.alive0() || s.alive1())) break;
#pragma unroll
    for (int h = 0; h < kBatch / kFwdThreads; ++h) {
      const int i = tid + h * kFwdThreads;
      const int k = b0 + i;
      if (k < n) {
        const int row = values[start + k];
        const float4 r0 = __ldg(rec + 3 * row), r1 = __ldg(rec + 3 * row + 1),
                     r2 = __ldg(rec + 3 * row + 2);
        s_spl[i][0] = make_float4(r0.x, r0.y, r1.y, r1.z);
        s_spl[i][1] = make_float4(__fmul_rn(r0.z, kQScale), __fmul_rn(r0.w, 2.0f * kQScale),
                                  __fmul_rn(r1.x, kQScale), 0.f);
        s_spl[i][2] = make_float4(r2.x, r2.y, r2.z, r1.z);
        s_raw[i] = make_float4(r0.z, r0.w, r1.x, r1.w);
        if (kScore || kCkpt >= 3) s_row[i] = row;
      }
    }
    __syncthreads();
    const int cnt = min(kBatch, n - b0);
    // chunks of 32 list positions == one checkpoint interval
    for (int c0 = 0; c0 < cnt; c0 += kGroup) {
      const unsigned live_lo = __ballot_sync(0xffffffffu, s.alive0()),
                     live_hi = __ballot_sync(0xffffffffu, s.alive1());
      if (!(live_lo | live_hi)) break;  // warp-level early exit
      // the test rectangle: the pixel centres of the block's LIVE pixels (a
      // dead pixel never blends again, forward.py:125-138), from the two
      // ballots: lane l holds column l & 7 and rows l >> 3 (live_lo), 4 + (l >> 3) (live_hi)
      const unsigned mm = live_lo | live_hi;
      const unsigned cols = (mm | (mm >> 8) | (mm >> 16) | (mm >> 24)) & 0xffu;
      auto rows_of = [](unsigned m) {
        return (unsigned)((m & 0xffu) != 0u) | ((unsigned)((m & 0xff00u) != 0u) << 1) |
               ((unsigned)((m & 0xff0000u) != 0u) << 2) | ((unsigned)((m & 0xff000000u) != 0u) << 3);
      };
      const unsigned rows = rows_of(live_lo) | (rows_of(live_hi) << 4);
      const float bx0 = sx0 + (float)(__ffs(cols) - 1), bx1 = sx0 + (float)(31 - __clz(cols));
      const float by0 = sy0 + (float)(__ffs(rows) - 1), by1 = sy0 + (float)(31 - __clz(rows));
      const int cend = min(kGroup, cnt - c0);
      const int pos0 = b0 + c0;
      if (kRegions && pos0 > 0 && (pos0 & (kSeg - 1)) == 0) {  // segment boundary
        if (lane == 0) {
          rg.seg[kNR * (segbase + s_next - 1) + reg0] = r_count;
          if (kCkpt == 4) rg.seg[kNR * (segbase + s_next - 1) + reg1] = r_count2;
        }
        ++s_next;
      }
      // lane j tests splat c0 + j against this warp's 8x8 block
      bool hit = false;
      if (lane < cend) {
        const float4 g = s_spl[c0 + lane][0], rw = s_raw[c0 + lane];
        hit = strip_hit(g.x, g.y, rw.x, rw.y, rw.z, rw.w, bx0, bx1, by0, by1);
      }
      // hits in list order from the bit-reversed ballot: entry j is the
      // leading one (clz, no per-hit bit reversal), and its bit is reused to
      // clear it and to mark the region lists
      unsigned rev = __brev(__ballot_sync(0xffffffffu, hit));
      // region lists: the chunk's positions that blend at >= 1 pixel of the
      // region (exactly the backward's participating entries), from the
      // blends below (bit-reversed like rev)
      unsigned pm0r = 0u, pm1r = 0u;
      const bool live_c0 = s.alive0(), live_c1 = s.alive1();
      const float4* cbase = s_spl[c0];
      while (rev) {
        const int f = 31 - __clz(rev);  // FLO
        const unsigned bit = 1u << f;
        const int j = 31 - f;
        rev ^= bit;
        const float4* sp = cbase + 3 * j;
        blend_pair(sp[0], sp[1], sp[2], pxf, pyf, pos0 + j, s);
        // per-pixel participation bits of the chunk (bit-reversed): their
        // popcounts are the blend counts, the last one a dead pixel's death
        // entry, and their warp OR the region lists' entries
        if (s.part0) pm0r |= bit;
        if (s.part1) pm1r |= bit;
        if (kScore) {
          const unsigned q0 = __ballot_sync(0xffffffffu, kScore == 3 ? s.strong0 && m0 : s.strong0);
          const unsigned q1 = __ballot_sync(0xffffffffu, kScore == 3 ? s.strong1 && m1 : s.strong1);
          const int nq = __popc(q0) + __popc(q1);
          if (kScore == 3) {
            if (lane == 0 && nq) atomicAdd(sc.row_score + s_row[c0 + j], sc.weight * (float)nq);
          } else {
            if (kScore == 2) {
              const long long row = s_row[c0 + j];
              if (s.strong0) {
                const long long o = sc_cursor + __popc(q0 & lt_mask);
                sc.out_pixel[o] = pix0;
                sc.out_row[o] = row;
              }
              if (s.strong1) {
                const long long o = sc_cursor + __popc(q0) + __popc(q1 & lt_mask);
                sc.out_pixel[o] = pix1;
                sc.out_row[o] = row;
              }
            }
            sc_cursor += nq;
          }
        }
      }
      s.nc0 += __popc(pm0r);
      s.nc1 += __popc(pm1r);
      // a pixel alive at the chunk start that is dead now died at its last
      // blend of the chunk (death needs a blend): it considered the list up
      // to and including that entry (pos0 + j, j = 32 - ffs(reversed bits) - 1)
      if (live_c0 && !s.alive0()) s.ncons0 = pos0 + 33 - __ffs(pm0r);
      if (live_c1 && !s.alive1()) s.ncons1 = pos0 + 33 - __ffs(pm1r);
      const unsigned pm0 =
          kRegions ? __brev(__reduce_or_sync(0xffffffffu, kCkpt == 4 ? pm0r : (pm0r | pm1r))) : 0u;
      const unsigned pm1 = kCkpt == 4 ? __brev(__reduce_or_sync(0xffffffffu, pm1r)) : 0u;
      if (kRegions) {
        if ((pm0 >> lane) & 1u)
          rl[r_count + __popc(pm0 & lt_mask)] = make_uint2((uint32_t)(pos0 + lane), (uint32_t)s_row[c0 + lane]);
        r_count += __popc(pm0);
      }
      if (kCkpt == 4) {
        if ((pm1 >> lane) & 1u)
          rl2[r_count2 + __popc(pm1 & lt_mask)] = make_uint2((uint32_t)(pos0 + lane), (uint32_t)s_row[c0 + lane]);
        r_count2 += __popc(pm1);
      }
      if (kCkpt && cend == kGroup &&
          (kCkpt == 1 || (kCkpt == 2 && ((pos0 >> 5) & 1)) ||
           (kRegions && ((pos0 + kGroup) & (kSeg - 1)) == 0))) {
        // state after list position pos0+31 -> record (pos0+32)/32 - 1, for
        // each pixel that consumed that position (still alive, or died there)
        float* dst = ck0 + (long long)(pos0 >> 5) * (5 * kTilePixels);
        if (s.alive0() || s.ncons0 == pos0 + kGroup) {
          dst[0] = s.T.x;
          dst[kTilePixels] = s.Cr.x;
          dst[2 * kTilePixels] = s.Cg.x;
          dst[3 * kTilePixels] = s.Cb.x;
          dst[4 * kTilePixels] = s.D.x;
        }
        if (s.alive1() || s.ncons1 == pos0 + kGroup) {
          dst += 4 * kTile;
          dst[0] = s.T.y;
          dst[kTilePixels] = s.Cr.y;
          dst[2 * kTilePixels] = s.Cg.y;
          dst[3 * kTilePixels] = s.Cb.y;
          dst[4 * kTilePixels] = s.D.y;
        }
      }
    }
  }
  if (kScore == 1 && lane == 0) sc.warp_counts[tile * 4 + warp] = sc_cursor;
  if (kRegions && lane == 0)  // the remaining segment ends (after an early exit)
    for (const int nseg = (n + kSeg - 1) >> kSegShift; s_next <= nseg; ++s_next) {
      rg.seg[kNR * (segbase + s_next - 1) + reg0] = r_count;
      if (kCkpt == 4) rg.seg[kNR * (segbase + s_next - 1) + reg1] = r_count2;
    }
  if (kRegions) {
    // the tile's K4r streams (tsr_common.cuh): one per (segment, region)
    // with entries, plus (segment 0, region 0) always (it counts merges)
    __syncthreads();  // every warp's segment counts are written
    const int nseg = (n + kSeg - 1) >> kSegShift;
    const long long cap = tsr_stream_bucket_cap(offsets[gridDim.x], gridDim.x);
    // stream records after the buckets (tsr_common.cuh): the buckets hold
    // record ids, so the backward's setup needs no offsets / segment reads
    uint4* recs = reinterpret_cast<uint4*>(rg.units + (long long)kStreamBuckets * cap);
    for (int i = tid; i < nseg * kNR; i += kFwdThreads) {
      const int sg = i / kNR, q = i - sg * kNR;
      const int e0 = sg > 0 ? rg.seg[kNR * (segbase + sg - 1) + q] : 0;
      const int len = rg.seg[kNR * (segbase + sg) + q] - e0;
      if (len > 0 || i == 0) {
        const int id = atomicAdd(rg.ctl + kStreamBuckets + 1, 1);
        recs[2 * id] = make_uint4(((uint32_t)tile << 16) | ((uint32_t)sg << 3) | (uint32_t)q,
                                  (uint32_t)start, (uint32_t)n, (uint32_t)e0);
        recs[2 * id + 1] = make_uint4((uint32_t)len, 0u, 0u, 0u);
        const int b = tsr_stream_bucket(len);
        const int at = atomicAdd(rg.ctl + b, 1);
        rg.units[b * cap + at] = (uint32_t)id;
      }
    }
  }


  // a pixel that never terminated considered the whole list (skipped
  // entries included); a terminated one stopped at its death position
  if (s.alive0()) s.ncons0 = n;
  if (s.alive1()) s.ncons1 = n;
  if (in0) {
    const long long pix = (long long)y0 * width + x;
    out_color[3 * pix] = fmaf(s.T.x, bg_r, s.Cr.x);
    out_color[3 * pix + 1] = fmaf(s.T.x, bg_g, s.Cg.x);
    out_color[3 * pix + 2] = fmaf(s.T.x, bg_b, s.Cb.x);
    out_depth[pix] = s.D.x;
    out_T[pix] = s.T.x;
    out_ncontrib[pix] = s.nc0;
    out_ncons[pix] = s.ncons0;
  }
  if (in1) {
    const long long pix = (long long)y1 * width + x;
    out_color[3 * pix] = fmaf(s.T.y, bg_r, s.Cr.y);
    out_color[3 * pix + 1] = fmaf(s.T.y, bg_g, s.Cg.y);
    out_color[3 * pix + 2] = fmaf(s.T.y, bg_b, s.Cb.y);
    out_depth[pix] = s.D.y;
    out_T[pix] = s.T.y;
    out_ncontrib[pix] = s.nc1;
    out_ncons[pix] = s.ncons1;
  }
}

// (Opt-in, TSR_K3_HW=1; measured slower: 301 vs 237 us at C2 -- 94 registers
// and 64-thread CTAs leave 20 warps per SM against 36, and the halves' hit
// counts differ.)  K3 for the training step's region mode with two 8x8
// blocks per warp: the
// CTA is 2 warps per tile, each warp half (16 lanes) owns one 8x8 block =
// one K4r region, 4 pixels per lane (column 8 bx + (l & 7), rows ry, ry + 2,
// ry + 4, ry + 6 with ry = 8 by + (l >> 3), as two vertical pairs).  The two
// halves walk their own blocks' hits in the same loop trip (a half whose
// block has no hit left idles), so one trip blends one splat into each of
// two blocks and the per-hit loop overhead is shared by 128 pixels.  Same
// arithmetic per pixel as render_fwd_kernel<3, 0>: outputs, checkpoint
// records, region lists (position, row), segment counts and K4r streams are
// identical.
constexpr int kHwThreads = 64;
__global__ void __launch_bounds__(kHwThreads) render_fwd_hw_kernel(
    const float4* __restrict__ rec, const int32_t* __restrict__ values,
    const int64_t* __restrict__ offsets, int width, int height, int tiles_x, float bg_r,
    float bg_g, float bg_b, float* __restrict__ out_color, float* __restrict__ out_depth,
    float* __restrict__ out_T, int32_t* __restrict__ out_ncontrib,
    int32_t* __restrict__ out_ncons, float* __restrict__ ckpt,
    const int64_t* __restrict__ ckpt_base, const int32_t* __restrict__ order, RegionArgs rg) {
  constexpr int kNR = 4;
  __shared__ float4 s_spl[kBatch][3];
  __shared__ float4 s_raw[kBatch];
  __shared__ int s_row[kBatch];
  const int tile = (order && order[gridDim.x]) ? order[blockIdx.x] : (int)blockIdx.x;
  const int tyi = tile / tiles_x, txi = tile - tyi * tiles_x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int hh = lane >> 4, l = lane & 15;
  const int bx = hh, by = warp, reg = 2 * by + bx;
  const int lx = 8 * bx + (l & 7), ry = 8 * by + (l >> 3);
  const int x = txi * kTile + lx;
  const int ya0 = tyi * kTile + ry, ya1 = ya0 + 4, yb0 = ya0 + 2, yb1 = ya0 + 6;
  const bool ina0 = x < width && ya0 < height, ina1 = x < width && ya1 < height;
  const bool inb0 = x < width && yb0 < height, inb1 = x < width && yb1 < height;
  const float pxf = (float)x + 0.5f;
  const float2 pya = make_float2((float)ya0 + 0.5f, (float)ya1 + 0.5f);
  const float2 pyb = make_float2((float)yb0 + 0.5f, (float)yb1 + 0.5f);
  const float sx0 = (float)(txi * kTile + 8 * bx) + 0.5f, sy0 = (float)(tyi * kTile + 8 * by) + 0.5f;
  const long long start = offsets[tile], end = offsets[tile + 1];
  const int n = (int)(end - start);
  float* ck0 = ckpt + ckpt_base[tile] * (5 * kTilePixels) + ry * kTile + lx;

  PixPair sa, sb;
  sa.T = make_float2(ina0 ? 1.f : 0.f, ina1 ? 1.f : 0.f);
  sb.T = make_float2(inb0 ? 1.f : 0.f, inb1 ? 1.f : 0.f);
  sa.Cr = sa.Cg = sa.Cb = sa.D = bc2(0.f);
  sb.Cr = sb.Cg = sb.Cb = sb.D = bc2(0.f);
  sa.nc0 = sa.nc1 = sb.nc0 = sb.nc1 = 0;
  sa.ncons0 = sa.ncons1 = sb.ncons0 = sb.ncons1 = 0;
  const unsigned half_bits = 0xffffu << (16 * hh);
  uint2* rl = reinterpret_cast<uint2*>(rg.list) + kNR * start + (long long)reg * n;
  int r_count = 0, s_next = 1;
  const long long segbase = (start >> kSegShift) + tile;
  // rows of the half's block held by the four pixel slots: ry - 8 by + {0, 4, 2, 6}
  const int r0 = l >> 3;

  for (int b0 = 0; b0 < n; b0 += kBatch) {
    if (!__syncthreads_or(sa.alive0() || sa.alive1() || sb.alive0() || sb.alive1())) break;
#pragma unroll
    for (int h = 0; h < kBatch / kHwThreads; ++h) {
      const int i = tid + h * kHwThreads;
      const int k = b0 + i;
      if (k < n) {
        const int row = values[start + k];
        const float4 q0 = __ldg(rec + 3 * row), q1 = __ldg(rec + 3 * row + 1),
                     q2 = __ldg(rec + 3 * row + 2);
        s_spl[i][0] = make_float4(q0.x, q0.y, q1.y, q1.z);
        s_spl[i][1] = make_float4(__fmul_rn(q0.z, kQScale), __fmul_rn(q0.w, 2.0f * kQScale),
                                  __fmul_rn(q1.x, kQScale), 0.f);
        s_spl[i][2] = make_float4(q2.x, q2.y, q2.z, q1.z);
        s_raw[i] = make_float4(q0.z, q0.w, q1.x, q1.w);
        s_row[i] = row;
      }
    }
    __syncthreads();
    const int cnt = min(kBatch, n - b0);
    for (int c0 = 0; c0 < cnt; c0 += kGroup) {
      const unsigned la0 = __ballot_sync(0xffffffffu, sa.alive0()),
                     la1 = __ballot_sync(0xffffffffu, sa.alive1()),
                     lb0 = __ballot_sync(0xffffffffu, sb.alive0()),
                     lb1 = __ballot_sync(0xffffffffu, sb.alive1());
      if (!(la0 | la1 | lb0 | lb1)) break;  // warp-level early exit (both blocks dead)
      // this half's live rectangle: lane l holds column l & 7 and rows
      // r0 + {0, 4, 2, 6} of the block (r0 = l >> 3)
      const unsigned ma0 = (la0 >> (16 * hh)) & 0xffffu, ma1 = (la1 >> (16 * hh)) & 0xffffu,
                     mb0 = (lb0 >> (16 * hh)) & 0xffffu, mb1 = (lb1 >> (16 * hh)) & 0xffffu;
      const unsigned mm = ma0 | ma1 | mb0 | mb1;
      const unsigned cols = (mm | (mm >> 8)) & 0xffu;
      auto rows2 = [](unsigned m, int off) {  // rows off (lanes 0-7) and off + 1 (lanes 8-15)
        return (((m & 0xffu) != 0u) ? (1u << off) : 0u) | (((m & 0xff00u) != 0u) ? (2u << off) : 0u);
      };
      const unsigned rows = rows2(ma0, 0) | rows2(ma1, 4) | rows2(mb0, 2) | rows2(mb1, 6);
      const float bx0 = sx0 + (float)(__ffs(cols) - 1), bx1 = sx0 + (float)(31 - __clz(cols));
      const float by0 = sy0 + (float)(__ffs(rows) - 1), by1 = sy0 + (float)(31 - __clz(rows));
      const int cend = min(kGroup, cnt - c0);
      const int pos0 = b0 + c0;
      if (pos0 > 0 && (pos0 & (kSeg - 1)) == 0) {  // segment boundary
        if (l == 0) rg.seg[kNR * (segbase + s_next - 1) + reg] = r_count;
        ++s_next;
      }
      // lane l tests splats c0 + l and c0 + 16 + l against this half's block
      bool h1 = false, h2 = false;
      if (mm) {
        if (l < cend) {
          const float4 g = s_spl[c0 + l][0], rw = s_raw[c0 + l];
          h1 = strip_hit(g.x, g.y, rw.x, rw.y, rw.z, rw.w, bx0, bx1, by0, by1);
        }
        if (l + 16 < cend) {
          const float4 g = s_spl[c0 + 16 + l][0], rw = s_raw[c0 + 16 + l];
          h2 = strip_hit(g.x, g.y, rw.x, rw.y, rw.z, rw.w, bx0, bx1, by0, by1);
        }
      }
      const unsigned q1 = __ballot_sync(0xffffffffu, h1), q2 = __ballot_sync(0xffffffffu, h2);
      const unsigned hm = ((q1 >> (16 * hh)) & 0xffffu) | (((q2 >> (16 * hh)) & 0xffffu) << 16);
      unsigned rev = __brev(hm);
      unsigned pa0 = 0u, pa1 = 0u, pb0 = 0u, pb1 = 0u;  // participation bits (bit-reversed)
      const bool lca0 = sa.alive0(), lca1 = sa.alive1(), lcb0 = sb.alive0(), lcb1 = sb.alive1();
      while (__any_sync(0xffffffffu, rev != 0u)) {
        if (rev) {
          const int f = 31 - __clz(rev);
          const unsigned bit = 1u << f;
          const int j = 31 - f;
          rev ^= bit;
          const float4* sp = s_spl[c0 + j];
          const float4 g0 = sp[0], g1 = sp[1], g2 = sp[2];
          blend_pair(g0, g1, g2, pxf, pya, pos0 + j, sa);
          if (sa.part0) pa0 |= bit;
          if (sa.part1) pa1 |= bit;
          blend_pair(g0, g1, g2, pxf, pyb, pos0 + j, sb);
          if (sb.part0) pb0 |= bit;
          if (sb.part1) pb1 |= bit;
        }
      }
      sa.nc0 += __popc(pa0);
      sa.nc1 += __popc(pa1);
      sb.nc0 += __popc(pb0);
      sb.nc1 += __popc(pb1);
      if (lca0 && !sa.alive0()) sa.ncons0 = pos0 + 33 - __ffs(pa0);
      if (lca1 && !sa.alive1()) sa.ncons1 = pos0 + 33 - __ffs(pa1);
      if (lcb0 && !sb.alive0()) sb.ncons0 = pos0 + 33 - __ffs(pb0);
      if (lcb1 && !sb.alive1()) sb.ncons1 = pos0 + 33 - __ffs(pb1);
      // region list entries of this half's block: the OR over its 16 lanes
      const unsigned pr = pa0 | pa1 | pb0 | pb1;
      const unsigned or_lo = __reduce_or_sync(0xffffffffu, hh == 0 ? pr : 0u);
      const unsigned or_hi = __reduce_or_sync(0xffffffffu, hh == 1 ? pr : 0u);
      const unsigned pm = __brev(hh ? or_hi : or_lo);
      const unsigned lt_l = (1u << l) - 1u;
      if ((pm >> l) & 1u)
        rl[r_count + __popc(pm & lt_l)] = make_uint2((uint32_t)(pos0 + l), (uint32_t)s_row[c0 + l]);
      if ((pm >> (l + 16)) & 1u)
        rl[r_count + __popc(pm & ((1u << (l + 16)) - 1u))] =
            make_uint2((uint32_t)(pos0 + 16 + l), (uint32_t)s_row[c0 + 16 + l]);
      r_count += __popc(pm);
      if (cend == kGroup && ((pos0 + kGroup) & (kSeg - 1)) == 0) {
        // segment-start record: the state after position pos0 + 31 of every
        // pixel that consumed it (still alive, or died there)
        float* dst = ck0 + (long long)(pos0 >> 5) * (5 * kTilePixels);
        auto put = [&](float* d, float T, float Cr, float Cg, float Cb, float D) {
          d[0] = T;
          d[kTilePixels] = Cr;
          d[2 * kTilePixels] = Cg;
          d[3 * kTilePixels] = Cb;
          d[4 * kTilePixels] = D;
        };
        if (sa.alive0() || sa.ncons0 == pos0 + kGroup) put(dst, sa.T.x, sa.Cr.x, sa.Cg.x, sa.Cb.x, sa.D.x);
        if (sa.alive1() || sa.ncons1 == pos0 + kGroup)
          put(dst + 4 * kTile, sa.T.y, sa.Cr.y, sa.Cg.y, sa.Cb.y, sa.D.y);
        if (sb.alive0() || sb.ncons0 == pos0 + kGroup)
          put(dst + 2 * kTile, sb.T.x, sb.Cr.x, sb.Cg.x, sb.Cb.x, sb.D.x);
        if (sb.alive1() || sb.ncons1 == pos0 + kGroup)
          put(dst + 6 * kTile, sb.T.y, sb.Cr.y, sb.Cg.y, sb.Cb.y, sb.D.y);
      }
    }
  }
  if (l == 0)  // the remaining segment ends (after an early exit)
    for (const int nseg = (n + kSeg - 1) >> kSegShift; s_next <= nseg; ++s_next)
      rg.seg[kNR * (segbase + s_next - 1) + reg] = r_count;
  {
    // the tile's K4r streams (as render_fwd_kernel)
    __syncthreads();
    const int nseg = (n + kSeg - 1) >> kSegShift;
    const long long cap = tsr_stream_bucket_cap(offsets[gridDim.x], gridDim.x);
    uint4* recs = reinterpret_cast<uint4*>(rg.units + (long long)kStreamBuckets * cap);
    for (int i = tid; i < nseg * kNR; i += kHwThreads) {
      const int sg = i / kNR, q = i - sg * kNR;
      const int e0 = sg > 0 ? rg.seg[kNR * (segbase + sg - 1) + q] : 0;
      const int len = rg.seg[kNR * (segbase + sg) + q] - e0;
      if (len > 0 || i == 0) {
        const int id = atomicAdd(rg.ctl + kStreamBuckets + 1, 1);
        recs[2 * id] = make_uint4(((uint32_t)tile << 16) | ((uint32_t)sg << 3) | (uint32_t)q,
                                  (uint32_t)start, (uint32_t)n, (uint32_t)e0);
        recs[2 * id + 1] = make_uint4((uint32_t)len, 0u, 0u, 0u);
        const int b = tsr_stream_bucket(len);
        const int at = atomicAdd(rg.ctl + b, 1);
        rg.units[b * cap + at] = (uint32_t)id;
      }
    }
  }
  auto out = [&](bool in, int y, float T, float Cr, float Cg, float Cb, float D, int ncb, int ncs) {
    if (!in) return;
    const long long pix = (long long)y * width + x;
    out_color[3 * pix] = fmaf(T, bg_r, Cr);
    out_color[3 * pix + 1] = fmaf(T, bg_g, Cg);
    out_color[3 * pix + 2] = fmaf(T, bg_b, Cb);
    out_depth[pix] = D;
    out_T[pix] = T;
    out_ncontrib[pix] = ncb;
    out_ncons[pix] = ncs;
  };
  out(ina0, ya0, sa.T.x, sa.Cr.x, sa.Cg.x, sa.Cb.x, sa.D.x, sa.nc0, sa.alive0() ? n : sa.ncons0);
  out(ina1, ya1, sa.T.y, sa.Cr.y, sa.Cg.y, sa.Cb.y, sa.D.y, sa.nc1, sa.alive1() ? n : sa.ncons1);
  out(inb0, yb0, sb.T.x, sb.Cr.x, sb.Cg.x, sb.Cb.x, sb.D.x, sb.nc0, sb.alive0() ? n : sb.ncons0);
  out(inb1, yb1, sb.T.y, sb.Cr.y, sb.Cg.y, sb.Cb.y, sb.D.y, sb.nc1, sb.alive1() ? n : sb.ncons1);
  (void)r0;
  (void)half_bits;
}

// Launch order of the per-tile kernels (K3, K4): the heavy tiles (list longer
// than 4x the mean) first, in raster order, then the others in raster order.
// order has n_tiles + 1 entries; order[n_tiles] = 0 when there is no heavy
// tile (raster order: the kernel then writes nothing else).
// Raster order keeps neighbouring tiles -- which share splats -- close in
// time (L2 reuse of the splat records); a heavy tile launched in the middle
// of the frame would finish last and set the tail (the low-opacity cluster
// of C3-lo: thousands of blends per pixel).  One CTA.
#ifndef TSR_ORDER_HEAVY_X2
#define TSR_ORDER_HEAVY_X2 8  // heavy: a list longer than (this / 2) x the mean tile list
#endif
constexpr int kOrderThreads = 1024;
constexpr int kOrderMaxTiles = 11264;  // 44 KB of list lengths in shared memory
__global__ void __launch_bounds__(kOrderThreads) tile_order_kernel(const int64_t* __restrict__ offsets,
                                                                   int n_tiles,
                                                                   int32_t* __restrict__ order) {
  __shared__ int s_len[kOrderMaxTiles];
  __shared__ int s_w[kOrderThreads / 32];
  __shared__ int s_tot;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const bool staged = n_tiles <= kOrderMaxTiles;
  // coalesced: every load of a thread in flight at once
  if (staged) {
    for (int t = tid; t < n_tiles; t += kOrderThreads)
      s_len[t] = (int)(offsets[t + 1] - offsets[t]);
  }
  const long long P = offsets[n_tiles] - offsets[0];
  const long long thr = max(TSR_ORDER_HEAVY_X2 * P / (2 * max(n_tiles, 1)), 64ll);
  __syncthreads();
  auto len = [&](int t) -> long long {
    return staged ? (long long)s_len[t] : offsets[t + 1] - offsets[t];
  };
  const int per = (n_tiles + kOrderThreads - 1) / kOrderThreads;
  const int t0 = tid * per, t1 = min(n_tiles, t0 + per);
  int heavy = 0;
  for (int t = t0; t < t1; ++t) heavy += len(t) > thr;
  int incl = heavy;
#pragma unroll
  for (int k = 1; k < 32; k <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, incl, k);
    if (lane >= k) incl += v;
  }
  if (lane == 31) s_w[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    const int w = s_w[lane];
    int wi = w;
#pragma unroll
    for (int k = 1; k < 32; k <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, wi, k);
      if (lane >= k) wi += v;
    }
    s_w[lane] = wi - w;
    if (lane == 31) s_tot = wi;
  }
  __syncthreads();
  if (s_tot == 0) {  // no heavy tile: raster order (order[n_tiles] = 0 says so)
    if (tid == 0) order[n_tiles] = 0;
    return;
  }
  if (tid == 0) order[n_tiles] = 1;
  int h = s_w[warp] + incl - heavy;  // heavy tiles before this thread's range
  int l = s_tot + (t0 - h);          // light tiles before it, after all heavy ones
  for (int t = t0; t < t1; ++t) {
    if (len(t) > thr) order[h++] = t;
    else order[l++] = t;
  }
}

}  // namespace tsr

using namespace tsr;

extern "C" int tsr_tile_order(const int64_t* offsets, int32_t n_tiles, int32_t* order,
                              void* stream) {
  if (!offsets || !order || n_tiles <= 0) return TSR_E_INVALID;
  tile_order_kernel<<<1, kOrderThreads, 0, (cudaStream_t)stream>>>(offsets, n_tiles, order);
  TSR_CHECK_LAUNCH();
  return TSR_OK;
}

extern "C" int tsr_render_fwd_ordered(const float* rec, const int32_t* values,
                                      const int64_t* offsets, int32_t width, int32_t height,
                                      const float* background_host, float* out_color,
                                      float* out_depth, float* out_final_T,
                                      int32_t* out_n_contrib, int32_t* out_n_considered,
                                      float* ckpt, const int64_t* ckpt_base, int32_t ckpt_stride,
                                      const int32_t* tile_order, void* stream) {
  if (width <= 0 || height <= 0 || !background_host) return TSR_E_INVALID;
  if (ckpt && !ckpt_base) return TSR_E_INVALID;
  if (ckpt && ckpt_stride != 1 && ckpt_stride != 2) return TSR_E_INVALID;
  const int tx = tiles_of(width), ty = tiles_of(height);
  const int n_tiles = tx * ty;
  cudaStream_t s = (cudaStream_t)stream;
  const ScoreArgs none{};
  auto* k = !ckpt ? render_fwd_kernel<0, 0>
            : ckpt_stride == 2 ? render_fwd_kernel<2, 0> : render_fwd_kernel<1, 0>;
  k<<<n_tiles, kFwdThreads, 0, s>>>((const float4*)rec, values, offsets, width, height, tx,
                                    background_host[0], background_host[1], background_host[2],
                                    out_color, out_depth, out_final_T, out_n_contrib,
                                    out_n_considered, ckpt, ckpt_base, none, tile_order, RegionArgs{});
  TSR_CHECK_LAUNCH();
  return TSR_OK;
}

// K3 for the region-culled backward: checkpoint records at segment starts
// only, plus the per-(tile, 8x8 region) lists of list positions that pass the
// region's block test (RegionArgs above).  region_list holds 4 x P entries,
// region_seg 4 x (P / kSeg + n_tiles + 1).
extern "C" int tsr_render_fwd_regions(const float* rec, const int32_t* values,
                                      const int64_t* offsets, int32_t width, int32_t height,
                                      const float* background_host, float* out_color,
                                      float* out_depth, float* out_final_T,
                                      int32_t* out_n_contrib, int32_t* out_n_considered,
                                      float* ckpt, const int64_t* ckpt_base,
                                      uint32_t* region_list, int32_t* region_seg,
                                      uint32_t* region_units, int32_t* region_ctl,
                                      int32_t region_height, const int32_t* tile_order,
                                      void* stream) {
  if (width <= 0 || height <= 0 || !background_host || !ckpt || !ckpt_base || !region_list ||
      !region_seg || !region_units || !region_ctl || (region_height != 8 && region_height != 4))
    return TSR_E_INVALID;
  const int tx = tiles_of(width), ty = tiles_of(height);
  const int n_tiles = tx * ty;
  cudaStream_t s = (cudaStream_t)stream;
  const ScoreArgs none{};
  if (cudaMemsetAsync(region_ctl, 0, kUnitCtl * sizeof(int32_t), s) != cudaSuccess) return TSR_E_CUDA;
  // the two-blocks-per-warp form is opt-in (TSR_K3_HW=1): measured 301 vs 237 us
  static const bool hw = getenv("TSR_K3_HW") && atoi(getenv("TSR_K3_HW")) == 1;
  if (region_height == 8 && hw) {
    render_fwd_hw_kernel<<<n_tiles, kHwThreads, 0, s>>>(
        (const float4*)rec, values, offsets, width, height, tx, background_host[0],
        background_host[1], background_host[2], out_color, out_depth, out_final_T, out_n_contrib,
        out_n_considered, ckpt, ckpt_base, tile_order,
        RegionArgs{region_list, region_seg, region_units, region_ctl});
    TSR_CHECK_LAUNCH();
    return TSR_OK;
  }
  auto* k = region_height == 8 ? render_fwd_kernel<3, 0> : render_fwd_kernel<4, 0>;
  k<<<n_tiles, kFwdThreads, 0, s>>>(
      (const float4*)rec, values, offsets, width, height, tx, background_host[0],
      background_host[1], background_host[2], out_color, out_depth, out_final_T, out_n_contrib,
      out_n_considered, ckpt, ckpt_base, none, tile_order,
      RegionArgs{region_list, region_seg, region_units, region_ctl});
  TSR_CHECK_LAUNCH();
  return TSR_OK;
}

extern "C" int tsr_render_fwd_ex(const float* rec, const int32_t* values, const int64_t* offsets,
                                  int32_t width, int32_t height, const float* background_host,
                                  float* out_color, float* out_depth, float* out_final_T,
                                  int32_t* out_n_contrib, int32_t* out_n_considered, float* ckpt,
                                  const int64_t* ckpt_base, int32_t ckpt_stride, void* stream) {
  if (width <= 0 || height <= 0 || !background_host) return TSR_E_INVALID;
  if (ckpt && !ckpt_base) return TSR_E_INVALID;
  if (ckpt && ckpt_stride != 1 && ckpt_stride != 2) return TSR_E_INVALID;
  const int tx = tiles_of(width), ty = tiles_of(height);
  const int n_tiles = tx * ty;
  cudaStream_t s = (cudaStream_t)stream;
  const ScoreArgs none{};
  auto* k = !ckpt ? render_fwd_kernel<0, 0>
            : ckpt_stride == 2 ? render_fwd_kernel<2, 0> : render_fwd_kernel<1, 0>;
  k<<<n_tiles, kFwdThreads, 0, s>>>((const float4*)rec, values, offsets, width, height, tx,
                                    background_host[0], background_host[1], background_host[2],
                                    out_color, out_depth, out_final_T, out_n_contrib,
                                    out_n_considered, ckpt, ckpt_base, none, nullptr, RegionArgs{});
  TSR_CHECK_LAUNCH();
  return TSR_OK;
}

extern "C" int tsr_render_fwd(const float* rec, const int32_t* values, const int64_t* offsets,
                              int32_t width, int32_t height, const float* background_host,
                              float* out_color, float* out_depth, float* out_final_T,
                              int32_t* out_n_contrib, int32_t* out_n_considered, float* ckpt,
                              const int64_t* ckpt_base, void* stream) {
  return tsr_render_fwd_ex(rec, values, offsets, width, height, background_host, out_color,
                           out_depth, out_final_T, out_n_contrib, out_n_considered, ckpt,
                           ckpt_base, 1, stream);
}

extern "C" int tsr_render_score(const float* rec, const int32_t* values, const int64_t* offsets,
                                int32_t width, int32_t height, const float* background_host,
                                int32_t mode, const uint8_t* mask, float weight,
                                float* row_score, int64_t* warp_counts,
                                const int64_t* warp_base, int64_t* out_pixel, int64_t* out_row,
                                float* out_color, float* out_depth, float* out_final_T,
                                int32_t* out_n_contrib, int32_t* out_n_considered,
                                void* stream) {
  if (width <= 0 || height <= 0 || !background_host) return TSR_E_INVALID;
  if (mode == 1 && !warp_counts) return TSR_E_INVALID;
  if (mode == 2 && (!warp_base || !out_pixel || !out_row)) return TSR_E_INVALID;
  if (mode == 3 && (!mask || !row_score)) return TSR_E_INVALID;
  if (mode < 1 || mode > 3) return TSR_E_INVALID;
  const int tx = tiles_of(width), ty = tiles_of(height);
  const int n_tiles = tx * ty;
  cudaStream_t s = (cudaStream_t)stream;
  ScoreArgs sc{mask, weight, row_score, (long long*)warp_counts, (const long long*)warp_base,
               (long long*)out_pixel, (long long*)out_row};
  auto* k = mode == 1 ? render_fwd_kernel<0, 1>
            : mode == 2 ? render_fwd_kernel<0, 2> : render_fwd_kernel<0, 3>;
  k<<<n_tiles, kFwdThreads, 0, s>>>((const float4*)rec, values, offsets, width, height, tx,
                                    background_host[0], background_host[1], background_host[2],
                                    out_color, out_depth, out_final_T, out_n_contrib,
                                    out_n_considered, nullptr, nullptr, sc, nullptr, RegionArgs{});
  TSR_CHECK_LAUNCH();
  return TSR_OK;
}
