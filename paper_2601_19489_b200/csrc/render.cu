// K3: forward rasterizer (render, forward.py:87-161).
//
// One CTA per 16x16 tile, one thread per pixel.  The tile's depth-sorted list
// is consumed in batches of 256 splats staged in shared memory (3 x float4
// per splat: mean/opacity, prescaled conic/depth, colour).  Per pixel:
//   alpha = min(0.99, o exp(-q/2)); blend iff alive && alpha >= 1/255;
//   C += T alpha c; D += T alpha d; T *= 1 - alpha; n_considered = k+1 while
//   alive; alive &= T >= 1e-4 AFTER blending (forward.py:125-138).
// Termination: a warp stops scanning a batch once its 32 pixels are dead
// (warp-level early exit) and the CTA stops at the next batch boundary once
// all 256 are dead (forward.py:141-145).
// Culling: a warp owns a 16x2 pixel strip.  For each chunk of 32 staged
// splats every lane tests one splat against the strip with the exact minimum
// of its quadratic over the strip's pixel-centre rectangle (min_q_box,
// binning.py:241-259, in FP32 with a safety margin); only splats that can
// reach alpha >= 1/255 somewhere in the strip are evaluated.  A skipped splat
// provably leaves T, C, D unchanged, so the outputs are identical;
// n_considered is restored from the termination position.
// Checkpoints (forward.py:139-140): after every 32nd list position the state
// (T, C, D) is stored for each pixel that consumed that position -- exactly
// the records the per-Gaussian backward reads (it enters group g of a pixel
// only when n_considered > 32 g).  Padding records of dead pixels are never
// written (they are never read).
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
    const float bc = -b / c, ba = -b / a;
    const float yx0 = fminf(fmaxf(bc * rx0, ry0), ry1), yx1 = fminf(fmaxf(bc * rx1, ry0), ry1);
    const float xy0 = fminf(fmaxf(ba * ry0, rx0), rx1), xy1 = fminf(fmaxf(ba * ry1, rx0), rx1);
    qmin = fminf(fminf(q(rx0, yx0), q(rx1, yx1)), fminf(q(xy0, ry0), q(xy1, ry1)));
  }
  return qmin <= fmaf(t, 1.001f, 1e-3f);
}

// One list entry for one pixel, branch-free (predicated): the warp executes
// it in lockstep, so a per-lane branch would only add reconvergence cost.
__device__ __forceinline__ void blend_one(const float4 g, const float4 c, const float4 col,
                                          float pxf, float pyf, int pos, bool& alive, float& T,
                                          float& Cr, float& Cg, float& Cb, float& D,
                                          int& ncontrib, int& ncons) {
  AlphaEval e = eval_alpha(pxf, pyf, g.x, g.y, c.x, c.y, c.z, g.z);
  const bool blend = alive && (e.alpha >= kMinAlpha);
  const float w = blend ? T * e.alpha : 0.f;
  Cr = fmaf(w, col.x, Cr);
  Cg = fmaf(w, col.y, Cg);
  Cb = fmaf(w, col.z, Cb);
  D = fmaf(w, col.w, D);
  T = blend ? T * (1.f - e.alpha) : T;
  ncontrib += blend ? 1 : 0;
  ncons = alive ? pos + 1 : ncons;
  alive = alive && (T >= kTTerminate);
}

template <bool kCkpt>
__global__ void __launch_bounds__(256) render_fwd_kernel(
    const float4* __restrict__ rec, const int32_t* __restrict__ values,
    const int64_t* __restrict__ offsets, int width, int height, int tiles_x, float bg_r,
    float bg_g, float bg_b, float* __restrict__ out_color, float* __restrict__ out_depth,
    float* __restrict__ out_T, int32_t* __restrict__ out_ncontrib,
    int32_t* __restrict__ out_ncons, float* __restrict__ ckpt,
    const int64_t* __restrict__ ckpt_base) {
  __shared__ float4 s_geo[256];
  __shared__ float4 s_con[256];
  __shared__ float4 s_col[256];
  __shared__ float4 s_raw[256];   // a, b, c (unscaled), level t

  const int tile = blockIdx.x;
  const int tyi = tile / tiles_x, txi = tile - tyi * tiles_x;
  const int tid = threadIdx.x;
  const int lx = tid & 15, ly = tid >> 4;
  const int x = txi * kTile + lx, y = tyi * kTile + ly;
  const bool inside = x < width && y < height;
  const float pxf = (float)x + 0.5f, pyf = (float)y + 0.5f;
  const int lane = tid & 31;
  // this warp's strip of pixel centres (rows 2w, 2w+1 of the tile)
  const float sx0 = (float)(txi * kTile) + 0.5f, sy0 = (float)(tyi * kTile + 2 * (tid >> 5)) + 0.5f;
  const long long start = offsets[tile], end = offsets[tile + 1];
  const int n = (int)(end - start);
  float* ck = nullptr;
  if (kCkpt) ck = ckpt + ckpt_base[tile] * (5 * kTilePixels) + tid;

  float T = 1.f, Cr = 0.f, Cg = 0.f, Cb = 0.f, D = 0.f;
  int ncontrib = 0, ncons = 0;
  bool alive = inside;

  for (int b0 = 0; b0 < n; b0 += 256) {
    if (!__syncthreads_or(alive)) break;
    const int k = b0 + tid;
    if (k < n) {
      const int row = values[start + k];
      const float4 r0 = __ldg(rec + 3 * row), r1 = __ldg(rec + 3 * row + 1),
                   r2 = __ldg(rec + 3 * row + 2);
      s_geo[tid] = make_float4(r0.x, r0.y, r1.y, r1.z);
      s_con[tid] = make_float4(__fmul_rn(r0.z, kQScale), __fmul_rn(r0.w, kQScale),
                               __fmul_rn(r1.x, kQScale), 0.f);
      s_col[tid] = make_float4(r2.x, r2.y, r2.z, r1.z);
      s_raw[tid] = make_float4(r0.z, r0.w, r1.x, r1.w);
    }
    __syncthreads();
    const int cnt = min(256, n - b0);
    // chunks of 32 list positions == one checkpoint interval
    for (int c0 = 0; c0 < cnt; c0 += kGroup) {
      if (!__any_sync(0xffffffffu, alive)) break;  // warp-level early exit
      const int cend = min(kGroup, cnt - c0);
      const int pos0 = b0 + c0;
      // lane j tests splat c0 + j against this warp's 16x2 strip
      bool hit = false;
      if (lane < cend) {
        const float4 g = s_geo[c0 + lane], rw = s_raw[c0 + lane];
        hit = strip_hit(g.x, g.y, rw.x, rw.y, rw.z, rw.w, sx0, sx0 + 15.f, sy0, sy0 + 1.f);
      }
      unsigned mask = __ballot_sync(0xffffffffu, hit);
      while (mask) {
        const int j = __ffs(mask) - 1;
        mask &= mask - 1u;
        blend_one(s_geo[c0 + j], s_con[c0 + j], s_col[c0 + j], pxf, pyf, pos0 + j, alive, T, Cr,
                  Cg, Cb, D, ncontrib, ncons);
      }
      if (cend == kGroup) {
        // consumed position pos0+31 <=> still alive, or died exactly there
        if (kCkpt && (alive || ncons == pos0 + kGroup)) {
          // state after list position pos0+31 -> record (pos0+32)/32 - 1
          float* dst = ck + (long long)(pos0 >> 5) * (5 * kTilePixels);
          dst[0] = T;
          dst[kTilePixels] = Cr;
          dst[2 * kTilePixels] = Cg;
          dst[3 * kTilePixels] = Cb;
          dst[4 * kTilePixels] = D;
        }
      }
    }
  }
  // a pixel that never terminated considered the whole list (skipped
  // entries included); a terminated one stopped at its death position
  if (alive) ncons = n;
  if (inside) {
    const long long pix = (long long)y * width + x;
    out_color[3 * pix] = fmaf(T, bg_r, Cr);
    out_color[3 * pix + 1] = fmaf(T, bg_g, Cg);
    out_color[3 * pix + 2] = fmaf(T, bg_b, Cb);
    out_depth[pix] = D;
    out_T[pix] = T;
    out_ncontrib[pix] = ncontrib;
    out_ncons[pix] = ncons;
  }
}

}  // namespace tsr

using namespace tsr;

extern "C" int tsr_render_fwd(const float* rec, const int32_t* values, const int64_t* offsets,
                              int32_t width, int32_t height, const float* background_host,
                              float* out_color, float* out_depth, float* out_final_T,
                              int32_t* out_n_contrib, int32_t* out_n_considered, float* ckpt,
                              const int64_t* ckpt_base, void* stream) {
  if (width <= 0 || height <= 0 || !background_host) return TSR_E_INVALID;
  if (ckpt && !ckpt_base) return TSR_E_INVALID;
  const int tx = tiles_of(width), ty = tiles_of(height);
  const int n_tiles = tx * ty;
  cudaStream_t s = (cudaStream_t)stream;
  if (ckpt) {
    render_fwd_kernel<true><<<n_tiles, 256, 0, s>>>(
        (const float4*)rec, values, offsets, width, height, tx, background_host[0],
        background_host[1], background_host[2], out_color, out_depth, out_final_T,
        out_n_contrib, out_n_considered, ckpt, ckpt_base);
  } else {
    render_fwd_kernel<false><<<n_tiles, 256, 0, s>>>(
        (const float4*)rec, values, offsets, width, height, tx, background_host[0],
        background_host[1], background_host[2], out_color, out_depth, out_final_T,
        out_n_contrib, out_n_considered, nullptr, nullptr);
  }
  TSR_CHECK_LAUNCH();
  return TSR_OK;
}
