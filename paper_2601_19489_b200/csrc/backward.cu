// K4: per-Gaussian raster backward (backward_per_gaussian, backward.py:137-223).
//
// One CTA per tile, 8 warps.  The tile list is cut into groups of 32 list
// positions (CHECKPOINT_INTERVAL); a warp owns one group at a time, lane j
// owning list position 32g+j (Taming-GS style: per-Gaussian parallel, no
// per-pixel atomics).  The warp walks the tile's pixels; for each pixel it
// restarts from the forward checkpoint of the group and needs, per lane,
//   T_j      = T_ckpt * prod_{i<j, part_i} (1 - alpha_i)  -> warp exclusive product scan
//   K_after_j = K_ckpt + sum_{i<=j} w_i gc_i              -> warp inclusive sum scan
// where gc_i = <g_color, c_i> + g_depth d_i folds the colour and depth
// suffixes of backward.py:195-205 into ONE scalar per pixel, and
//   dL/dalpha_j = T_j gc_j - (Ktot + g_T T_f - K_after_j) / (1 - alpha_j)
// (the g_T channel is backward.py:170,204-205).  part = p < n_considered and
// alpha >= 1/255 (backward.py:189); capped alphas get zero conic/mean/opacity
// gradient (backward.py:64,72).  Gradients accumulate in registers over the
// tile's pixels and are merged once per (splat, tile) with atomics
// (backward.py:214-222).  The group loop is bounded by the tile's maximum
// n_considered: later groups contribute exactly zero.
#include <cuda_runtime.h>

#include "tsr_common.cuh"

namespace tsr {

constexpr int kBwdWarps = 8;

__global__ void __launch_bounds__(256) render_bwd_kernel(
    const float4* __restrict__ rec, const int32_t* __restrict__ values,
    const int64_t* __restrict__ offsets, int width, int height, int tiles_x,
    const float* __restrict__ color, const float* __restrict__ depth,
    const float* __restrict__ final_T, const int32_t* __restrict__ n_considered,
    const float* __restrict__ ckpt, const int64_t* __restrict__ ckpt_base,
    const float* __restrict__ grad_color, const float* __restrict__ grad_depth,
    const float* __restrict__ grad_final_T, float* __restrict__ grad2d,
    unsigned long long* __restrict__ merges) {
  __shared__ float4 s_g[kTilePixels];  // g_r, g_g, g_b, g_d
  __shared__ float s_k[kTilePixels];   // Ktot + g_T * T_final
  __shared__ int s_nc[kTilePixels];
  __shared__ float s_T0[kBwdWarps][kTilePixels];
  __shared__ float s_R0[kBwdWarps][kTilePixels];
  __shared__ int s_maxnc;

  const int tile = blockIdx.x;
  const long long start = offsets[tile], end = offsets[tile + 1];
  const int n = (int)(end - start);
  if (n == 0) return;
  const int tyi = tile / tiles_x, txi = tile - tyi * tiles_x;
  const int tid = threadIdx.x;
  {
    const int x = txi * kTile + (tid & 15), y = tyi * kTile + (tid >> 4);
    const bool inside = x < width && y < height;
    float gr = 0.f, gg = 0.f, gb = 0.f, gd = 0.f, gt = 0.f, k = 0.f;
    int nc = 0;
    if (inside) {
      const long long pix = (long long)y * width + x;
      gr = grad_color[3 * pix];
      gg = grad_color[3 * pix + 1];
      gb = grad_color[3 * pix + 2];
      if (grad_depth) gd = grad_depth[pix];
      if (grad_final_T) gt = grad_final_T[pix];
      nc = n_considered[pix];
      k = gr * color[3 * pix] + gg * color[3 * pix + 1] + gb * color[3 * pix + 2] +
          gd * depth[pix] + gt * final_T[pix];
    }
    const bool nz = (gr != 0.f) || (gg != 0.f) || (gb != 0.f) || (gd != 0.f) || (gt != 0.f);
    s_g[tid] = make_float4(gr, gg, gb, gd);
    s_k[tid] = k;
    s_nc[tid] = nc;
    if (tid == 0) s_maxnc = 0;
    // tile skipped when its upstream is all zero (backward.py:156-158)
    if (!__syncthreads_or(nz)) return;
    atomicMax(&s_maxnc, nc);
    if (tid == 0) atomicAdd(merges, (unsigned long long)n);
  }
  __syncthreads();
  const int n_groups = (s_maxnc + kGroup - 1) / kGroup;
  const int lane = tid & 31, warp = tid >> 5;
  const float mean_scale = -2.0f / kQScale;
  long long rbase = 0;
  if (ckpt_base) rbase = ckpt_base[tile];

  for (int g = warp; g < n_groups; g += kBwdWarps) {
    const int p0 = g * kGroup;
    const int p = p0 + lane;
    const bool valid = p < n;
    float mx = 0.f, my = 0.f, a = 0.f, b = 0.f, c = 0.f, o = 0.f, cr = 0.f, cg = 0.f,
          cb = 0.f, dep = 0.f;
    int row = 0;
    if (valid) {
      row = values[start + p];
      const float4 r0 = rec[3 * row], r1 = rec[3 * row + 1], r2 = rec[3 * row + 2];
      mx = r0.x; my = r0.y;
      a = __fmul_rn(r0.z, kQScale);
      b = __fmul_rn(r0.w, kQScale);
      c = __fmul_rn(r1.x, kQScale);
      o = r1.y; dep = r1.z;
      cr = r2.x; cg = r2.y; cb = r2.z;
    }
    // group prologue: checkpoint state per pixel -> (T0, R0 = s_k - K_ckpt)
    for (int px = lane; px < kTilePixels; px += 32) {
      if (s_nc[px] > p0) {
        float T0 = 1.f, K0 = 0.f;
        if (g > 0) {
          const float* src = ckpt + (rbase + g - 1) * (5 * kTilePixels) + px;
          const float4 gv = s_g[px];
          T0 = src[0];
          K0 = gv.x * src[kTilePixels] + gv.y * src[2 * kTilePixels] +
               gv.z * src[3 * kTilePixels] + gv.w * src[4 * kTilePixels];
        }
        s_T0[warp][px] = T0;
        s_R0[warp][px] = s_k[px] - K0;
      }
    }
    __syncwarp();

    float acc_mx = 0.f, acc_my = 0.f, acc_a = 0.f, acc_b = 0.f, acc_c = 0.f, acc_o = 0.f;
    float acc_r = 0.f, acc_g = 0.f, acc_bl = 0.f, acc_d = 0.f;
    bool touched = false;
    const float ox = (float)(txi * kTile) + 0.5f, oy = (float)(tyi * kTile) + 0.5f;
    for (int px = 0; px < kTilePixels; ++px) {
      const int nc = s_nc[px];
      if (nc <= p0) continue;  // pixel terminated before this group
      const float pxf = ox + (float)(px & 15), pyf = oy + (float)(px >> 4);
      AlphaEval e = eval_alpha(pxf, pyf, mx, my, a, b, c, o);
      const bool part = valid && (p < nc) && (e.alpha >= kMinAlpha);
      if (__ballot_sync(0xffffffffu, part) == 0u) continue;
      const float om = __fsub_rn(1.f, e.alpha);
      float pr = part ? om : 1.f;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const float t = __shfl_up_sync(0xffffffffu, pr, d);
        if (lane >= d) pr *= t;
      }
      float ex = __shfl_up_sync(0xffffffffu, pr, 1);
      if (lane == 0) ex = 1.f;
      const float4 gv = s_g[px];
      const float T = s_T0[warp][px] * ex;
      const float w = part ? T * e.alpha : 0.f;
      const float gcj = fmaf(gv.x, cr, fmaf(gv.y, cg, fmaf(gv.z, cb, gv.w * dep)));
      float sc = w * gcj;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const float t = __shfl_up_sync(0xffffffffu, sc, d);
        if (lane >= d) sc += t;
      }
      if (part) {
        touched = true;
        const float num = s_R0[warp][px] - sc;
        const float dLda = T * gcj - __fdividef(num, om);
        const bool capped = e.raw > e.alpha;
        const float gq = capped ? 0.f : -0.5f * e.alpha * dLda;
        acc_a = fmaf(gq * e.dx, e.dx, acc_a);
        acc_b = fmaf(gq * 2.f * e.dx, e.dy, acc_b);
        acc_c = fmaf(gq * e.dy, e.dy, acc_c);
        acc_mx = fmaf(gq, e.u, acc_mx);
        acc_my = fmaf(gq, e.v, acc_my);
        if (!capped) acc_o = fmaf(dLda, e.gauss, acc_o);
        acc_r = fmaf(w, gv.x, acc_r);
        acc_g = fmaf(w, gv.y, acc_g);
        acc_bl = fmaf(w, gv.z, acc_bl);
        acc_d = fmaf(w, gv.w, acc_d);
      }
    }
    __syncwarp();
    if (valid && touched) {
      float* dst = grad2d + (long long)row * TSR_GRAD2D_FLOATS;
      atomicAdd(dst + 0, acc_mx * mean_scale);
      atomicAdd(dst + 1, acc_my * mean_scale);
      atomicAdd(dst + 2, acc_a);
      atomicAdd(dst + 3, acc_b);
      atomicAdd(dst + 4, acc_c);
      atomicAdd(dst + 5, acc_o);
      atomicAdd(dst + 6, acc_r);
      atomicAdd(dst + 7, acc_g);
      atomicAdd(dst + 8, acc_bl);
      atomicAdd(dst + 9, acc_d);
    }
  }
}

}  // namespace tsr

using namespace tsr;

extern "C" int tsr_render_bwd(const float* rec, const int32_t* values, const int64_t* offsets,
                              int32_t width, int32_t height, const float* color,
                              const float* depth, const float* final_T,
                              const int32_t* n_considered, const float* ckpt,
                              const int64_t* ckpt_base, const float* grad_color,
                              const float* grad_depth, const float* grad_final_T,
                              float* grad2d, unsigned long long* merges, void* stream) {
  if (width <= 0 || height <= 0 || !grad_color || !merges) return TSR_E_INVALID;
  if (ckpt && !ckpt_base) return TSR_E_INVALID;
  const int tx = tiles_of(width), ty = tiles_of(height);
  render_bwd_kernel<<<tx * ty, 256, 0, (cudaStream_t)stream>>>(
      (const float4*)rec, values, offsets, width, height, tx, color, depth, final_T,
      n_considered, ckpt, ckpt_base, grad_color, grad_depth, grad_final_T, grad2d, merges);
  TSR_CHECK_LAUNCH();
  return TSR_OK;
}
