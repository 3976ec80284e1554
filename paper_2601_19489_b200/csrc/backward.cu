// K4: per-Gaussian raster backward (backward_per_gaussian, backward.py:137-223).
//
// One CTA per tile, 8 warps.  The tile list is cut into groups of 32 list
// positions (CHECKPOINT_INTERVAL); a warp owns one group at a time, lane j
// owning list position 32g+j (Taming-GS style: per-Gaussian parallel, no
// per-pixel atomics).  For a pixel, lane j needs
//   T_j = T_ckpt * prod_{i<j, part_i} (1 - alpha_i)       and
//   R_j = Ktot + g_T T_f - K_ckpt - sum_{i<=j} w_i gc_i
// where gc_i = <g_color, c_i> + g_depth d_i folds the colour and depth
// suffixes of backward.py:195-205 into ONE scalar per pixel, giving
//   dL/dalpha_j = T_j gc_j - R_j / (1 - alpha_j)
// (the g_T channel is backward.py:170,204-205).  Both are computed by a
// SYSTOLIC pipeline: the group's active pixels (n_considered > 32g) are
// compacted into a list; at step t lane j works on list entry t-j and takes
// (T, R) from lane j-1, which finished the same pixel one step earlier -- one
// shuffle per quantity per step instead of a log-depth warp scan.
// part = p < n_considered and alpha >= 1/255 (backward.py:189); capped alphas
// get zero conic/mean/opacity gradient (backward.py:64,72).  Gradients
// accumulate in registers and are merged once per (splat, tile) with atomics
// (backward.py:214-222).  The group loop is bounded by the tile's maximum
// n_considered: later groups contribute exactly zero.
#include <cuda_runtime.h>

#include "tsr_common.cuh"

namespace tsr {

constexpr int kBwdWarps = 4;
constexpr int kBwdThreads = 32 * kBwdWarps;

__device__ __forceinline__ float fast_rcp(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// per-pixel record (index kTilePixels is a dummy pixel with n_considered 0,
// used as the sentinel of the padded systolic lists)
constexpr int kPixSlots = kTilePixels + 1;
constexpr int kListPad = 32;

__global__ void __launch_bounds__(kBwdThreads) render_bwd_kernel(
    const float4* __restrict__ rec, const int32_t* __restrict__ values,
    const int64_t* __restrict__ offsets, int width, int height, int tiles_x,
    const float* __restrict__ color, const float* __restrict__ depth,
    const float* __restrict__ final_T, const int32_t* __restrict__ n_considered,
    const float* __restrict__ ckpt, const int64_t* __restrict__ ckpt_base,
    const float* __restrict__ grad_color, const float* __restrict__ grad_depth,
    const float* __restrict__ grad_final_T, float* __restrict__ grad2d,
    unsigned long long* __restrict__ merges) {
  __shared__ float4 s_pa[kPixSlots];  // pixel centre x, y, g_depth, n_considered (int bits)
  __shared__ float4 s_pb[kPixSlots];  // g_r, g_g, g_b, Ktot + g_T T_final
  __shared__ unsigned short s_list[kBwdWarps][kTilePixels + 2 * kListPad];
  __shared__ float2 s_tr[kBwdWarps][kTilePixels + kListPad];  // (T_ckpt, R_ckpt)
  __shared__ int s_maxnc;
  __shared__ int s_next_group;

  const int tile = blockIdx.x;
  const long long start = offsets[tile], end = offsets[tile + 1];
  const int n = (int)(end - start);
  if (n == 0) return;
  const int tyi = tile / tiles_x, txi = tile - tyi * tiles_x;
  const int tid = threadIdx.x;
  if (tid == 0) {
    s_maxnc = 0;
    s_next_group = kBwdWarps;  // groups 0..kBwdWarps-1 are taken statically
    s_pa[kTilePixels] = make_float4(-65536.f, -65536.f, 0.f, __int_as_float(0));  // finite: gauss -> 0
    s_pb[kTilePixels] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
  bool nz = false;
  int my_max = 0;
  for (int px = tid; px < kTilePixels; px += kBwdThreads) {
    const int x = txi * kTile + (px & 15), y = tyi * kTile + (px >> 4);
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
    nz |= (gr != 0.f) || (gg != 0.f) || (gb != 0.f) || (gd != 0.f) || (gt != 0.f);
    my_max = max(my_max, nc);
    s_pa[px] = make_float4((float)x + 0.5f, (float)y + 0.5f, gd, __int_as_float(nc));
    s_pb[px] = make_float4(gr, gg, gb, k);
  }
  // tile skipped when its upstream is all zero (backward.py:156-158)
  if (!__syncthreads_or(nz)) return;
  atomicMax(&s_maxnc, my_max);
  if (tid == 0) atomicAdd(merges, (unsigned long long)n);
  __syncthreads();
  const int n_groups = (s_maxnc + kGroup - 1) / kGroup;
  const int lane = tid & 31, warp = tid >> 5;
  const unsigned lt_mask = (1u << lane) - 1u;
  const float mean_scale = -2.0f / kQScale;
  long long rbase = 0;
  if (ckpt_base) rbase = ckpt_base[tile];
  unsigned short* list = s_list[warp];
  float2* tr = s_tr[warp];
  list[lane] = (unsigned short)kTilePixels;  // leading sentinels (pipeline fill)

  for (int g = warp; g < n_groups;) {
    const int p0 = g * kGroup;
    // invalid lanes (p >= n) never satisfy p < n_considered <= n
    const int p = p0 + lane < n ? p0 + lane : 0x7fffffff;
    float mx = 0.f, my = 0.f, a = 0.f, b = 0.f, c = 0.f, o = 0.f, cr = 0.f, cg = 0.f,
          cb = 0.f, dep = 0.f;
    int row = 0;
    if (p0 + lane < n) {
      row = values[start + p0 + lane];
      const float4 r0 = __ldg(rec + 3 * row), r1 = __ldg(rec + 3 * row + 1),
                   r2 = __ldg(rec + 3 * row + 2);
      mx = r0.x; my = r0.y;
      a = __fmul_rn(r0.z, kQScale);
      b = __fmul_rn(r0.w, kQScale);
      c = __fmul_rn(r1.x, kQScale);
      o = r1.y; dep = r1.z;
      cr = r2.x; cg = r2.y; cb = r2.z;
    }
    // prologue: compact the pixels that entered this group, with their
    // checkpoint state (T0, R0 = Ktot + g_T T_f - K_ckpt)
    int n_act = 0;
    for (int base = 0; base < kTilePixels; base += 32) {
      const int px = base + lane;
      const bool act = __float_as_int(s_pa[px].w) > p0;
      const unsigned bal = __ballot_sync(0xffffffffu, act);
      if (act) {
        const int kk = n_act + __popc(bal & lt_mask);
        float T0 = 1.f, K0 = 0.f;
        const float4 gv = s_pb[px];
        if (g > 0) {
          const float* src = ckpt + (rbase + g - 1) * (5 * kTilePixels) + px;
          T0 = src[0];
          K0 = gv.x * src[kTilePixels] + gv.y * src[2 * kTilePixels] +
               gv.z * src[3 * kTilePixels] + s_pa[px].z * src[4 * kTilePixels];
        }
        list[kListPad + kk] = (unsigned short)px;
        tr[kk] = make_float2(T0, gv.w - K0);
      }
      n_act += __popc(bal);
    }
    list[kListPad + n_act + lane] = (unsigned short)kTilePixels;  // trailing sentinels
    __syncwarp();

    float acc_mx = 0.f, acc_my = 0.f, acc_a = 0.f, acc_b = 0.f, acc_c = 0.f, acc_o = 0.f;
    float acc_r = 0.f, acc_g = 0.f, acc_bl = 0.f, acc_d = 0.f;
    float T_out = 1.f, R_out = 0.f;
    const unsigned short* my_list = list + kListPad - lane;
    const int steps = n_act + 31;
    for (int t = 0; t < steps; ++t) {
      const int px = my_list[t];
      float T_in = __shfl_up_sync(0xffffffffu, T_out, 1);
      float R_in = __shfl_up_sync(0xffffffffu, R_out, 1);
      if (lane == 0) {
        const float2 v = tr[t];
        T_in = v.x;
        R_in = v.y;
      }
      const float4 pa = s_pa[px];
      const float4 pb = s_pb[px];
      AlphaEval e = eval_alpha(pa.x, pa.y, mx, my, a, b, c, o);
      const bool part = (p < __float_as_int(pa.w)) && (e.alpha >= kMinAlpha);
      const float om = __fsub_rn(1.f, e.alpha);
      const float gcj = fmaf(pb.x, cr, fmaf(pb.y, cg, fmaf(pb.z, cb, pa.z * dep)));
      const float w = part ? T_in * e.alpha : 0.f;
      const float num = fmaf(-w, gcj, R_in);
      const float dLda = fmaf(-num, fast_rcp(om), T_in * gcj);
      T_out = part ? T_in * om : T_in;
      R_out = num;
      const bool live = part && !(e.raw > e.alpha);  // uncapped participant
      const float ld = live ? dLda : 0.f;
      const float gq = ld * e.alpha;  // x (-1/2) folded into the merge
      const float gqdx = gq * e.dx, gqdy = gq * e.dy;
      acc_a = fmaf(gqdx, e.dx, acc_a);
      acc_b = fmaf(gqdx, e.dy, acc_b);
      acc_c = fmaf(gqdy, e.dy, acc_c);
      acc_mx = fmaf(gq, e.u, acc_mx);
      acc_my = fmaf(gq, e.v, acc_my);
      acc_o = fmaf(ld, e.gauss, acc_o);
      acc_r = fmaf(w, pb.x, acc_r);
      acc_g = fmaf(w, pb.y, acc_g);
      acc_bl = fmaf(w, pb.z, acc_bl);
      acc_d = fmaf(w, pa.z, acc_d);
    }
    __syncwarp();
    // next group: dynamic, so warps of a tile finish together
    int next = 0;
    if (lane == 0) next = atomicAdd(&s_next_group, 1);
    g = __shfl_sync(0xffffffffu, next, 0);
    const bool touched = (acc_o != 0.f) | (acc_r != 0.f) | (acc_g != 0.f) | (acc_bl != 0.f) |
                         (acc_d != 0.f) | (acc_a != 0.f);
    if (p0 + lane < n && touched) {
      float* dst = grad2d + (long long)row * TSR_GRAD2D_FLOATS;
      atomicAdd(dst + 0, -0.5f * mean_scale * acc_mx);
      atomicAdd(dst + 1, -0.5f * mean_scale * acc_my);
      atomicAdd(dst + 2, -0.5f * acc_a);
      atomicAdd(dst + 3, -acc_b);
      atomicAdd(dst + 4, -0.5f * acc_c);
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
  render_bwd_kernel<<<tx * ty, kBwdThreads, 0, (cudaStream_t)stream>>>(
      (const float4*)rec, values, offsets, width, height, tx, color, depth, final_T,
      n_considered, ckpt, ckpt_base, grad_color, grad_depth, grad_final_T, grad2d, merges);
  TSR_CHECK_LAUNCH();
  return TSR_OK;
}
