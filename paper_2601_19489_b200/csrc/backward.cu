// K4: per-Gaussian raster backward (backward_per_gaussian, backward.py:137-223).
//
// One CTA per tile, 4 warps.  Per pixel and list position p, with gc_p =
// <g_color, c_p> + g_depth d_p folding the colour and depth suffixes of
// backward.py:195-205 into ONE scalar per (pixel, splat):
//   T_p = T_ckpt * prod_{i<p, part_i} (1 - alpha_i)
//   R_p = Ktot + g_T T_f - K_ckpt - sum_{i<=p} w_i gc_i
//   dL/dalpha_p = T_p gc_p - R_p / (1 - alpha_p)
// (the g_T channel is backward.py:170,204-205).
//
// Systolic schedule.  A warp owns a SUPERGROUP of 64 list positions (two
// 32-entry checkpoint groups, forward.py:28); lane j owns the adjacent pair
// (64G + 2j, 64G + 2j + 1) and runs both of its splats on the same pixel in
// one step: the alpha evaluation and every gradient accumulation are packed
// FP32x2 instructions (FFMA2/FMUL2/FADD2, one issue slot for two splats);
// only the T/R chain between the two splats is scalar.  The supergroup's
// active pixels (n_considered > 64G) are compacted into a list; at step t
// lane j works on list entry t - j and takes (T, R) from lane j - 1 by one
// shuffle each.  Per position this halves both the issued instructions and
// the pipeline fill of the one-splat-per-lane form.
//
// part = p < n_considered and alpha >= 1/255 (backward.py:189); capped alphas
// get zero conic/mean/opacity gradient (backward.py:64,72).  Gradients
// accumulate in registers and are merged once per (splat, tile) with atomics
// (backward.py:214-222).  The supergroup loop is bounded by the tile's
// maximum n_considered: later positions contribute exactly zero.  Alphas are
// bit-identical to K3's (same operation sequence; the packed instructions
// round each half exactly like the scalar ones).
#include <cuda_runtime.h>

#include "tsr_common.cuh"
#include "tsr_vjp_adam.cuh"

namespace tsr {

constexpr int kBwdWarps = 4;
constexpr int kBwdThreads = 32 * kBwdWarps;
constexpr int kSuper = 2 * kGroup;  // positions per warp work unit

__device__ __forceinline__ float fast_rcp(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ float2 f2(float x, float y) { return make_float2(x, y); }
__device__ __forceinline__ float2 bc(float x) { return make_float2(x, x); }

// per-pixel record (index kTilePixels is a dummy pixel with n_considered 0,
// used as the sentinel of the padded systolic lists)
constexpr int kPixSlots = kTilePixels + 1;
constexpr int kListPad = 32;

// per-pixel record, split in two 16-byte planes (structure of arrays) so the
// 32 lanes of a systolic step, which read 32 different pixels, spread over
// all eight 16-byte bank groups:
//   a = pixel centre x, y, g_depth, n_considered (int bits)
//   b = g_r, g_g, g_b, Ktot + g_T T_final

// K4 with the projection VJP and Adam fused into its tail (SH 0 training
// step).  Every CTA, after its merges, counts its list's pairs into a per-row
// counter; the CTA that completes a row (count == K1's pair count of the row:
// every tile holding the row has merged) runs that Gaussian's VJP + Adam, from
// a shared-memory queue so the work is convergent.  The HBM-bound update
// (~450 B per Gaussian) thus runs inside the FP32-bound backward instead of
// as a separate 90 us kernel after it; vjp_adam_rest_kernel updates the
// Gaussians without any pair and re-arms the counters.
struct FusedAdamArgs {
  tsr_camera_t cam;
  AdamGroups groups;
  const int32_t* source_ids;  // row -> Gaussian
  const int32_t* counts;      // K1: pairs of each row
  int32_t* row_done;          // merged (tile, row) pairs so far (zero between steps)
  const float* scal;          // per-step [lr, bc1, bc2] x 5 (device), or null: by value
  const int32_t* gate;        // K2's overflow flag (skip the update)
  const float* loss_guard;    // the step's loss (non-finite: skip the update)
  unsigned long long* skipped;
};

constexpr int kRowQueue = 1024;

__device__ __forceinline__ void fused_row_epilogue(const FusedAdamArgs& fa,
                                                   const int32_t* __restrict__ values,
                                                   long long start, int n,
                                                   const float4* __restrict__ rec,
                                                   float* __restrict__ grad2d, int* s_q,
                                                   int* s_qn) {
  __syncthreads();  // every warp of the CTA has issued its merges ...
  __threadfence();  // ... and they are visible before its counts
  const bool update = !((fa.gate && *fa.gate) || (fa.loss_guard && !isfinite(*fa.loss_guard)));
  unsigned long long skipped = 0;
  for (int base = 0; base < n; base += kRowQueue) {
    if (threadIdx.x == 0) *s_qn = 0;
    __syncthreads();
    for (int j = threadIdx.x; j < kRowQueue && base + j < n; j += kBwdThreads) {
      const int row = values[start + base + j];
      if (atomicAdd(fa.row_done + row, 1) == fa.counts[row] - 1) s_q[atomicAdd(s_qn, 1)] = row;
    }
    __syncthreads();
    const int qn = *s_qn;
    if (qn) __threadfence();  // the other tiles' merges of the completed rows
    for (int q = threadIdx.x; q < qn; q += kBwdThreads) {
      const int row = s_q[q];
      bool vis;
      float pose[12];
      skipped += vjp_adam_row_sh0<false, true>(fa.cam, fa.groups, fa.source_ids[row], row, rec,
                                               grad2d, fa.scal, update, pose, vis);
    }
    __syncthreads();
  }
  for (int d = 16; d > 0; d >>= 1) skipped += __shfl_xor_sync(0xffffffffu, skipped, d);
  if ((threadIdx.x & 31) == 0 && skipped) atomicAdd(fa.skipped, skipped);
}

// kDet: deterministic merge -- instead of atomics into grad2d, every pair of
// a processed supergroup writes its 10 scaled sums to slot[pair] (plain
// stores, one writer per pair) and the tile records how many list positions
// it processed; grad_reduce_kernel then sums each row's slots in emission
// order, so results are bitwise reproducible.
template <bool kDepth, bool kDet, bool kFused = false>
__global__ void __launch_bounds__(kBwdThreads, 5) render_bwd_kernel(
    const float4* __restrict__ rec, const int32_t* __restrict__ values,
    const int64_t* __restrict__ offsets, int width, int height, int tiles_x,
    const float* __restrict__ color, const float* __restrict__ depth,
    const float* __restrict__ final_T, const int32_t* __restrict__ n_considered,
    const float* __restrict__ ckpt, const int64_t* __restrict__ ckpt_base,
    const float* __restrict__ grad_color, const float* __restrict__ grad_depth,
    const float* __restrict__ grad_final_T, float* __restrict__ grad2d,
    unsigned long long* __restrict__ merges, float* __restrict__ slots,
    int32_t* __restrict__ processed, const int32_t* __restrict__ order,
    FusedAdamArgs fa = FusedAdamArgs{}) {
  __shared__ float4 s_pa[kPixSlots];
  __shared__ int s_q[kFused ? kRowQueue : 1];
  __shared__ int s_qn;
  __shared__ float4 s_pb[kPixSlots];
  // byte offsets; the step count is rounded up to a multiple of 4, hence
  // kListPad + 3 trailing sentinels
  __shared__ unsigned short s_list[kBwdWarps][kTilePixels + 2 * kListPad + 4];
  __shared__ float2 s_tr[kBwdWarps][kTilePixels + kListPad + 4];  // (T_ckpt, R_ckpt)
  __shared__ int s_maxnc;
  __shared__ int s_next;

  const int tile = (order && order[gridDim.x]) ? order[blockIdx.x]  // heavy tiles first
                                                : (int)blockIdx.x;
  const long long start = offsets[tile], end = offsets[tile + 1];
  const int n = (int)(end - start);
  if (n == 0) return;
  const int tyi = tile / tiles_x, txi = tile - tyi * tiles_x;
  const int tid = threadIdx.x;
  if (tid == 0) {
    s_maxnc = 0;
    s_next = kBwdWarps;  // supergroups 0..kBwdWarps-1 are taken statically
    s_pa[kTilePixels] = make_float4(-65536.f, -65536.f, 0.f, __int_as_float(0));  // gauss -> 0
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
      if (kDepth && grad_depth) gd = grad_depth[pix];
      if (grad_final_T) gt = grad_final_T[pix];
      nc = n_considered[pix];
      k = gr * color[3 * pix] + gg * color[3 * pix + 1] + gb * color[3 * pix + 2] + gt * final_T[pix];
      if (kDepth) k += gd * depth[pix];
    }
    nz |= (gr != 0.f) || (gg != 0.f) || (gb != 0.f) || (gd != 0.f) || (gt != 0.f);
    my_max = max(my_max, nc);
    s_pa[px] = make_float4((float)x + 0.5f, (float)y + 0.5f, gd, __int_as_float(nc));
    s_pb[px] = make_float4(gr, gg, gb, k);
  }
  // tile skipped when its upstream is all zero (backward.py:156-158); the
  // fused form still counts its pairs (their rows' updates wait on them)
  if (!__syncthreads_or(nz)) {
    if (kDet && tid == 0) processed[tile] = 0;
    if (kFused) fused_row_epilogue(fa, values, start, n, rec, grad2d, s_q, &s_qn);
    return;
  }
  atomicMax(&s_maxnc, my_max);
  if (tid == 0) atomicAdd(merges, (unsigned long long)n);
  __syncthreads();
  const int n_super = (s_maxnc + kSuper - 1) / kSuper;
  if (kDet && tid == 0) processed[tile] = n_super * kSuper;
  const int lane = tid & 31, warp = tid >> 5;
  const unsigned lt_mask = (1u << lane) - 1u;
  long long rbase = 0;
  if (ckpt_base) rbase = ckpt_base[tile];
  unsigned short* list = s_list[warp];
  float2* tr = s_tr[warp];
  const unsigned short kSentinel = (unsigned short)(kTilePixels * sizeof(float4));
  list[lane] = kSentinel;  // leading sentinels (pipeline fill)
  const char* pa_base = reinterpret_cast<const char*>(s_pa);
  const char* pb_base = reinterpret_cast<const char*>(s_pb);

  for (int G = warp; G < n_super;) {
    const int P0 = G * kSuper;
    const int p = P0 + 2 * lane;  // this lane's first position; second is p + 1
    // splat pair (invalid positions >= n never satisfy p < n_considered <= n)
    float2 mxn = bc(0.f), myn = bc(0.f), ca = bc(0.f), cb = bc(0.f), cc = bc(0.f), op = bc(0.f);
    float2 cr = bc(0.f), cg = bc(0.f), cbl = bc(0.f), dep = bc(0.f);
    int row0 = -1, row1 = -1;
    if (p < n) row0 = values[start + p];
    if (p + 1 < n) row1 = values[start + p + 1];
    if (row0 >= 0) {
      const float4 r0 = __ldg(rec + 3 * row0), r1 = __ldg(rec + 3 * row0 + 1),
                   r2 = __ldg(rec + 3 * row0 + 2);
      mxn.x = -r0.x; myn.x = -r0.y;
      ca.x = __fmul_rn(r0.z, kQScale);
      cb.x = __fmul_rn(r0.w, 2.0f * kQScale);
      cc.x = __fmul_rn(r1.x, kQScale);
      op.x = r1.y; dep.x = r1.z;
      cr.x = r2.x; cg.x = r2.y; cbl.x = r2.z;
    }
    if (row1 >= 0) {
      const float4 r0 = __ldg(rec + 3 * row1), r1 = __ldg(rec + 3 * row1 + 1),
                   r2 = __ldg(rec + 3 * row1 + 2);
      mxn.y = -r0.x; myn.y = -r0.y;
      ca.y = __fmul_rn(r0.z, kQScale);
      cb.y = __fmul_rn(r0.w, 2.0f * kQScale);
      cc.y = __fmul_rn(r1.x, kQScale);
      op.y = r1.y; dep.y = r1.z;
      cr.y = r2.x; cg.y = r2.y; cbl.y = r2.z;
    }
    // prologue: compact the pixels that entered this supergroup, with their
    // checkpoint state (T0, R0 = Ktot + g_T T_f - K_ckpt).  All checkpoint
    // loads of a lane are issued before any is consumed.
    {
      const float* src0 = G > 0 ? ckpt + (rbase + 2 * G - 1) * (5 * kTilePixels) : nullptr;
      bool act[kTilePixels / 32];
      float cT[kTilePixels / 32], c1[kTilePixels / 32], c2[kTilePixels / 32],
          c3[kTilePixels / 32], c4[kTilePixels / 32];
#pragma unroll
      for (int s = 0; s < kTilePixels / 32; ++s) {
        const int px = 32 * s + lane;
        act[s] = __float_as_int(s_pa[px].w) > P0;
        cT[s] = 1.f; c1[s] = c2[s] = c3[s] = c4[s] = 0.f;
        if (src0 && act[s]) {
          cT[s] = src0[px];
          c1[s] = src0[kTilePixels + px];
          c2[s] = src0[2 * kTilePixels + px];
          c3[s] = src0[3 * kTilePixels + px];
          if (kDepth) c4[s] = src0[4 * kTilePixels + px];
        }
      }
      int n_act = 0;
#pragma unroll
      for (int s = 0; s < kTilePixels / 32; ++s) {
        const int px = 32 * s + lane;
        const unsigned bal = __ballot_sync(0xffffffffu, act[s]);
        if (act[s]) {
          const int kk = n_act + __popc(bal & lt_mask);
          const float4 pra = s_pa[px], prb = s_pb[px];
          float K0 = prb.x * c1[s] + prb.y * c2[s] + prb.z * c3[s];
          if (kDepth) K0 += pra.z * c4[s];
          list[kListPad + kk] = (unsigned short)(px * sizeof(float4));
          tr[kk] = make_float2(cT[s], prb.w - K0);
        }
        n_act += __popc(bal);
      }
      // trailing sentinels; their (T, R) entries are finite zeros so the
      // sentinel steps contribute exact zeros (w = T * 0)
      list[kListPad + n_act + lane] = kSentinel;
      tr[n_act + lane] = make_float2(0.f, 0.f);
      if (lane < 3) {
        list[kListPad + n_act + 32 + lane] = kSentinel;
        tr[n_act + 32 + lane] = make_float2(0.f, 0.f);
      }
      __syncwarp();

      float2 acc_a = bc(0.f), acc_b = bc(0.f), acc_c = bc(0.f), acc_mx = bc(0.f), acc_my = bc(0.f);
      float2 acc_o = bc(0.f), acc_r = bc(0.f), acc_g = bc(0.f), acc_bl = bc(0.f), acc_d = bc(0.f);
      float T_out = 1.f, R_out = 0.f;
      const unsigned short* my_list = list + kListPad - lane;
      const int steps = (n_act + 31 + 3) & ~3;  // sentinel steps pad to a multiple of 4
      const float2 one = bc(1.f);
      // one systolic step of this lane's splat pair on pixel record (pa, pb)
      auto step = [&](const float4& pa, const float4& pb, int t) {
        float T_in = __shfl_up_sync(0xffffffffu, T_out, 1);
        float R_in = __shfl_up_sync(0xffffffffu, R_out, 1);
        if (lane == 0) {
          const float2 v = tr[t];
          T_in = v.x;
          R_in = v.y;
        }
        const int nc = __float_as_int(pa.w);
        // alpha of both splats at this pixel (eval_alpha, packed)
        const float2 dx = __fadd2_rn(bc(pa.x), mxn);
        const float2 dy = __fadd2_rn(bc(pa.y), myn);
        const float2 dxx = __fmul2_rn(dx, dx), dxy = __fmul2_rn(dx, dy), dyy = __fmul2_rn(dy, dy);
        const float2 qs = __ffma2_rn(ca, dxx, __ffma2_rn(cb, dxy, __fmul2_rn(cc, dyy)));
        const float2 gauss = f2(fast_exp2(qs.x), fast_exp2(qs.y));
        // two scalar multiplies (bitwise the packed product): the opacity
        // pair does not live in an aligned register pair, and a packed
        // multiply would copy it every step
        const float2 raw = f2(__fmul_rn(op.x, gauss.x), __fmul_rn(op.y, gauss.y));
        const float2 alpha = f2(fminf(kAlphaCap, raw.x), fminf(kAlphaCap, raw.y));
        // predicates chained so each costs one compare (alpha >= 1/255 <=>
        // raw >= 1/255 since the cap is above it)
        // a = (p < nc && alpha >= 1/255) ? alpha : 0 as one chained compare
        // + select per splat (inline PTX: the compiler otherwise splits the
        // chain into two selects).  Non-participants get a = 0: w = T * 0 = 0
        // and T * (1 - 0) = T exactly (no selects on the chain; their
        // 1 / (1 - a) is unused).
        float a0, a1;
        asm("{\n\t.reg .pred q;\n\t"
            "setp.lt.s32 q, %1, %2;\n\t"
            "setp.ge.and.f32 q, %3, %4, q;\n\t"
            "selp.f32 %0, %3, 0f00000000, q;\n\t}"
            : "=f"(a0) : "r"(p), "r"(nc), "f"(alpha.x), "f"(kMinAlpha));
        asm("{\n\t.reg .pred q;\n\t"
            "setp.lt.s32 q, %1, %2;\n\t"
            "setp.ge.and.f32 q, %3, %4, q;\n\t"
            "selp.f32 %0, %3, 0f00000000, q;\n\t}"
            : "=f"(a1) : "r"(p + 1), "r"(nc), "f"(alpha.y), "f"(kMinAlpha));
        const float2 a = f2(a0, a1);
        const float2 om = __fadd2_rn(one, f2(-a.x, -a.y));
        float2 gc = __ffma2_rn(bc(pb.x), cr, __ffma2_rn(bc(pb.y), cg, __fmul2_rn(bc(pb.z), cbl)));
        if (kDepth) gc = __ffma2_rn(bc(pa.z), dep, gc);
        // scalar chain through the pair
        const float w0 = T_in * a.x;
        const float T1 = T_in * om.x;
        const float w1 = T1 * a.y;
        T_out = T1 * om.y;
        const float num0 = fmaf(-w0, gc.x, R_in);
        const float num1 = fmaf(-w1, gc.y, num0);
        R_out = num1;
        const float2 rcp = f2(fast_rcp(om.x), fast_rcp(om.y));
        const float2 dLda = f2(fmaf(-num0, rcp.x, T_in * gc.x), fmaf(-num1, rcp.y, T1 * gc.y));
        // uncapped participants only (backward.py:64,72): 1/255 <= raw <= 0.99
        // (then alpha == raw); x(-1/2) folded into the merge
        // one compare: a == raw holds exactly for uncapped participants
        // (a = alpha = raw), fails for capped ones (a = 0.99 < raw) and for
        // non-participants with raw != 0 (a = 0); a non-participant with
        // raw == 0 keeps its finite dLda but has alpha = gauss = 0, so every
        // product below is zero
        const float2 ld = f2(a.x == raw.x ? dLda.x : 0.f, a.y == raw.y ? dLda.y : 0.f);
        const float2 gq = __fmul2_rn(ld, alpha);
        acc_a = __ffma2_rn(gq, dxx, acc_a);
        acc_b = __ffma2_rn(gq, dxy, acc_b);
        acc_c = __ffma2_rn(gq, dyy, acc_c);
        acc_mx = __ffma2_rn(gq, dx, acc_mx);  // sum gq dx; times the conic at the merge
        acc_my = __ffma2_rn(gq, dy, acc_my);
        acc_o = __ffma2_rn(ld, gauss, acc_o);
        const float2 w = f2(w0, w1);
        acc_r = __ffma2_rn(w, bc(pb.x), acc_r);
        acc_g = __ffma2_rn(w, bc(pb.y), acc_g);
        acc_bl = __ffma2_rn(w, bc(pb.z), acc_bl);
        if (kDepth) acc_d = __ffma2_rn(w, bc(pa.z), acc_d);
      };
      // software pipeline, unrolled by four with ping-pong registers: the
      // next step's pixel record is loaded while this step computes (the
      // padded list makes the loads past the end read sentinels)
      float4 pa0 = *reinterpret_cast<const float4*>(pa_base + my_list[0]);
      float4 pb0 = *reinterpret_cast<const float4*>(pb_base + my_list[0]);
      float4 pa1, pb1;
      auto load = [&](float4& a, float4& b, int t) {
        const unsigned off = my_list[t];
        a = *reinterpret_cast<const float4*>(pa_base + off);
        b = *reinterpret_cast<const float4*>(pb_base + off);
      };
      for (int t = 0; t < steps; t += 4) {
        load(pa1, pb1, t + 1);
        step(pa0, pb0, t);
        load(pa0, pb0, t + 2);
        step(pa1, pb1, t + 1);
        load(pa1, pb1, t + 3);
        step(pa0, pb0, t + 2);
        load(pa0, pb0, t + 4);
        step(pa1, pb1, t + 3);
      }
      __syncwarp();
      // next supergroup: dynamic, so the warps of a tile finish together
      int next = 0;
      if (lane == 0) next = atomicAdd(&s_next, 1);
      G = __shfl_sync(0xffffffffu, next, 0);
      const float ms = 2.0f / kQScale;  // d/dmean of the prescaled quadratic, x(-1/2)
      // sum gq u = a' sum gq dx + b' sum gq dy (b' = b2' / 2), likewise v
      {
        const float2 hb = __fmul2_rn(cb, bc(0.5f));
        const float2 u = __ffma2_rn(ca, acc_mx, __fmul2_rn(hb, acc_my));
        const float2 v = __ffma2_rn(hb, acc_mx, __fmul2_rn(cc, acc_my));
        acc_mx = u;
        acc_my = v;
      }
      if (kDet) {
        if (row0 >= 0) {
          float* dst = slots + (start + p) * TSR_GRAD2D_FLOATS;
          dst[0] = ms * 0.5f * acc_mx.x; dst[1] = ms * 0.5f * acc_my.x;
          dst[2] = -0.5f * acc_a.x; dst[3] = -acc_b.x; dst[4] = -0.5f * acc_c.x;
          dst[5] = acc_o.x; dst[6] = acc_r.x; dst[7] = acc_g.x; dst[8] = acc_bl.x;
          dst[9] = kDepth ? acc_d.x : 0.f;
        }
        if (row1 >= 0) {
          float* dst = slots + (start + p + 1) * TSR_GRAD2D_FLOATS;
          dst[0] = ms * 0.5f * acc_mx.y; dst[1] = ms * 0.5f * acc_my.y;
          dst[2] = -0.5f * acc_a.y; dst[3] = -acc_b.y; dst[4] = -0.5f * acc_c.y;
          dst[5] = acc_o.y; dst[6] = acc_r.y; dst[7] = acc_g.y; dst[8] = acc_bl.y;
          dst[9] = kDepth ? acc_d.y : 0.f;
        }
        continue;
      }
      if (row0 >= 0 && ((acc_o.x != 0.f) | (acc_r.x != 0.f) | (acc_g.x != 0.f) |
                        (acc_bl.x != 0.f) | (acc_d.x != 0.f) | (acc_a.x != 0.f))) {
        float* dst = grad2d + (long long)row0 * TSR_GRAD2D_FLOATS;
        atomicAdd(dst + 0, ms * 0.5f * acc_mx.x);
        atomicAdd(dst + 1, ms * 0.5f * acc_my.x);
        atomicAdd(dst + 2, -0.5f * acc_a.x);
        atomicAdd(dst + 3, -acc_b.x);
        atomicAdd(dst + 4, -0.5f * acc_c.x);
        atomicAdd(dst + 5, acc_o.x);
        atomicAdd(dst + 6, acc_r.x);
        atomicAdd(dst + 7, acc_g.x);
        atomicAdd(dst + 8, acc_bl.x);
        if (kDepth) atomicAdd(dst + 9, acc_d.x);
      }
      if (row1 >= 0 && ((acc_o.y != 0.f) | (acc_r.y != 0.f) | (acc_g.y != 0.f) |
                        (acc_bl.y != 0.f) | (acc_d.y != 0.f) | (acc_a.y != 0.f))) {
        float* dst = grad2d + (long long)row1 * TSR_GRAD2D_FLOATS;
        atomicAdd(dst + 0, ms * 0.5f * acc_mx.y);
        atomicAdd(dst + 1, ms * 0.5f * acc_my.y);
        atomicAdd(dst + 2, -0.5f * acc_a.y);
        atomicAdd(dst + 3, -acc_b.y);
        atomicAdd(dst + 4, -0.5f * acc_c.y);
        atomicAdd(dst + 5, acc_o.y);
        atomicAdd(dst + 6, acc_r.y);
        atomicAdd(dst + 7, acc_g.y);
        atomicAdd(dst + 8, acc_bl.y);
        if (kDepth) atomicAdd(dst + 9, acc_d.y);
      }
    }
  }
  if (kFused) fused_row_epilogue(fa, values, start, n, rec, grad2d, s_q, &s_qn);
}

// ---- K4, work-unit form ---------------------------------------------------
// The same systolic supergroup step, scheduled per WARP instead of per tile.
// A work unit is one (tile, supergroup G) pair; the units of all tiles are
// laid out in raster order (unit_plan_kernel) and every warp of a persistent
// grid grabs the next unit from a global counter.  So a heavy tile's
// supergroups spread over as many warps as the GPU has free (the paper's
// work redistribution across heavy tiles), and no warp of
// a CTA idles while a sibling finishes a tile (the per-tile CTA form leaves
// ~20 % of the warp slots empty: 4 warps share 3-9 supergroups).
//
// Each warp compacts the unit's active pixels (n_considered > 64 G) into its
// own shared-memory records, with the supergroup's entry state folded in:
//   a = (x + 1/2, y + 1/2, T0, n_considered)   b = (g_r, g_g, g_b, R0)
// (T0, R0) = checkpoint record 2G - 1 (T, Ktot + g_T T_f - <g, C> - g_d D),
// or (1, Ktot + g_T T_f) for G = 0.  The records sit at [32, 32 + n_act)
// between sentinel records (x = -65536: alpha 0; T0 = R0 = 0), so lane j at
// step t reads record 32 + t - j at a lane-constant base + 16 t: no list
// indirection, and lane 0 takes (T0, R0) from the record it loads anyway.
constexpr int kRecPad = 32;
constexpr int kRecSlots = kRecPad + kTilePixels + kListPad + 4;

// unit plan, part 1: supergroups per tile = ceil(max n_considered / 64) (one
// warp per tile).  Later positions contribute exactly zero.
__global__ void __launch_bounds__(256) unit_count_kernel(const int64_t* __restrict__ offsets,
                                                         const int32_t* __restrict__ n_considered,
                                                         int width, int height, int tiles_x,
                                                         int n_tiles, int32_t* __restrict__ nsup) {
  const int tile = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (tile >= n_tiles) return;
  const int tyi = tile / tiles_x, txi = tile - tyi * tiles_x;
  int mx = 0;
#pragma unroll
  for (int s = 0; s < kTilePixels / 32; ++s) {
    const int px = 32 * s + lane;
    const int x = txi * kTile + (px & 15), y = tyi * kTile + (px >> 4);
    if (x < width && y < height) mx = max(mx, n_considered[(long long)y * width + x]);
  }
  mx = __reduce_max_sync(0xffffffffu, mx);
  if (lane == 0) {
    const long long n = offsets[tile + 1] - offsets[tile];
    const long long m = min((long long)mx, n);
    nsup[tile] = (int32_t)((m + kSuper - 1) / kSuper);
  }
}

// unit plan, part 2 (one CTA): exclusive scan of the per-tile counts ->
// units[U_t + g] = tile << 16 | g; the unit count; the grab counter reset;
// and, for the deterministic merge, processed[t] = 64 x supergroups.
constexpr int kPlanThreads = 1024;
constexpr int kPlanMaxTiles = 12288;  // staged counts (48 KB); larger frames read global
__global__ void __launch_bounds__(kPlanThreads) unit_plan_kernel(
    const int32_t* __restrict__ nsup, int n_tiles, uint32_t* __restrict__ units,
    long long units_cap, int32_t* __restrict__ n_units, int32_t* __restrict__ counter,
    int32_t* __restrict__ processed) {
  extern __shared__ int s_n[];  // per-tile supergroup counts (coalesced stage)
  __shared__ int s_w[kPlanThreads / 32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const bool staged = n_tiles <= kPlanMaxTiles;
  if (staged)
    for (int t = tid; t < n_tiles; t += kPlanThreads) s_n[t] = nsup[t];
  __syncthreads();
  auto cnt = [&](int t) { return staged ? s_n[t] : nsup[t]; };
  const int per = (n_tiles + kPlanThreads - 1) / kPlanThreads;
  const int t0 = tid * per, t1 = min(n_tiles, t0 + per);
  int sum = 0;
  for (int t = t0; t < t1; ++t) sum += cnt(t);
  int incl = sum;
#pragma unroll
  for (int k = 1; k < 32; k <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, incl, k);
    if (lane >= k) incl += v;
  }
  if (lane == 31) s_w[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    int w = s_w[lane], wi = w;
#pragma unroll
    for (int k = 1; k < 32; k <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, wi, k);
      if (lane >= k) wi += v;
    }
    s_w[lane] = wi - w;  // exclusive prefix of the warps
  }
  __syncthreads();
  long long u = (long long)s_w[warp] + incl - sum;
  for (int t = t0; t < t1; ++t) {
    const int k = cnt(t);
    if (processed) processed[t] = k * kSuper;
    for (int g = 0; g < k; ++g, ++u)
      if (u < units_cap) units[u] = ((uint32_t)t << 16) | (uint32_t)g;
  }
  if (tid == kPlanThreads - 1) {
    *n_units = (int32_t)min(u, units_cap);
    *counter = 0;
  }
}

template <bool kDepth, bool kDet>
__global__ void __launch_bounds__(kBwdThreads, 5) render_bwd_units_kernel(
    const float4* __restrict__ rec, const int32_t* __restrict__ values,
    const int64_t* __restrict__ offsets, int width, int height, int tiles_x,
    const float* __restrict__ color, const float* __restrict__ depth,
    const float* __restrict__ final_T, const int32_t* __restrict__ n_considered,
    const float* __restrict__ ckpt, const int64_t* __restrict__ ckpt_base,
    const float* __restrict__ grad_color, const float* __restrict__ grad_depth,
    const float* __restrict__ grad_final_T, float* __restrict__ grad2d,
    unsigned long long* __restrict__ merges, float* __restrict__ slots,
    const uint32_t* __restrict__ units, const int32_t* __restrict__ n_units_dev,
    int32_t* __restrict__ counter, int32_t* __restrict__ processed) {
  __shared__ float4 s_pa[kBwdWarps][kRecSlots];
  __shared__ float4 s_pb[kBwdWarps][kRecSlots];
  __shared__ float s_gd[kDepth ? kBwdWarps : 1][kDepth ? kRecSlots : 1];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned lt_mask = (1u << lane) - 1u;
  float4* pa = s_pa[warp];
  float4* pb = s_pb[warp];
  float* gdv = kDepth ? s_gd[warp] : nullptr;
  const float4 sent_a = make_float4(-65536.f, -65536.f, 0.f, __int_as_float(0));
  const float4 sent_b = make_float4(0.f, 0.f, 0.f, 0.f);
  pa[lane] = sent_a;  // leading sentinels (records start at kRecPad)
  pb[lane] = sent_b;
  if (kDepth) gdv[lane] = 0.f;
  const int n_units = *n_units_dev;
  for (;;) {
    int u = 0;
    if (lane == 0) u = atomicAdd(counter, 1);
    u = __shfl_sync(0xffffffffu, u, 0);
    if (u >= n_units) break;
    const uint32_t code = units[u];
    const int tile = (int)(code >> 16), G = (int)(code & 0xffffu);
    const long long start = offsets[tile], end = offsets[tile + 1];
    const int n = (int)(end - start);
    const int tyi = tile / tiles_x, txi = tile - tyi * tiles_x;
    const int P0 = G * kSuper;
    const int p = P0 + 2 * lane;  // this lane's first position; second is p + 1
    int row0 = -1, row1 = -1;
    if (p < n) row0 = values[start + p];
    if (p + 1 < n) row1 = values[start + p + 1];
    // ---- compact the unit's active pixels with their entry state
    const float* src0 = G > 0 ? ckpt + (ckpt_base[tile] + 2 * G - 1) * (5 * kTilePixels) : nullptr;
    int nc[kTilePixels / 32];
    long long pix[kTilePixels / 32];
#pragma unroll
    for (int s = 0; s < kTilePixels / 32; ++s) {
      const int px = 32 * s + lane;
      const int x = txi * kTile + (px & 15), y = tyi * kTile + (px >> 4);
      const bool inside = x < width && y < height;
      pix[s] = (long long)y * width + x;
      nc[s] = inside ? n_considered[pix[s]] : 0;
    }
    bool nz = false;
    int n_act = 0;
#pragma unroll
    for (int s = 0; s < kTilePixels / 32; ++s) {
      const bool act = nc[s] > P0;
      const unsigned bal = __ballot_sync(0xffffffffu, act);
      if (act) {
        const int px = 32 * s + lane;
        const long long q = pix[s];
        const float gr = grad_color[3 * q], gg = grad_color[3 * q + 1], gb = grad_color[3 * q + 2];
        const float gd = (kDepth && grad_depth) ? grad_depth[q] : 0.f;
        const float gt = grad_final_T ? grad_final_T[q] : 0.f;
        float k = gr * color[3 * q] + gg * color[3 * q + 1] + gb * color[3 * q + 2] + gt * final_T[q];
        if (kDepth) k += gd * depth[q];
        float T0 = 1.f, K0 = 0.f;
        if (src0) {
          T0 = src0[px];
          K0 = gr * src0[kTilePixels + px] + gg * src0[2 * kTilePixels + px] +
               gb * src0[3 * kTilePixels + px];
          if (kDepth) K0 += gd * src0[4 * kTilePixels + px];
        }
        nz |= (gr != 0.f) || (gg != 0.f) || (gb != 0.f) || (gd != 0.f) || (gt != 0.f);
        const int kk = kRecPad + n_act + __popc(bal & lt_mask);
        pa[kk] = make_float4((float)(txi * kTile + (px & 15)) + 0.5f,
                             (float)(tyi * kTile + (px >> 4)) + 0.5f, T0, __int_as_float(nc[s]));
        pb[kk] = make_float4(gr, gg, gb, k - K0);
        if (kDepth) gdv[kk] = gd;
      }
      n_act += __popc(bal);
    }
    // tile skipped when its upstream is all zero (backward.py:156-158): the
    // G = 0 unit sees every in-image pixel; a later unit whose active pixels
    // carry no upstream contributes exact zeros
    if (!__any_sync(0xffffffffu, nz)) {
      if (kDet) {  // the reducer reads slots below processed[tile]
        if (G == 0) {
          if (lane == 0) processed[tile] = 0;  // skipped tile
        } else {
#pragma unroll
          for (int j = 0; j < TSR_GRAD2D_FLOATS; ++j) {
            if (row0 >= 0) slots[(start + p) * TSR_GRAD2D_FLOATS + j] = 0.f;
            if (row1 >= 0) slots[(start + p + 1) * TSR_GRAD2D_FLOATS + j] = 0.f;
          }
        }
      }
      continue;
    }
    if (G == 0 && lane == 0) atomicAdd(merges, (unsigned long long)n);
    // trailing sentinels (finite zero T0, R0: the sentinel steps add zeros)
    pa[kRecPad + n_act + lane] = sent_a;
    pb[kRecPad + n_act + lane] = sent_b;
    if (kDepth) gdv[kRecPad + n_act + lane] = 0.f;
    if (lane < 4) {
      pa[kRecPad + n_act + 32 + lane] = sent_a;
      pb[kRecPad + n_act + 32 + lane] = sent_b;
      if (kDepth) gdv[kRecPad + n_act + 32 + lane] = 0.f;
    }
    float2 mxn = bc(0.f), myn = bc(0.f), ca = bc(0.f), cb = bc(0.f), cc = bc(0.f), op = bc(0.f);
    float2 cr = bc(0.f), cg = bc(0.f), cbl = bc(0.f), dep = bc(0.f);
    if (row0 >= 0) {
      const float4 r0 = __ldg(rec + 3 * row0), r1 = __ldg(rec + 3 * row0 + 1),
                   r2 = __ldg(rec + 3 * row0 + 2);
      mxn.x = -r0.x; myn.x = -r0.y;
      ca.x = __fmul_rn(r0.z, kQScale);
      cb.x = __fmul_rn(r0.w, 2.0f * kQScale);
      cc.x = __fmul_rn(r1.x, kQScale);
      op.x = r1.y; dep.x = r1.z;
      cr.x = r2.x; cg.x = r2.y; cbl.x = r2.z;
    }
    if (row1 >= 0) {
      const float4 r0 = __ldg(rec + 3 * row1), r1 = __ldg(rec + 3 * row1 + 1),
                   r2 = __ldg(rec + 3 * row1 + 2);
      mxn.y = -r0.x; myn.y = -r0.y;
      ca.y = __fmul_rn(r0.z, kQScale);
      cb.y = __fmul_rn(r0.w, 2.0f * kQScale);
      cc.y = __fmul_rn(r1.x, kQScale);
      op.y = r1.y; dep.y = r1.z;
      cr.y = r2.x; cg.y = r2.y; cbl.y = r2.z;
    }
    __syncwarp();

    float2 acc_a = bc(0.f), acc_b = bc(0.f), acc_c = bc(0.f), acc_mx = bc(0.f), acc_my = bc(0.f);
    float2 acc_o = bc(0.f), acc_r = bc(0.f), acc_g = bc(0.f), acc_bl = bc(0.f), acc_d = bc(0.f);
    float T_out = 1.f, R_out = 0.f;
    const char* a_base = reinterpret_cast<const char*>(pa + kRecPad - lane);
    const char* b_base = reinterpret_cast<const char*>(pb + kRecPad - lane);
    const float* g_base = kDepth ? gdv + kRecPad - lane : nullptr;
    const int steps = (n_act + 31 + 3) & ~3;  // sentinel steps pad to a multiple of 4
    const float2 one = bc(1.f);
    auto step = [&](const float4& ra, const float4& rb, float gdp) {
      float T_in = __shfl_up_sync(0xffffffffu, T_out, 1);
      float R_in = __shfl_up_sync(0xffffffffu, R_out, 1);
      if (lane == 0) {
        T_in = ra.z;
        R_in = rb.w;
      }
      const int ncp = __float_as_int(ra.w);
      const float2 dx = __fadd2_rn(bc(ra.x), mxn);
      const float2 dy = __fadd2_rn(bc(ra.y), myn);
      const float2 dxx = __fmul2_rn(dx, dx), dxy = __fmul2_rn(dx, dy), dyy = __fmul2_rn(dy, dy);
      const float2 qs = __ffma2_rn(ca, dxx, __ffma2_rn(cb, dxy, __fmul2_rn(cc, dyy)));
      const float2 gauss = f2(fast_exp2(qs.x), fast_exp2(qs.y));
      const float2 raw = f2(__fmul_rn(op.x, gauss.x), __fmul_rn(op.y, gauss.y));
      const float2 alpha = f2(fminf(kAlphaCap, raw.x), fminf(kAlphaCap, raw.y));
      float a0, a1;
      asm("{\n\t.reg .pred q;\n\t"
          "setp.lt.s32 q, %1, %2;\n\t"
          "setp.ge.and.f32 q, %3, %4, q;\n\t"
          "selp.f32 %0, %3, 0f00000000, q;\n\t}"
          : "=f"(a0) : "r"(p), "r"(ncp), "f"(alpha.x), "f"(kMinAlpha));
      asm("{\n\t.reg .pred q;\n\t"
          "setp.lt.s32 q, %1, %2;\n\t"
          "setp.ge.and.f32 q, %3, %4, q;\n\t"
          "selp.f32 %0, %3, 0f00000000, q;\n\t}"
          : "=f"(a1) : "r"(p + 1), "r"(ncp), "f"(alpha.y), "f"(kMinAlpha));
      const float2 a = f2(a0, a1);
      const float2 om = __fadd2_rn(one, f2(-a.x, -a.y));
      float2 gc = __ffma2_rn(bc(rb.x), cr, __ffma2_rn(bc(rb.y), cg, __fmul2_rn(bc(rb.z), cbl)));
      if (kDepth) gc = __ffma2_rn(bc(gdp), dep, gc);
      const float w0 = T_in * a.x;
      const float T1 = T_in * om.x;
      const float w1 = T1 * a.y;
      T_out = T1 * om.y;
      const float num0 = fmaf(-w0, gc.x, R_in);
      const float num1 = fmaf(-w1, gc.y, num0);
      R_out = num1;
      const float2 rcp = f2(fast_rcp(om.x), fast_rcp(om.y));
      const float2 dLda = f2(fmaf(-num0, rcp.x, T_in * gc.x), fmaf(-num1, rcp.y, T1 * gc.y));
      const float2 ld = f2(a.x == raw.x ? dLda.x : 0.f, a.y == raw.y ? dLda.y : 0.f);
      const float2 gq = __fmul2_rn(ld, alpha);
      acc_a = __ffma2_rn(gq, dxx, acc_a);
      acc_b = __ffma2_rn(gq, dxy, acc_b);
      acc_c = __ffma2_rn(gq, dyy, acc_c);
      acc_mx = __ffma2_rn(gq, dx, acc_mx);
      acc_my = __ffma2_rn(gq, dy, acc_my);
      acc_o = __ffma2_rn(ld, gauss, acc_o);
      const float2 w = f2(w0, w1);
      acc_r = __ffma2_rn(w, bc(rb.x), acc_r);
      acc_g = __ffma2_rn(w, bc(rb.y), acc_g);
      acc_bl = __ffma2_rn(w, bc(rb.z), acc_bl);
      if (kDepth) acc_d = __ffma2_rn(w, bc(gdp), acc_d);
    };
    auto ld_a = [&](int t) { return *reinterpret_cast<const float4*>(a_base + 16 * t); };
    auto ld_b = [&](int t) { return *reinterpret_cast<const float4*>(b_base + 16 * t); };
    auto ld_g = [&](int t) { return kDepth ? g_base[t] : 0.f; };
    float4 a0r = ld_a(0), b0r = ld_b(0), a1r, b1r;
    float g0r = ld_g(0), g1r;
    for (int t = 0; t < steps; t += 4) {
      a1r = ld_a(t + 1); b1r = ld_b(t + 1); g1r = ld_g(t + 1);
      step(a0r, b0r, g0r);
      a0r = ld_a(t + 2); b0r = ld_b(t + 2); g0r = ld_g(t + 2);
      step(a1r, b1r, g1r);
      a1r = ld_a(t + 3); b1r = ld_b(t + 3); g1r = ld_g(t + 3);
      step(a0r, b0r, g0r);
      a0r = ld_a(t + 4); b0r = ld_b(t + 4); g0r = ld_g(t + 4);
      step(a1r, b1r, g1r);
    }
    __syncwarp();  // records are rewritten by the next unit
    const float ms = 2.0f / kQScale;
    {
      const float2 hb = __fmul2_rn(cb, bc(0.5f));
      const float2 uu = __ffma2_rn(ca, acc_mx, __fmul2_rn(hb, acc_my));
      const float2 vv = __ffma2_rn(hb, acc_mx, __fmul2_rn(cc, acc_my));
      acc_mx = uu;
      acc_my = vv;
    }
    if (kDet) {
      if (row0 >= 0) {
        float* dst = slots + (start + p) * TSR_GRAD2D_FLOATS;
        dst[0] = ms * 0.5f * acc_mx.x; dst[1] = ms * 0.5f * acc_my.x;
        dst[2] = -0.5f * acc_a.x; dst[3] = -acc_b.x; dst[4] = -0.5f * acc_c.x;
        dst[5] = acc_o.x; dst[6] = acc_r.x; dst[7] = acc_g.x; dst[8] = acc_bl.x;
        dst[9] = kDepth ? acc_d.x : 0.f;
      }
      if (row1 >= 0) {
        float* dst = slots + (start + p + 1) * TSR_GRAD2D_FLOATS;
        dst[0] = ms * 0.5f * acc_mx.y; dst[1] = ms * 0.5f * acc_my.y;
        dst[2] = -0.5f * acc_a.y; dst[3] = -acc_b.y; dst[4] = -0.5f * acc_c.y;
        dst[5] = acc_o.y; dst[6] = acc_r.y; dst[7] = acc_g.y; dst[8] = acc_bl.y;
        dst[9] = kDepth ? acc_d.y : 0.f;
      }
      continue;
    }
    if (row0 >= 0 && ((acc_o.x != 0.f) | (acc_r.x != 0.f) | (acc_g.x != 0.f) |
                      (acc_bl.x != 0.f) | (acc_d.x != 0.f) | (acc_a.x != 0.f))) {
      float* dst = grad2d + (long long)row0 * TSR_GRAD2D_FLOATS;
      atomicAdd(dst + 0, ms * 0.5f * acc_mx.x);
      atomicAdd(dst + 1, ms * 0.5f * acc_my.x);
      atomicAdd(dst + 2, -0.5f * acc_a.x);
      atomicAdd(dst + 3, -acc_b.x);
      atomicAdd(dst + 4, -0.5f * acc_c.x);
      atomicAdd(dst + 5, acc_o.x);
      atomicAdd(dst + 6, acc_r.x);
      atomicAdd(dst + 7, acc_g.x);
      atomicAdd(dst + 8, acc_bl.x);
      if (kDepth) atomicAdd(dst + 9, acc_d.x);
    }
    if (row1 >= 0 && ((acc_o.y != 0.f) | (acc_r.y != 0.f) | (acc_g.y != 0.f) |
                      (acc_bl.y != 0.f) | (acc_d.y != 0.f) | (acc_a.y != 0.f))) {
      float* dst = grad2d + (long long)row1 * TSR_GRAD2D_FLOATS;
      atomicAdd(dst + 0, ms * 0.5f * acc_mx.y);
      atomicAdd(dst + 1, ms * 0.5f * acc_my.y);
      atomicAdd(dst + 2, -0.5f * acc_a.y);
      atomicAdd(dst + 3, -acc_b.y);
      atomicAdd(dst + 4, -0.5f * acc_c.y);
      atomicAdd(dst + 5, acc_o.y);
      atomicAdd(dst + 6, acc_r.y);
      atomicAdd(dst + 7, acc_g.y);
      atomicAdd(dst + 8, acc_bl.y);
      if (kDepth) atomicAdd(dst + 9, acc_d.y);
    }
  }
}

// Deterministic merge, second half: one thread per depth rank sums its
// row's slots in emission order (binning.py:217-221: the row's pairs are a
// contiguous emission range [rank_off, rank_off + rank_count), and K2's
// inverse permutation gives each pair's sorted position); a slot counts only
// if its tile processed that list position.  No searches, no atomics.
__global__ void __launch_bounds__(256) grad_reduce_kernel(
    const uint32_t* __restrict__ rank_row, const uint32_t* __restrict__ rank_count,
    const uint32_t* __restrict__ rank_off, const uint32_t* __restrict__ inv_perm,
    const int64_t* __restrict__ keys, const int64_t* __restrict__ offsets,
    const int32_t* __restrict__ processed, const float* __restrict__ slots, long long m,
    const int64_t* __restrict__ m_dev, float* __restrict__ grad2d) {
  const long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (m_dev && *m_dev < m) m = *m_dev;  // rows on the device (capacity launch)
  if (q >= m) return;
  float acc[TSR_GRAD2D_FLOATS];
#pragma unroll
  for (int j = 0; j < TSR_GRAD2D_FLOATS; ++j) acc[j] = 0.f;
  const uint32_t e0 = rank_off[q], c = rank_count[q];
  const int* khi = reinterpret_cast<const int*>(keys) + 1;  // tile = high word
  // 4 pairs in flight per round (independent gathers), summed in order
  for (uint32_t e = e0; e < e0 + c; e += 4) {
    uint32_t k[4];
    int t[4];
    bool ok[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) k[u] = e + u < e0 + c ? inv_perm[e + u] : 0u;
#pragma unroll
    for (int u = 0; u < 4; ++u) t[u] = e + u < e0 + c ? khi[2 * (long long)k[u]] : 0;
#pragma unroll
    for (int u = 0; u < 4; ++u)
      ok[u] = e + u < e0 + c && (long long)k[u] - offsets[t[u]] < processed[t[u]];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (!ok[u]) continue;
      const float2* sl = reinterpret_cast<const float2*>(slots + (long long)k[u] * TSR_GRAD2D_FLOATS);
#pragma unroll
      for (int j = 0; j < TSR_GRAD2D_FLOATS / 2; ++j) {
        const float2 v = sl[j];
        acc[2 * j] += v.x;
        acc[2 * j + 1] += v.y;
      }
    }
  }
  float* dst = grad2d + (long long)rank_row[q] * TSR_GRAD2D_FLOATS;
#pragma unroll
  for (int j = 0; j < TSR_GRAD2D_FLOATS; ++j) dst[j] = acc[j];
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
  auto* k = grad_depth ? render_bwd_kernel<true, false> : render_bwd_kernel<false, false>;
  k<<<tx * ty, kBwdThreads, 0, (cudaStream_t)stream>>>(
      (const float4*)rec, values, offsets, width, height, tx, color, depth, final_T,
      n_considered, ckpt, ckpt_base, grad_color, grad_depth, grad_final_T, grad2d, merges,
      nullptr, nullptr, nullptr, FusedAdamArgs{});
  TSR_CHECK_LAUNCH();
  return TSR_OK;
}

extern "C" int tsr_render_bwd_ordered(const float* rec, const int32_t* values,
                                      const int64_t* offsets, int32_t width, int32_t height,
                                      const float* color, const float* depth,
                                      const float* final_T, const int32_t* n_considered,
                                      const float* ckpt, const int64_t* ckpt_base,
                                      const float* grad_color, const float* grad_depth,
                                      const float* grad_final_T, float* grad2d,
                                      unsigned long long* merges, const int32_t* tile_order,
                                      void* stream) {
  if (width <= 0 || height <= 0 || !grad_color || !merges) return TSR_E_INVALID;
  if (ckpt && !ckpt_base) return TSR_E_INVALID;
  const int tx = tiles_of(width), ty = tiles_of(height);
  auto* k = grad_depth ? render_bwd_kernel<true, false> : render_bwd_kernel<false, false>;
  k<<<tx * ty, kBwdThreads, 0, (cudaStream_t)stream>>>(
      (const float4*)rec, values, offsets, width, height, tx, color, depth, final_T,
      n_considered, ckpt, ckpt_base, grad_color, grad_depth, grad_final_T, grad2d, merges,
      nullptr, nullptr, tile_order, FusedAdamArgs{});
  TSR_CHECK_LAUNCH();
  return TSR_OK;
}

extern "C" int tsr_render_bwd_det(const float* rec, const int32_t* values, const int64_t* offsets,
                                  int32_t width, int32_t height, const float* color,
                                  const float* depth, const float* final_T,
                                  const int32_t* n_considered, const float* ckpt,
                                  const int64_t* ckpt_base, const float* grad_color,
                                  const float* grad_depth, const float* grad_final_T,
                                  unsigned long long* merges, float* slots, int32_t* processed,
                                  const uint32_t* inv_perm, const uint32_t* rank_row,
                                  const uint32_t* rank_count, const uint32_t* rank_off,
                                  const int64_t* keys, int64_t m, const int64_t* m_dev,
                                  float* grad2d, void* stream) {
  if (width <= 0 || height <= 0 || !grad_color || !merges || !slots || !processed ||
      !inv_perm || !rank_row || !rank_count || !rank_off || !keys || m < 0 || !grad2d)
    return TSR_E_INVALID;
  if (ckpt && !ckpt_base) return TSR_E_INVALID;
  const int tx = tiles_of(width), ty = tiles_of(height);
  cudaStream_t s = (cudaStream_t)stream;
  auto* k = grad_depth ? render_bwd_kernel<true, true> : render_bwd_kernel<false, true>;
  k<<<tx * ty, kBwdThreads, 0, s>>>((const float4*)rec, values, offsets, width, height, tx,
                                    color, depth, final_T, n_considered, ckpt, ckpt_base,
                                    grad_color, grad_depth, grad_final_T, nullptr, merges, slots,
                                    processed, nullptr, FusedAdamArgs{});
  TSR_CHECK_LAUNCH();
  if (m > 0) {
    grad_reduce_kernel<<<(int)((m + 255) / 256), 256, 0, s>>>(
        rank_row, rank_count, rank_off, inv_perm, keys, offsets, processed, slots, m, m_dev,
        grad2d);
    TSR_CHECK_LAUNCH();
  }
  return TSR_OK;
}

// ---- work-unit K4 entry points ---------------------------------------------
namespace {
struct UnitWs {
  int32_t* nsup;
  int32_t* n_units;
  int32_t* counter;
  uint32_t* units;
  long long cap;
};

size_t units_cap(int n_tiles, int64_t p_bound) {
  // units = sum_t ceil(min(max n_cons, n_t) / 64) <= P / 64 + n_tiles
  return (size_t)(p_bound > 0 ? p_bound : 0) / kSuper + (size_t)n_tiles + 1;
}

size_t units_ws_bytes(int n_tiles, int64_t p_bound) {
  return ((size_t)n_tiles * 4 + 255) / 256 * 256 + 256 + units_cap(n_tiles, p_bound) * 4;
}

UnitWs carve(void* ws, int n_tiles, int64_t p_bound) {
  UnitWs u;
  char* b = (char*)ws;
  u.nsup = (int32_t*)b;
  b += ((size_t)n_tiles * 4 + 255) / 256 * 256;
  u.n_units = (int32_t*)b;
  u.counter = (int32_t*)(b + 4);
  b += 256;
  u.units = (uint32_t*)b;
  u.cap = (long long)units_cap(n_tiles, p_bound);
  return u;
}

template <bool kDepth, bool kDet>
int launch_units(const float* rec, const int32_t* values, const int64_t* offsets, int width,
                 int height, const float* color, const float* depth, const float* final_T,
                 const int32_t* n_considered, const float* ckpt, const int64_t* ckpt_base,
                 const float* grad_color, const float* grad_depth, const float* grad_final_T,
                 float* grad2d, unsigned long long* merges, float* slots, int32_t* processed,
                 const UnitWs& u, cudaStream_t s) {
  const int tx = tiles_of(width), ty = tiles_of(height), n_tiles = tx * ty;
  unit_count_kernel<<<(n_tiles + 7) / 8, 256, 0, s>>>(offsets, n_considered, width, height, tx,
                                                      n_tiles, u.nsup);
  TSR_CHECK_LAUNCH();
  const size_t plan_smem = n_tiles <= kPlanMaxTiles ? (size_t)n_tiles * sizeof(int) : 0;
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(unit_plan_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         kPlanMaxTiles * (int)sizeof(int));
    attr_set = true;
  }
  unit_plan_kernel<<<1, kPlanThreads, plan_smem, s>>>(u.nsup, n_tiles, u.units, u.cap,
                                                      u.n_units, u.counter, processed);
  TSR_CHECK_LAUNCH();
  auto* k = render_bwd_units_kernel<kDepth, kDet>;
  static int per_sm = 0, sms = 0;  // occupancy of this instantiation (host-side constant)
  if (per_sm == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, kBwdThreads, 0);
    if (per_sm < 1) per_sm = 1;
  }
  k<<<sms * per_sm, kBwdThreads, 0, s>>>((const float4*)rec, values, offsets, width, height, tx,
                                         color, depth, final_T, n_considered, ckpt, ckpt_base,
                                         grad_color, grad_depth, grad_final_T, grad2d, merges,
                                         slots, u.units, u.n_units, u.counter, processed);
  TSR_CHECK_LAUNCH();
  return TSR_OK;
}
}  // namespace

extern "C" size_t tsr_render_bwd_workspace(int32_t width, int32_t height, int64_t p_bound) {
  if (width <= 0 || height <= 0) return 0;
  return units_ws_bytes(tiles_of(width) * tiles_of(height), p_bound);
}

extern "C" int tsr_render_bwd_ws(const float* rec, const int32_t* values, const int64_t* offsets,
                                 int32_t width, int32_t height, const float* color,
                                 const float* depth, const float* final_T,
                                 const int32_t* n_considered, const float* ckpt,
                                 const int64_t* ckpt_base, const float* grad_color,
                                 const float* grad_depth, const float* grad_final_T,
                                 float* grad2d, unsigned long long* merges, int64_t p_bound,
                                 void* workspace, size_t workspace_bytes, void* stream) {
  if (width <= 0 || height <= 0 || !grad_color || !merges || !grad2d || !workspace)
    return TSR_E_INVALID;
  if (ckpt && !ckpt_base) return TSR_E_INVALID;
  const int n_tiles = tiles_of(width) * tiles_of(height);
  if (n_tiles >= (1 << 16)) return TSR_E_INVALID;
  if (workspace_bytes < units_ws_bytes(n_tiles, p_bound)) return TSR_E_WORKSPACE;
  const UnitWs u = carve(workspace, n_tiles, p_bound);
  cudaStream_t s = (cudaStream_t)stream;
  return grad_depth
             ? launch_units<true, false>(rec, values, offsets, width, height, color, depth, final_T,
                                         n_considered, ckpt, ckpt_base, grad_color, grad_depth,
                                         grad_final_T, grad2d, merges, nullptr, nullptr, u, s)
             : launch_units<false, false>(rec, values, offsets, width, height, color, depth,
                                          final_T, n_considered, ckpt, ckpt_base, grad_color,
                                          grad_depth, grad_final_T, grad2d, merges, nullptr,
                                          nullptr, u, s);
}

extern "C" int tsr_render_bwd_ws_det(const float* rec, const int32_t* values,
                                     const int64_t* offsets, int32_t width, int32_t height,
                                     const float* color, const float* depth, const float* final_T,
                                     const int32_t* n_considered, const float* ckpt,
                                     const int64_t* ckpt_base, const float* grad_color,
                                     const float* grad_depth, const float* grad_final_T,
                                     unsigned long long* merges, float* slots, int32_t* processed,
                                     const uint32_t* inv_perm, const uint32_t* rank_row,
                                     const uint32_t* rank_count, const uint32_t* rank_off,
                                     const int64_t* keys, int64_t m, const int64_t* m_dev,
                                     float* grad2d, int64_t p_bound, void* workspace,
                                     size_t workspace_bytes, void* stream) {
  if (width <= 0 || height <= 0 || !grad_color || !merges || !slots || !processed ||
      !inv_perm || !rank_row || !rank_count || !rank_off || !keys || m < 0 || !grad2d ||
      !workspace)
    return TSR_E_INVALID;
  if (ckpt && !ckpt_base) return TSR_E_INVALID;
  const int n_tiles = tiles_of(width) * tiles_of(height);
  if (n_tiles >= (1 << 16)) return TSR_E_INVALID;
  if (workspace_bytes < units_ws_bytes(n_tiles, p_bound)) return TSR_E_WORKSPACE;
  const UnitWs u = carve(workspace, n_tiles, p_bound);
  cudaStream_t s = (cudaStream_t)stream;
  const int rc =
      grad_depth
          ? launch_units<true, true>(rec, values, offsets, width, height, color, depth, final_T,
                                     n_considered, ckpt, ckpt_base, grad_color, grad_depth,
                                     grad_final_T, nullptr, merges, slots, processed, u, s)
          : launch_units<false, true>(rec, values, offsets, width, height, color, depth, final_T,
                                      n_considered, ckpt, ckpt_base, grad_color, grad_depth,
                                      grad_final_T, nullptr, merges, slots, processed, u, s);
  if (rc != TSR_OK) return rc;
  if (m > 0) {
    grad_reduce_kernel<<<(int)((m + 255) / 256), 256, 0, s>>>(
        rank_row, rank_count, rank_off, inv_perm, keys, offsets, processed, slots, m, m_dev,
        grad2d);
    TSR_CHECK_LAUNCH();
  }
  return TSR_OK;
}

extern "C" int tsr_render_bwd_adam(
    const float* rec, const int32_t* values, const int64_t* offsets, int32_t width,
    int32_t height, const float* color, const float* depth, const float* final_T,
    const int32_t* n_considered, const float* ckpt, const int64_t* ckpt_base,
    const float* grad_color, const float* grad_depth, const float* grad_final_T, float* grad2d,
    unsigned long long* merges, const int32_t* tile_order, const tsr_gaussians_t* g,
    const tsr_camera_t* cam, const tsr_adam_group_t* groups_host, const float* group_scalars,
    const int32_t* source_ids, const int32_t* row_of_source, const int32_t* counts,
    int32_t* row_done, unsigned long long* skipped, const int32_t* gate, int32_t* gated_steps,
    const float* loss_guard, void* stream) {
  if (width <= 0 || height <= 0 || !grad_color || !merges || !grad2d || !g || !cam ||
      !source_ids || !row_of_source || !counts || !row_done || !skipped)
    return TSR_E_INVALID;
  if (ckpt && !ckpt_base) return TSR_E_INVALID;
  if (g->sh_coeffs != 1) return TSR_E_INVALID;  // the SH-0 fast path only
  FusedAdamArgs fa{};
  if (!fill_adam_groups(groups_host, 5, fa.groups)) return TSR_E_INVALID;
  for (int k = 0; k < 5; ++k)
    if (fa.groups.g[k].rows != g->n || !fa.groups.g[k].exp_avg || !fa.groups.g[k].exp_avg_sq)
      return TSR_E_INVALID;
  if (fa.groups.g[0].width != 3 || fa.groups.g[1].width != 3 || fa.groups.g[2].width != 4 ||
      fa.groups.g[3].width != 1 || fa.groups.g[4].width != 3)
    return TSR_E_INVALID;
  fa.cam = *cam;
  fa.source_ids = source_ids;
  fa.counts = counts;
  fa.row_done = row_done;
  fa.scal = group_scalars;
  fa.gate = gate;
  fa.loss_guard = loss_guard;
  fa.skipped = skipped;
  const int tx = tiles_of(width), ty = tiles_of(height);
  cudaStream_t s = (cudaStream_t)stream;
  auto* k = grad_depth ? render_bwd_kernel<true, false, true> : render_bwd_kernel<false, false, true>;
  k<<<tx * ty, kBwdThreads, 0, s>>>((const float4*)rec, values, offsets, width, height, tx, color,
                                    depth, final_T, n_considered, ckpt, ckpt_base, grad_color,
                                    grad_depth, grad_final_T, grad2d, merges, nullptr, nullptr,
                                    tile_order, fa);
  TSR_CHECK_LAUNCH();
  return tsr_launch_vjp_adam_rest(*cam, g->n, rec, row_of_source, counts, row_done, grad2d,
                                  fa.groups, skipped, group_scalars, gate, gated_steps,
                                  loss_guard, s);
}
