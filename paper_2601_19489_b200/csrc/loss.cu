// Fused photometric loss: E = (1 - lam) mean|r - g| + lam (1 - SSIM) and
// dE/dr (losses.py:44-91) -- SURVEY.md §8(f) next #1.
//
// Two tile kernels over 32x32 output tiles, one CTA per (tile, channel) (separable 11-tap Gaussian,
// sigma 1.5, zero padding, window passed as a kernel parameter):
//   ssim_fwd: per channel, stage r, g (tile + 5-pixel halo) in shared memory,
//             filter the 5 moments (mu1, mu2, E[r^2], E[g^2], E[rg]), form the
//             SSIM map and its three backward sources
//                 g_mu1 = 2 mu2 (dA1 - dA2) + 2 mu1 (dB1 - dB2), g_v1 = dB2,
//                 g_v12 = 2 dA2       (losses.py:59-68, scaled by 1/N)
//             -> planar scratch Q[c][3][H][W]; block partial sums of the map
//             and |r - g| in double.
//   ssim_bwd: filter Q (the filter is symmetric, so its transpose is itself)
//             and combine grad = (1-lam) sign(r-g)/N
//                              - lam (F g_mu1 + 2 r F g_v1 + g F g_v12).
//   finalize: the first CTA of ssim_bwd reduces the forward's block partials
//             (complete when it starts) to (E, l1, ssim) -- no third launch.
#include <cuda_runtime.h>

#include "tsr_common.cuh"

namespace tsr {

#ifndef TSR_SSIM_MINB
#define TSR_SSIM_MINB 4  // 5 (51 registers) measured slower: 70 / 71 us
#endif
constexpr int kLT = 32;              // output tile
constexpr int kLR = 5;               // filter radius
constexpr int kLIn = kLT + 2 * kLR;  // 42 rows/cols incl. halo
constexpr int kLS = 48;              // padded smem row stride (8-B aligned float2 reads)

// the window travels as a kernel parameter (constant bank): no device globals
struct Win {
  float w[11];
};

__device__ __forceinline__ float2 bc2(float x) { return make_float2(x, x); }

// Load a (kLIn x kLIn) halo tile of one channel of the interleaved (H,W,3)
// images r and g (zero outside) into s[row][col] = (r, g) (row stride kLS).
// All loads of a thread are issued before any shared store.
// Row-wise halo loads: warp w stages rows w, w + 8, ... of the 42-row halo;
// lane l loads column l and lanes 0-9 also column 32 + l.  A row's validity
// is warp-uniform and its base address is formed once (no per-element
// division or 64-bit index arithmetic); all loads of a thread are issued
// before any shared store.
constexpr int kHaloRows = (kLIn + 7) / 8;  // rows per warp (6; warps 2-7 load 5)
// The halo lies inside the image for every tile but the frame's border ring
// (CTA-uniform): those load unguarded, from one 32-bit offset per row.
__device__ __forceinline__ bool halo_inside(int H, int W, int ty0, int tx0) {
  return ty0 >= kLR && tx0 >= kLR && ty0 - kLR + kLIn <= H && tx0 - kLR + kLIn <= W;
}
__device__ __forceinline__ void load_halo2(const float* __restrict__ r, const float* __restrict__ g,
                                           int c, int H, int W, int ty0, int tx0, float2* s) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int x0 = tx0 - kLR + lane, x1 = x0 + 32;
  float2 v0[kHaloRows], v1[kHaloRows];
  if (halo_inside(H, W, ty0, tx0)) {
    const float* rb = r + ((long long)(ty0 - kLR) * W + x0) * 3 + c;
    const float* gb = g + ((long long)(ty0 - kLR) * W + x0) * 3 + c;
    const bool two = lane < kLIn - 32;
#pragma unroll
    for (int k = 0; k < kHaloRows; ++k) {
      const int row = warp + 8 * k;
      const int o = row * 3 * W;  // < 2^31 for frames below ~700 Mpixel
      v0[k] = v1[k] = make_float2(0.f, 0.f);
      if (row < kLIn) {
        v0[k] = make_float2(__ldg(rb + o), __ldg(gb + o));
        if (two) v1[k] = make_float2(__ldg(rb + o + 96), __ldg(gb + o + 96));
      }
    }
  } else {
    const bool in0 = x0 >= 0 && x0 < W, in1 = lane < kLIn - 32 && x1 >= 0 && x1 < W;
#pragma unroll
    for (int k = 0; k < kHaloRows; ++k) {
      const int row = warp + 8 * k;
      const int y = ty0 - kLR + row;
      v0[k] = v1[k] = make_float2(0.f, 0.f);
      if (row < kLIn && y >= 0 && y < H) {
        const float* rr = r + ((long long)y * W) * 3 + c;
        const float* gg = g + ((long long)y * W) * 3 + c;
        if (in0) v0[k] = make_float2(__ldg(rr + 3 * x0), __ldg(gg + 3 * x0));
        if (in1) v1[k] = make_float2(__ldg(rr + 3 * x1), __ldg(gg + 3 * x1));
      }
    }
  }
#pragma unroll
  for (int k = 0; k < kHaloRows; ++k) {
    const int row = warp + 8 * k;
    if (row < kLIn) {
      s[row * kLS + lane] = v0[k];
      if (lane < kLIn - 32) s[row * kLS + 32 + lane] = v1[k];
    }
  }
}

// The two images (and in the backward the first two SSIM sources) travel as
// one packed FP32x2 pair through both filter passes: each tap is one FFMA2
// for (mu1, mu2), one for (E[r^2], E[g^2]) and one scalar FFMA for E[rg]
// (5 FFMA before); every lane of a packed op is an IEEE FMA, so the sums are
// bit-identical to the scalar form.
__global__ void __launch_bounds__(256, TSR_SSIM_MINB) ssim_fwd_kernel(const float* __restrict__ r,
                                                       const float* __restrict__ g, int H, int W,
                                                       float inv_n, float2* __restrict__ Q01,
                                                       float* __restrict__ Q2,
                                                       double* __restrict__ partials, Win win) {
  __shared__ __align__(16) float2 s_rg[kLIn * kLS];
  __shared__ __align__(16) float2 s_h2[2][kLIn][kLT + 1];  // (mu1, mu2), (E11, E22)
  __shared__ float s_h1[kLIn][kLT + 1];                    // E12
  __shared__ double s_red[2][8];
  const int tid = threadIdx.x;
  // one CTA per (tile, channel); the 3 channel CTAs of a tile are adjacent
  // in launch order, so the interleaved image sectors are shared in L2
  const int c = blockIdx.x % 3;
  const int tx0 = (blockIdx.x / 3) * kLT, ty0 = blockIdx.y * kLT;
  const long long HW = (long long)H * W;
  double acc_ssim = 0.0, acc_l1 = 0.0;
  float f_ssim = 0.f, f_l1 = 0.f;  // this thread's 4 pixels, widened once
  {
    load_halo2(r, g, c, H, W, ty0, tx0, s_rg);
    __syncthreads();
    // horizontal: item = (row, 2 consecutive output cols); 42 x 16 items
    for (int it = tid; it < kLIn * (kLT / 2); it += 256) {
      const int row = it >> 4, c0 = (it & 15) * 2;
      float2 ab[12];
      {
        const float4* pr = reinterpret_cast<const float4*>(s_rg + row * kLS + c0);
#pragma unroll
        for (int k = 0; k < 6; ++k) {
          const float4 x = pr[k];
          ab[2 * k] = make_float2(x.x, x.y);
          ab[2 * k + 1] = make_float2(x.z, x.w);
        }
      }
      float2 m[2] = {bc2(0.f), bc2(0.f)}, q[2] = {bc2(0.f), bc2(0.f)};
      float q12[2] = {0.f, 0.f};
#pragma unroll
      for (int k = 0; k < 12; ++k) {
        const float2 sq = __fmul2_rn(ab[k], ab[k]);
        const float p = __fmul_rn(ab[k].x, ab[k].y);
#pragma unroll
        for (int o = 0; o < 2; ++o) {
          const int tap = k - o;
          if (tap >= 0 && tap < 11) {
            const float w = win.w[tap];
            m[o] = __ffma2_rn(bc2(w), ab[k], m[o]);
            q[o] = __ffma2_rn(bc2(w), sq, q[o]);
            q12[o] = fmaf(w, p, q12[o]);
          }
        }
      }
#pragma unroll
      for (int o = 0; o < 2; ++o) {
        s_h2[0][row][c0 + o] = m[o];
        s_h2[1][row][c0 + o] = q[o];
        s_h1[row][c0 + o] = q12[o];
      }
    }
    __syncthreads();
    // vertical: item = (col, 4 consecutive output rows); 32 x 8 items = 256
    {
      const int col = tid & 31, r0 = (tid >> 5) * 4;
      float2 vm[4], vq[4];
      float v12[4];
#pragma unroll
      for (int o = 0; o < 4; ++o) {
        vm[o] = vq[o] = bc2(0.f);
        v12[o] = 0.f;
      }
#pragma unroll
      for (int k = 0; k < 14; ++k) {
        const float2 hm = s_h2[0][r0 + k][col], hq = s_h2[1][r0 + k][col];
        const float h12 = s_h1[r0 + k][col];
#pragma unroll
        for (int o = 0; o < 4; ++o) {
          const int tap = k - o;
          if (tap >= 0 && tap < 11) {
            const float w = win.w[tap];
            vm[o] = __ffma2_rn(bc2(w), hm, vm[o]);
            vq[o] = __ffma2_rn(bc2(w), hq, vq[o]);
            v12[o] = fmaf(w, h12, v12[o]);
          }
        }
      }
      const float C1 = 0.0001f, C2 = 0.0009f;
#pragma unroll
      for (int o = 0; o < 4; ++o) {
        const int y = ty0 + r0 + o, x = tx0 + col;
        if (y >= H || x >= W) continue;
        const float mu1 = vm[o].x, mu2 = vm[o].y;
        const float s1 = vq[o].x - mu1 * mu1, s2 = vq[o].y - mu2 * mu2, s12 = v12[o] - mu1 * mu2;
        const float A1 = 2.f * mu1 * mu2 + C1, A2 = 2.f * s12 + C2;
        const float B1 = mu1 * mu1 + mu2 * mu2 + C1, B2 = s1 + s2 + C2;
        const float inv_b = 1.0f / (B1 * B2);
        const float map = A1 * A2 * inv_b;
        const float dA1 = inv_n * A2 * inv_b, dA2 = inv_n * A1 * inv_b;
        const float dB1 = -inv_n * map * (B2 * inv_b), dB2 = -inv_n * map * (B1 * inv_b);
        const long long pix = (long long)y * W + x;
        Q01[c * HW + pix] = make_float2(2.f * mu2 * (dA1 - dA2) + 2.f * mu1 * (dB1 - dB2), dB2);
        Q2[c * HW + pix] = 2.f * dA2;
        f_ssim += map;
        const float2 rg = s_rg[(r0 + o + kLR) * kLS + col + kLR];
        f_l1 += fabsf(rg.x - rg.y);
      }
      acc_ssim = (double)f_ssim;
      acc_l1 = (double)f_l1;
    }
    __syncthreads();
  }
  // block reduce the two partial sums
  const int lane = tid & 31, warp = tid >> 5;
  for (int d = 16; d > 0; d >>= 1) {
    acc_ssim += __shfl_xor_sync(0xffffffffu, acc_ssim, d);
    acc_l1 += __shfl_xor_sync(0xffffffffu, acc_l1, d);
  }
  if (lane == 0) {
    s_red[0][warp] = acc_ssim;
    s_red[1][warp] = acc_l1;
  }
  __syncthreads();
  if (tid < 2) {
    double sum = 0.0;
    for (int w = 0; w < 8; ++w) sum += s_red[tid][w];
    partials[2 * (blockIdx.y * gridDim.x + blockIdx.x) + tid] = sum;
  }
}

// (E, l1, ssim) from the forward's block partials, in a fixed order (the
// first CTA of ssim_bwd runs it: the partials are complete when it starts).
__device__ void loss_finalize(const double* __restrict__ partials, int n_blocks, double inv_n,
                              float lam, float* __restrict__ out) {
  __shared__ double s[2][8];
  double a = 0.0, b = 0.0;
  constexpr int kU = 8;
  for (int i0 = threadIdx.x; i0 < n_blocks; i0 += 256 * kU) {
    double2 v[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int i = i0 + 256 * u;
      v[u] = i < n_blocks ? reinterpret_cast<const double2*>(partials)[i] : make_double2(0.0, 0.0);
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      a += v[u].x;
      b += v[u].y;
    }
  }
  for (int d = 16; d > 0; d >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, d);
    b += __shfl_xor_sync(0xffffffffu, b, d);
  }
  if ((threadIdx.x & 31) == 0) {
    s[0][threadIdx.x >> 5] = a;
    s[1][threadIdx.x >> 5] = b;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double ss = 0.0, l1 = 0.0;
    for (int w = 0; w < 8; ++w) {
      ss += s[0][w];
      l1 += s[1][w];
    }
    ss *= inv_n;
    l1 *= inv_n;
    out[0] = (float)((1.0 - lam) * l1 + lam * (1.0 - ss));
    out[1] = (float)l1;
    out[2] = (float)ss;
  }
}

__global__ void __launch_bounds__(256, TSR_SSIM_MINB) ssim_bwd_kernel(
    const float* __restrict__ r, const float* __restrict__ g, int H, int W, float lam,
    float inv_n, const float2* __restrict__ Q01, const float* __restrict__ Q2,
    float* __restrict__ grad, Win win, const double* __restrict__ partials, int n_blocks,
    double inv_n_d, float* __restrict__ out3) {
  __shared__ __align__(16) float2 s_q2[kLIn * kLS];
  __shared__ __align__(16) float s_q1[kLIn * kLS];
  __shared__ float2 s_h2[kLIn][kLT + 1];
  __shared__ float s_h1[kLIn][kLT + 1];
  const int tid = threadIdx.x;
  const int c = blockIdx.x % 3;
  const int tx0 = (blockIdx.x / 3) * kLT, ty0 = blockIdx.y * kLT;
  const long long HW = (long long)H * W;
  if (blockIdx.x == 0 && blockIdx.y == 0)
    loss_finalize(partials, n_blocks, inv_n_d, lam, out3);
  // the epilogue's r, g values: loads issued now, consumed after the filters
  const int col = tid & 31, r0 = (tid >> 5) * 4;
  float rv[4], gv[4];
#pragma unroll
  for (int o = 0; o < 4; ++o) {
    const int y = ty0 + r0 + o, x = tx0 + col;
    const bool in = y < H && x < W;
    const long long p = ((long long)y * W + x) * 3 + c;
    rv[o] = in ? __ldg(r + p) : 0.f;
    gv[o] = in ? __ldg(g + p) : 0.f;
  }
  {
    // row-wise halo of the planar SSIM sources (see load_halo2)
    {
      const int lane = tid & 31, warp = tid >> 5;
      const int x0 = tx0 - kLR + lane, x1 = x0 + 32;
      float2 v2a[kHaloRows], v2b[kHaloRows];
      float v1a[kHaloRows], v1b[kHaloRows];
      if (halo_inside(H, W, ty0, tx0)) {  // unguarded, one 32-bit offset per row
        const float2* qa = Q01 + c * HW + (long long)(ty0 - kLR) * W + x0;
        const float* qb = Q2 + c * HW + (long long)(ty0 - kLR) * W + x0;
        const bool two = lane < kLIn - 32;
#pragma unroll
        for (int k = 0; k < kHaloRows; ++k) {
          const int row = warp + 8 * k;
          const int o = row * W;
          v2a[k] = v2b[k] = bc2(0.f);
          v1a[k] = v1b[k] = 0.f;
          if (row < kLIn) {
            v2a[k] = __ldg(qa + o);
            v1a[k] = __ldg(qb + o);
            if (two) {
              v2b[k] = __ldg(qa + o + 32);
              v1b[k] = __ldg(qb + o + 32);
            }
          }
        }
      } else {
        const bool in0 = x0 >= 0 && x0 < W, in1 = lane < kLIn - 32 && x1 >= 0 && x1 < W;
#pragma unroll
        for (int k = 0; k < kHaloRows; ++k) {
          const int row = warp + 8 * k;
          const int y = ty0 - kLR + row;
          v2a[k] = v2b[k] = bc2(0.f);
          v1a[k] = v1b[k] = 0.f;
          if (row < kLIn && y >= 0 && y < H) {
            const long long o = c * HW + (long long)y * W;
            if (in0) {
              v2a[k] = __ldg(Q01 + o + x0);
              v1a[k] = __ldg(Q2 + o + x0);
            }
            if (in1) {
              v2b[k] = __ldg(Q01 + o + x1);
              v1b[k] = __ldg(Q2 + o + x1);
            }
          }
        }
      }
#pragma unroll
      for (int k = 0; k < kHaloRows; ++k) {
        const int row = warp + 8 * k;
        if (row < kLIn) {
          s_q2[row * kLS + lane] = v2a[k];
          s_q1[row * kLS + lane] = v1a[k];
          if (lane < kLIn - 32) {
            s_q2[row * kLS + 32 + lane] = v2b[k];
            s_q1[row * kLS + 32 + lane] = v1b[k];
          }
        }
      }
    }
    __syncthreads();
    for (int it = tid; it < kLIn * (kLT / 2); it += 256) {
      const int row = it >> 4, c0 = (it & 15) * 2;
      float2 a2[12];
      float a1[12];
      {
        const float4* p2 = reinterpret_cast<const float4*>(s_q2 + row * kLS + c0);
        const float2* p1 = reinterpret_cast<const float2*>(s_q1 + row * kLS + c0);
#pragma unroll
        for (int k = 0; k < 6; ++k) {
          const float4 x = p2[k];
          const float2 y = p1[k];
          a2[2 * k] = make_float2(x.x, x.y);
          a2[2 * k + 1] = make_float2(x.z, x.w);
          a1[2 * k] = y.x;
          a1[2 * k + 1] = y.y;
        }
      }
      float2 h2[2] = {bc2(0.f), bc2(0.f)};
      float h1[2] = {0.f, 0.f};
#pragma unroll
      for (int k = 0; k < 12; ++k)
#pragma unroll
        for (int o = 0; o < 2; ++o) {
          const int tap = k - o;
          if (tap >= 0 && tap < 11) {
            h2[o] = __ffma2_rn(bc2(win.w[tap]), a2[k], h2[o]);
            h1[o] = fmaf(win.w[tap], a1[k], h1[o]);
          }
        }
#pragma unroll
      for (int o = 0; o < 2; ++o) {
        s_h2[row][c0 + o] = h2[o];
        s_h1[row][c0 + o] = h1[o];
      }
    }
    __syncthreads();
    {
      float2 v2o[4];
      float v1o[4];
#pragma unroll
      for (int o = 0; o < 4; ++o) {
        v2o[o] = bc2(0.f);
        v1o[o] = 0.f;
      }
#pragma unroll
      for (int k = 0; k < 14; ++k) {
        const float2 h2 = s_h2[r0 + k][col];
        const float h1 = s_h1[r0 + k][col];
#pragma unroll
        for (int o = 0; o < 4; ++o) {
          const int tap = k - o;
          if (tap >= 0 && tap < 11) {
            v2o[o] = __ffma2_rn(bc2(win.w[tap]), h2, v2o[o]);
            v1o[o] = fmaf(win.w[tap], h1, v1o[o]);
          }
        }
      }
#pragma unroll
      for (int o = 0; o < 4; ++o) {
        const int y = ty0 + r0 + o, x = tx0 + col;
        if (y >= H || x >= W) continue;
        const long long p = ((long long)y * W + x) * 3 + c;
        const float d = rv[o] - gv[o];
        const float sgn = d > 0.f ? 1.f : (d < 0.f ? -1.f : 0.f);
        const float gs = v2o[o].x + v2o[o].y * 2.f * rv[o] + v1o[o] * gv[o];
        grad[p] = (1.f - lam) * sgn * inv_n - lam * gs;
      }
    }
  }
}

static Win make_window() {
  // 11-tap Gaussian, sigma 1.5, normalised (losses.py:21-22), computed in FP64
  double w[11], sum = 0.0;
  for (int k = 0; k < 11; ++k) {
    w[k] = exp(-((k - 5.0) * (k - 5.0)) / (2.0 * 1.5 * 1.5));
    sum += w[k];
  }
  Win out;
  for (int k = 0; k < 11; ++k) out.w[k] = (float)(w[k] / sum);
  return out;
}

}  // namespace tsr

using namespace tsr;

static size_t q_bytes(int32_t height, int32_t width) {
  // planar SSIM sources, rounded up so the double partials stay 256-B aligned
  return ((9 * (size_t)height * width * sizeof(float)) + 255) & ~(size_t)255;
}

extern "C" size_t tsr_photometric_workspace(int32_t height, int32_t width) {
  const size_t tiles = (size_t)((width + kLT - 1) / kLT) * ((height + kLT - 1) / kLT);
  return q_bytes(height, width) + 3 * tiles * 2 * sizeof(double) + 256;
}

extern "C" int tsr_photometric(const float* rendered, const float* gt, int32_t height,
                               int32_t width, float lam, float* grad, float* out3,
                               void* workspace, size_t workspace_bytes, void* stream) {
  if (height <= 0 || width <= 0 || !rendered || !gt || !grad || !out3) return TSR_E_INVALID;
  if (!(lam >= 0.f && lam <= 1.f)) return TSR_E_INVALID;
  if (workspace_bytes < tsr_photometric_workspace(height, width)) return TSR_E_WORKSPACE;
  const Win win = make_window();
  cudaStream_t s = (cudaStream_t)stream;
  dim3 grid(3 * ((width + kLT - 1) / kLT), (height + kLT - 1) / kLT);
  const int n_blocks = grid.x * grid.y;
  float* Q = (float*)workspace;  // planar (Q0, Q1) pairs [3][H][W] + Q2 [3][H][W]
  float2* Q01 = reinterpret_cast<float2*>(Q);
  float* Q2 = Q + 6 * (size_t)height * width;
  double* partials = (double*)((char*)workspace + q_bytes(height, width));
  const double n = 3.0 * (double)height * width;
  ssim_fwd_kernel<<<grid, 256, 0, s>>>(rendered, gt, height, width, (float)(1.0 / n), Q01, Q2,
                                       partials, win);
  TSR_CHECK_LAUNCH();
  ssim_bwd_kernel<<<grid, 256, 0, s>>>(rendered, gt, height, width, lam, (float)(1.0 / n), Q01,
                                       Q2, grad, win, partials, n_blocks, 1.0 / n, out3);
  TSR_CHECK_LAUNCH();
  return TSR_OK;
}
