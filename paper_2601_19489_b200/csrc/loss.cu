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
//   finalize: one block reduces the partials to (E, l1, ssim).
#include <cuda_runtime.h>

#include "tsr_common.cuh"

namespace tsr {

constexpr int kLT = 32;              // output tile
constexpr int kLR = 5;               // filter radius
constexpr int kLIn = kLT + 2 * kLR;  // 42 rows/cols incl. halo
constexpr int kLS = 48;              // padded smem row stride (8-B aligned float2 reads)

// the window travels as a kernel parameter (constant bank): no device globals
struct Win {
  float w[11];
};

// Load a (kLIn x kLIn) halo tile of one channel of an interleaved (H,W,3)
// image (zero outside) into s[row][col] (row stride kLS).
// All (up to 7) loads of a thread are issued before any shared store.
constexpr int kHaloIters = (kLIn * kLIn + 255) / 256;
__device__ __forceinline__ void load_halo(const float* __restrict__ img, int c, int H, int W,
                                          int ty0, int tx0, float* s) {
  float v[kHaloIters];
  int dst[kHaloIters];
#pragma unroll
  for (int k = 0; k < kHaloIters; ++k) {
    const int i = threadIdx.x + 256 * k;
    const int yy = i / kLIn, xx = i - yy * kLIn;
    const int y = ty0 - kLR + yy, x = tx0 - kLR + xx;
    v[k] = 0.f;
    dst[k] = i < kLIn * kLIn ? yy * kLS + xx : -1;
    if (i < kLIn * kLIn && y >= 0 && y < H && x >= 0 && x < W)
      v[k] = __ldg(img + ((long long)y * W + x) * 3 + c);
  }
#pragma unroll
  for (int k = 0; k < kHaloIters; ++k)
    if (dst[k] >= 0) s[dst[k]] = v[k];
}

__global__ void __launch_bounds__(256, 4) ssim_fwd_kernel(const float* __restrict__ r,
                                                       const float* __restrict__ g, int H, int W,
                                                       float inv_n, float* __restrict__ Q,
                                                       double* __restrict__ partials, Win win) {
  __shared__ __align__(16) float s_r[kLIn * kLS];
  __shared__ __align__(16) float s_g[kLIn * kLS];
  __shared__ float s_h[5][kLIn][kLT + 1];
  __shared__ double s_red[2][8];
  const int tid = threadIdx.x;
  // one CTA per (tile, channel); the 3 channel CTAs of a tile are adjacent
  // in launch order, so the interleaved image sectors are shared in L2
  const int c = blockIdx.x % 3;
  const int tx0 = (blockIdx.x / 3) * kLT, ty0 = blockIdx.y * kLT;
  const long long HW = (long long)H * W;
  double acc_ssim = 0.0, acc_l1 = 0.0;
  {
    load_halo(r, c, H, W, ty0, tx0, s_r);
    load_halo(g, c, H, W, ty0, tx0, s_g);
    __syncthreads();
    // horizontal: item = (row, 2 consecutive output cols); 42 x 16 items
    for (int it = tid; it < kLIn * (kLT / 2); it += 256) {
      const int row = it >> 4, c0 = (it & 15) * 2;
      float a[12], b[12];
      {
        const float2* pr = reinterpret_cast<const float2*>(s_r + row * kLS + c0);
        const float2* pg = reinterpret_cast<const float2*>(s_g + row * kLS + c0);
#pragma unroll
        for (int k = 0; k < 6; ++k) {
          const float2 x = pr[k], y = pg[k];
          a[2 * k] = x.x; a[2 * k + 1] = x.y;
          b[2 * k] = y.x; b[2 * k + 1] = y.y;
        }
      }
      float m1[2] = {0, 0}, m2[2] = {0, 0}, q11[2] = {0, 0}, q22[2] = {0, 0}, q12[2] = {0, 0};
#pragma unroll
      for (int k = 0; k < 12; ++k) {
        const float ak = a[k], bk = b[k], aa = ak * ak, bb = bk * bk, ab = ak * bk;
#pragma unroll
        for (int o = 0; o < 2; ++o) {
          const int tap = k - o;
          if (tap >= 0 && tap < 11) {
            const float w = win.w[tap];
            m1[o] = fmaf(w, ak, m1[o]);
            m2[o] = fmaf(w, bk, m2[o]);
            q11[o] = fmaf(w, aa, q11[o]);
            q22[o] = fmaf(w, bb, q22[o]);
            q12[o] = fmaf(w, ab, q12[o]);
          }
        }
      }
#pragma unroll
      for (int o = 0; o < 2; ++o) {
        s_h[0][row][c0 + o] = m1[o];
        s_h[1][row][c0 + o] = m2[o];
        s_h[2][row][c0 + o] = q11[o];
        s_h[3][row][c0 + o] = q22[o];
        s_h[4][row][c0 + o] = q12[o];
      }
    }
    __syncthreads();
    // vertical: item = (col, 4 consecutive output rows); 32 x 8 items = 256
    {
      const int col = tid & 31, r0 = (tid >> 5) * 4;
      float v[5][4];
#pragma unroll
      for (int q = 0; q < 5; ++q)
#pragma unroll
        for (int o = 0; o < 4; ++o) v[q][o] = 0.f;
#pragma unroll
      for (int k = 0; k < 14; ++k) {
#pragma unroll
        for (int q = 0; q < 5; ++q) {
          const float h = s_h[q][r0 + k][col];
#pragma unroll
          for (int o = 0; o < 4; ++o) {
            const int tap = k - o;
            if (tap >= 0 && tap < 11) v[q][o] = fmaf(win.w[tap], h, v[q][o]);
          }
        }
      }
      const float C1 = 0.0001f, C2 = 0.0009f;
#pragma unroll
      for (int o = 0; o < 4; ++o) {
        const int y = ty0 + r0 + o, x = tx0 + col;
        if (y >= H || x >= W) continue;
        const float mu1 = v[0][o], mu2 = v[1][o];
        const float s1 = v[2][o] - mu1 * mu1, s2 = v[3][o] - mu2 * mu2, s12 = v[4][o] - mu1 * mu2;
        const float A1 = 2.f * mu1 * mu2 + C1, A2 = 2.f * s12 + C2;
        const float B1 = mu1 * mu1 + mu2 * mu2 + C1, B2 = s1 + s2 + C2;
        const float inv_b = 1.0f / (B1 * B2);
        const float map = A1 * A2 * inv_b;
        const float dA1 = inv_n * A2 * inv_b, dA2 = inv_n * A1 * inv_b;
        const float dB1 = -inv_n * map * (B2 * inv_b), dB2 = -inv_n * map * (B1 * inv_b);
        const long long pix = (long long)y * W + x;
        Q[(c * 3 + 0) * HW + pix] = 2.f * mu2 * (dA1 - dA2) + 2.f * mu1 * (dB1 - dB2);
        Q[(c * 3 + 1) * HW + pix] = dB2;
        Q[(c * 3 + 2) * HW + pix] = 2.f * dA2;
        acc_ssim += (double)map;
        const int yy = r0 + o + kLR, xx = col + kLR;
        acc_l1 += (double)fabsf(s_r[yy * kLS + xx] - s_g[yy * kLS + xx]);
      }
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

__global__ void __launch_bounds__(256, 4) ssim_bwd_kernel(const float* __restrict__ r,
                                                       const float* __restrict__ g, int H, int W,
                                                       float lam, float inv_n,
                                                       const float* __restrict__ Q,
                                                       float* __restrict__ grad, Win win) {
  __shared__ __align__(16) float s_q[3][kLIn * kLS];
  __shared__ float s_h[3][kLIn][kLT + 1];
  const int tid = threadIdx.x;
  const int c = blockIdx.x % 3;
  const int tx0 = (blockIdx.x / 3) * kLT, ty0 = blockIdx.y * kLT;
  const long long HW = (long long)H * W;
  {
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      float v[kHaloIters];
      int dst[kHaloIters];
#pragma unroll
      for (int k = 0; k < kHaloIters; ++k) {
        const int i = tid + 256 * k;
        const int yy = i / kLIn, xx = i - yy * kLIn;
        const int y = ty0 - kLR + yy, x = tx0 - kLR + xx;
        v[k] = 0.f;
        dst[k] = i < kLIn * kLIn ? yy * kLS + xx : -1;
        if (i < kLIn * kLIn && y >= 0 && y < H && x >= 0 && x < W)
          v[k] = __ldg(Q + (c * 3 + q) * HW + (long long)y * W + x);
      }
#pragma unroll
      for (int k = 0; k < kHaloIters; ++k)
        if (dst[k] >= 0) s_q[q][dst[k]] = v[k];
    }
    __syncthreads();
    for (int it = tid; it < kLIn * (kLT / 2); it += 256) {
      const int row = it >> 4, c0 = (it & 15) * 2;
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        float a[12];
        const float2* pq = reinterpret_cast<const float2*>(s_q[q] + row * kLS + c0);
#pragma unroll
        for (int k = 0; k < 6; ++k) {
          const float2 x = pq[k];
          a[2 * k] = x.x; a[2 * k + 1] = x.y;
        }
        float h[2] = {0, 0};
#pragma unroll
        for (int k = 0; k < 12; ++k)
#pragma unroll
          for (int o = 0; o < 2; ++o) {
            const int tap = k - o;
            if (tap >= 0 && tap < 11) h[o] = fmaf(win.w[tap], a[k], h[o]);
          }
#pragma unroll
        for (int o = 0; o < 2; ++o) s_h[q][row][c0 + o] = h[o];
      }
    }
    __syncthreads();
    {
      const int col = tid & 31, r0 = (tid >> 5) * 4;
      float v[3][4];
#pragma unroll
      for (int q = 0; q < 3; ++q)
#pragma unroll
        for (int o = 0; o < 4; ++o) v[q][o] = 0.f;
#pragma unroll
      for (int k = 0; k < 14; ++k)
#pragma unroll
        for (int q = 0; q < 3; ++q) {
          const float h = s_h[q][r0 + k][col];
#pragma unroll
          for (int o = 0; o < 4; ++o) {
            const int tap = k - o;
            if (tap >= 0 && tap < 11) v[q][o] = fmaf(win.w[tap], h, v[q][o]);
          }
        }
#pragma unroll
      for (int o = 0; o < 4; ++o) {
        const int y = ty0 + r0 + o, x = tx0 + col;
        if (y >= H || x >= W) continue;
        const long long p = ((long long)y * W + x) * 3 + c;
        const float rv = r[p], gv = g[p];
        const float d = rv - gv;
        const float sgn = d > 0.f ? 1.f : (d < 0.f ? -1.f : 0.f);
        const float gs = v[0][o] + v[1][o] * 2.f * rv + v[2][o] * gv;
        grad[p] = (1.f - lam) * sgn * inv_n - lam * gs;
      }
    }
    __syncthreads();
  }
}

__global__ void __launch_bounds__(256) loss_finalize_kernel(const double* __restrict__ partials,
                                                            int n_blocks, double inv_n,
                                                            float lam, float* __restrict__ out) {
  __shared__ double s[2][8];
  double a = 0.0, b = 0.0;
  for (int i = threadIdx.x; i < n_blocks; i += 256) {
    a += partials[2 * i];
    b += partials[2 * i + 1];
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
  float* Q = (float*)workspace;
  double* partials = (double*)((char*)workspace + q_bytes(height, width));
  const double n = 3.0 * (double)height * width;
  ssim_fwd_kernel<<<grid, 256, 0, s>>>(rendered, gt, height, width, (float)(1.0 / n), Q,
                                       partials, win);
  TSR_CHECK_LAUNCH();
  ssim_bwd_kernel<<<grid, 256, 0, s>>>(rendered, gt, height, width, lam, (float)(1.0 / n), Q,
                                       grad, win);
  TSR_CHECK_LAUNCH();
  loss_finalize_kernel<<<1, 256, 0, s>>>(partials, n_blocks, 1.0 / n, lam, out3);
  TSR_CHECK_LAUNCH();
  return TSR_OK;
}
