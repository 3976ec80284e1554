// Fused photometric loss: E = (1 - lam) mean|r - g| + lam (1 - SSIM) and
// dE/dr (losses.py:44-91) -- SURVEY.md §8(f) next #1.
//
// Two tile kernels over 32x32 output tiles (separable 11-tap Gaussian,
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

constexpr int kLT = 32;            // output tile
constexpr int kLR = 5;             // filter radius
constexpr int kLIn = kLT + 2 * kLR;  // 42

// the window travels as a kernel parameter (constant bank): no device globals
struct Win {
  float w[11];
};

__global__ void __launch_bounds__(256) ssim_fwd_kernel(const float* __restrict__ r,
                                                       const float* __restrict__ g, int H, int W,
                                                       float inv_n, float* __restrict__ Q,
                                                       double* __restrict__ partials, Win win) {
  __shared__ float s_r[kLIn][kLIn + 1];
  __shared__ float s_g[kLIn][kLIn + 1];
  __shared__ float s_h[5][kLIn][kLT + 1];
  __shared__ double s_red[2][8];
  const int tid = threadIdx.x;
  const int tx0 = blockIdx.x * kLT, ty0 = blockIdx.y * kLT;
  const long long HW = (long long)H * W;
  double acc_ssim = 0.0, acc_l1 = 0.0;
  for (int c = 0; c < 3; ++c) {
    for (int i = tid; i < kLIn * kLIn; i += 256) {
      const int yy = i / kLIn, xx = i - yy * kLIn;
      const int y = ty0 - kLR + yy, x = tx0 - kLR + xx;
      float rv = 0.f, gv = 0.f;
      if (y >= 0 && y < H && x >= 0 && x < W) {
        const long long p = ((long long)y * W + x) * 3 + c;
        rv = r[p];
        gv = g[p];
      }
      s_r[yy][xx] = rv;
      s_g[yy][xx] = gv;
    }
    __syncthreads();
    for (int i = tid; i < kLIn * kLT; i += 256) {
      const int row = i / kLT, col = i - row * kLT;
      float m1 = 0.f, m2 = 0.f, q11 = 0.f, q22 = 0.f, q12 = 0.f;
#pragma unroll
      for (int k = 0; k < 11; ++k) {
        const float a = s_r[row][col + k], b = s_g[row][col + k], w = win.w[k];
        m1 = fmaf(w, a, m1);
        m2 = fmaf(w, b, m2);
        q11 = fmaf(w, a * a, q11);
        q22 = fmaf(w, b * b, q22);
        q12 = fmaf(w, a * b, q12);
      }
      s_h[0][row][col] = m1;
      s_h[1][row][col] = m2;
      s_h[2][row][col] = q11;
      s_h[3][row][col] = q22;
      s_h[4][row][col] = q12;
    }
    __syncthreads();
    for (int i = tid; i < kLT * kLT; i += 256) {
      const int row = i / kLT, col = i - row * kLT;
      const int y = ty0 + row, x = tx0 + col;
      if (y >= H || x >= W) continue;
      float v[5] = {0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int k = 0; k < 11; ++k) {
        const float w = win.w[k];
#pragma unroll
        for (int q = 0; q < 5; ++q) v[q] = fmaf(w, s_h[q][row + k][col], v[q]);
      }
      const float mu1 = v[0], mu2 = v[1];
      const float s1 = v[2] - mu1 * mu1, s2 = v[3] - mu2 * mu2, s12 = v[4] - mu1 * mu2;
      const float C1 = 0.0001f, C2 = 0.0009f;
      const float A1 = 2.f * mu1 * mu2 + C1, A2 = 2.f * s12 + C2;
      const float B1 = mu1 * mu1 + mu2 * mu2 + C1, B2 = s1 + s2 + C2;
      const float inv_b = 1.0f / (B1 * B2);
      const float map = A1 * A2 * inv_b;
      const float dA1 = inv_n * A2 * inv_b, dA2 = inv_n * A1 * inv_b;
      const float dB1 = -inv_n * map / B1, dB2 = -inv_n * map / B2;
      const long long pix = (long long)y * W + x;
      Q[(c * 3 + 0) * HW + pix] = 2.f * mu2 * (dA1 - dA2) + 2.f * mu1 * (dB1 - dB2);
      Q[(c * 3 + 1) * HW + pix] = dB2;
      Q[(c * 3 + 2) * HW + pix] = 2.f * dA2;
      acc_ssim += (double)map;
      acc_l1 += (double)fabsf(s_r[row + kLR][col + kLR] - s_g[row + kLR][col + kLR]);
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
    double s = 0.0;
    for (int w = 0; w < 8; ++w) s += s_red[tid][w];
    partials[2 * (blockIdx.y * gridDim.x + blockIdx.x) + tid] = s;
  }
}

__global__ void __launch_bounds__(256) ssim_bwd_kernel(const float* __restrict__ r,
                                                       const float* __restrict__ g, int H, int W,
                                                       float lam, float inv_n,
                                                       const float* __restrict__ Q,
                                                       float* __restrict__ grad, Win win) {
  __shared__ float s_q[3][kLIn][kLIn + 1];
  __shared__ float s_h[3][kLIn][kLT + 1];
  const int tid = threadIdx.x;
  const int tx0 = blockIdx.x * kLT, ty0 = blockIdx.y * kLT;
  const long long HW = (long long)H * W;
  for (int c = 0; c < 3; ++c) {
    for (int i = tid; i < kLIn * kLIn; i += 256) {
      const int yy = i / kLIn, xx = i - yy * kLIn;
      const int y = ty0 - kLR + yy, x = tx0 - kLR + xx;
      const bool in = y >= 0 && y < H && x >= 0 && x < W;
      const long long pix = (long long)y * W + x;
#pragma unroll
      for (int q = 0; q < 3; ++q) s_q[q][yy][xx] = in ? Q[(c * 3 + q) * HW + pix] : 0.f;
    }
    __syncthreads();
    for (int i = tid; i < kLIn * kLT; i += 256) {
      const int row = i / kLT, col = i - row * kLT;
      float v[3] = {0.f, 0.f, 0.f};
#pragma unroll
      for (int k = 0; k < 11; ++k) {
        const float w = win.w[k];
#pragma unroll
        for (int q = 0; q < 3; ++q) v[q] = fmaf(w, s_q[q][row][col + k], v[q]);
      }
#pragma unroll
      for (int q = 0; q < 3; ++q) s_h[q][row][col] = v[q];
    }
    __syncthreads();
    for (int i = tid; i < kLT * kLT; i += 256) {
      const int row = i / kLT, col = i - row * kLT;
      const int y = ty0 + row, x = tx0 + col;
      if (y >= H || x >= W) continue;
      float v[3] = {0.f, 0.f, 0.f};
#pragma unroll
      for (int k = 0; k < 11; ++k) {
        const float w = win.w[k];
#pragma unroll
        for (int q = 0; q < 3; ++q) v[q] = fmaf(w, s_h[q][row + k][col], v[q]);
      }
      const long long p = ((long long)y * W + x) * 3 + c;
      const float rv = r[p], gv = g[p];
      const float d = rv - gv;
      const float sgn = d > 0.f ? 1.f : (d < 0.f ? -1.f : 0.f);
      const float gs = v[0] + v[1] * 2.f * rv + v[2] * gv;
      grad[p] = (1.f - lam) * sgn * inv_n - lam * gs;
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
  return q_bytes(height, width) + tiles * 2 * sizeof(double) + 256;
}

extern "C" int tsr_photometric(const float* rendered, const float* gt, int32_t height,
                               int32_t width, float lam, float* grad, float* out3,
                               void* workspace, size_t workspace_bytes, void* stream) {
  if (height <= 0 || width <= 0 || !rendered || !gt || !grad || !out3) return TSR_E_INVALID;
  if (!(lam >= 0.f && lam <= 1.f)) return TSR_E_INVALID;
  if (workspace_bytes < tsr_photometric_workspace(height, width)) return TSR_E_WORKSPACE;
  const Win win = make_window();
  cudaStream_t s = (cudaStream_t)stream;
  dim3 grid((width + kLT - 1) / kLT, (height + kLT - 1) / kLT);
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
