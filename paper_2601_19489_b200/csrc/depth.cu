// Depth supervision chain of the training step (second
// half): the disparity loss on the normalised render depth and its chain
// back to the raster outputs (trainer.py:201-214, losses.py:94-112):
//   mask   = n_contrib > 0 [& valid]
//   d      = D / (1 - T_f)                       (normalized_depth)
//   diff   = 1 / max(d, eps) - 1 / max(prior, eps)
//   L      = w * mean_mask |diff|                (0 when the mask is empty)
//   g      = w sign(diff) (-1 / max(d, eps)^2) / n_mask, 0 where d < eps
//   dL/dD  = g / (1 - T_f),  dL/dT_f = g D / (1 - T_f)^2     (mask only)
// Two kernels: a reduction (per-block partial |diff| sums and mask counts,
// the last block reducing them in a fixed order -> loss, 1 / n_mask) and the
// per-pixel gradients.  Replaces ~15 elementwise torch ops + two host-free
// reductions; the weight may come from device memory (CUDA-graph replay).
#include <cuda_runtime.h>

#include "tsr_common.cuh"

namespace tsr {

constexpr float kDispEps = 1e-4f;  // DISPARITY_EPS (losses.py:19)
constexpr int kDcThreads = 256;
constexpr int kDcBlocks = 148 * 4;

struct DcWs {
  double sum[kDcBlocks];
  unsigned int cnt[kDcBlocks];
  unsigned int ticket;
  float scale;  // w / n_mask (0 when the mask is empty)
};

__device__ __forceinline__ bool dc_diff(long long p, const float* depth, const float* final_T,
                                        const int32_t* n_contrib, const float* prior,
                                        const uint8_t* valid, float& d, float& dr, float& diff) {
  const bool m = n_contrib[p] > 0 && (!valid || valid[p]);
  if (!m) return false;
  d = depth[p] / (1.0f - final_T[p]);
  dr = fmaxf(d, kDispEps);
  const float dp = fmaxf(prior[p], kDispEps);
  diff = 1.0f / dr - 1.0f / dp;
  return true;
}

__global__ void __launch_bounds__(kDcThreads) depth_chain_reduce_kernel(
    const float* __restrict__ depth, const float* __restrict__ final_T,
    const int32_t* __restrict__ n_contrib, const float* __restrict__ prior,
    const uint8_t* __restrict__ valid, long long n, float weight,
    const float* __restrict__ weight_dev, const float* __restrict__ e_photo,
    float* __restrict__ loss_out, float* __restrict__ total_out, DcWs* __restrict__ ws) {
  __shared__ double s_sum[kDcThreads / 32];
  __shared__ unsigned int s_cnt[kDcThreads / 32];
  __shared__ bool s_last;
  double sum = 0.0;
  unsigned int cnt = 0;
  for (long long p = (long long)blockIdx.x * kDcThreads + threadIdx.x; p < n;
       p += (long long)gridDim.x * kDcThreads) {
    float d, dr, diff;
    if (dc_diff(p, depth, final_T, n_contrib, prior, valid, d, dr, diff)) {
      sum += fabsf(diff);
      ++cnt;
    }
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int k = 16; k > 0; k >>= 1) {
    sum += __shfl_xor_sync(0xffffffffu, sum, k);
    cnt += __shfl_xor_sync(0xffffffffu, cnt, k);
  }
  if (lane == 0) {
    s_sum[warp] = sum;
    s_cnt[warp] = cnt;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double bs = 0.0;
    unsigned int bc = 0;
    for (int w = 0; w < kDcThreads / 32; ++w) {
      bs += s_sum[w];
      bc += s_cnt[w];
    }
    ws->sum[blockIdx.x] = bs;
    ws->cnt[blockIdx.x] = bc;
    __threadfence();
    s_last = atomicAdd(&ws->ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!s_last || threadIdx.x != 0) return;
  // the last block: fixed-order reduction of the partials
  __threadfence();
  double tot = 0.0;
  unsigned long long nm = 0;
  for (unsigned int b = 0; b < gridDim.x; ++b) {
    tot += ((volatile double*)ws->sum)[b];
    nm += ((volatile unsigned int*)ws->cnt)[b];
  }
  const float w = weight_dev ? *weight_dev : weight;
  const float loss = nm ? (float)((double)w * tot / (double)nm) : 0.0f;
  ws->scale = nm ? (float)((double)w / (double)nm) : 0.0f;
  ws->ticket = 0;  // ready for the next call (stream-ordered)
  if (loss_out) *loss_out = loss;
  if (total_out) *total_out = (e_photo ? *e_photo : 0.0f) + loss;
}

__global__ void __launch_bounds__(kDcThreads) depth_chain_grad_kernel(
    const float* __restrict__ depth, const float* __restrict__ final_T,
    const int32_t* __restrict__ n_contrib, const float* __restrict__ prior,
    const uint8_t* __restrict__ valid, long long n, const DcWs* __restrict__ ws,
    float* __restrict__ grad_depth, float* __restrict__ grad_final_T) {
  const float scale = ws->scale;
  for (long long p = (long long)blockIdx.x * kDcThreads + threadIdx.x; p < n;
       p += (long long)gridDim.x * kDcThreads) {
    float d, dr, diff, gd = 0.f, gt = 0.f;
    if (dc_diff(p, depth, final_T, n_contrib, prior, valid, d, dr, diff) && d >= kDispEps) {
      const float sgn = diff > 0.f ? 1.f : (diff < 0.f ? -1.f : 0.f);
      const float g = scale * sgn * (-1.0f / (dr * dr));
      const float den = 1.0f - final_T[p];
      gd = g / den;
      gt = g * depth[p] / (den * den);
    }
    grad_depth[p] = gd;
    grad_final_T[p] = gt;
  }
}

}  // namespace tsr

using namespace tsr;

extern "C" size_t tsr_depth_chain_workspace(void) { return sizeof(DcWs); }

extern "C" int tsr_depth_chain(const float* depth, const float* final_T, const int32_t* n_contrib,
                               const float* prior, const uint8_t* valid, int32_t height,
                               int32_t width, float weight, const float* weight_dev,
                               const float* e_photo, float* loss_out, float* total_out,
                               float* grad_depth, float* grad_final_T, void* workspace,
                               size_t workspace_bytes, void* stream) {
  if (height <= 0 || width <= 0 || !depth || !final_T || !n_contrib || !prior || !grad_depth ||
      !grad_final_T || !workspace)
    return TSR_E_INVALID;
  if (workspace_bytes < sizeof(DcWs)) return TSR_E_WORKSPACE;
  const long long n = (long long)height * width;
  cudaStream_t s = (cudaStream_t)stream;
  DcWs* ws = (DcWs*)workspace;
  depth_chain_reduce_kernel<<<kDcBlocks, kDcThreads, 0, s>>>(
      depth, final_T, n_contrib, prior, valid, n, weight, weight_dev, e_photo, loss_out,
      total_out, ws);
  TSR_CHECK_LAUNCH();
  depth_chain_grad_kernel<<<kDcBlocks, kDcThreads, 0, s>>>(depth, final_T, n_contrib, prior,
                                                           valid, n, ws, grad_depth,
                                                           grad_final_T);
  TSR_CHECK_LAUNCH();
  return TSR_OK;
}
