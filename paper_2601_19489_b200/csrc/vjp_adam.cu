// K4b preprocess backward (project_vjp + colour/SH chain) and K5 fused Adam.
//
//   project_vjp   projection.py:139-241  (conic -> Sigma2 -> A, J, R -> p_cam,
//                                         M -> scales, quaternion with the
//                                         normalisation projection, opacity
//                                         logit, pose sums)
//   _full_grads   trainer.py:231-257, eval_sh_vjp scene.py:279-291
//   Adam.step     optim.py:60-88 (dense, non-finite rows skipped+counted,
//                                 quaternion rows renormalised)
// tsr_preprocess_bwd_adam fuses the two for the single-view training step so
// the 3D gradient never round-trips through HBM.
#include <cuda_runtime.h>

#include "tsr_common.cuh"
#include "tsr_vjp_adam.cuh"

namespace tsr {

// Per-Gaussian chain; returns false (all-zero gradient) for culled rows.
__device__ __forceinline__ bool vjp_one(const tsr_gaussians_t& G, const tsr_camera_t& cam,
                                        const float4* rec, const int32_t* row_of_source,
                                        const float* grad2d, long long i, Vjp& out) {
  const int row = row_of_source[i];
  if (row < 0) return false;
  const float ls[3] = {G.log_scales[3 * i], G.log_scales[3 * i + 1], G.log_scales[3 * i + 2]};
  const float qv[4] = {G.rotations[4 * i], G.rotations[4 * i + 1], G.rotations[4 * i + 2],
                       G.rotations[4 * i + 3]};
  const float px = G.positions[3 * i], py = G.positions[3 * i + 1], pz = G.positions[3 * i + 2];
  vjp_core(cam, px, py, pz, ls, qv, rec[3 * row], rec[3 * row + 1],
           grad2d + (long long)row * TSR_GRAD2D_FLOATS, out);
  // SH > 0: unit-direction chain back to positions (trainer.py:247-254)
  const int C = G.sh_coeffs;
  if (C > 1) {
    float vx = px - cam.center[0], vy = py - cam.center[1], vz = pz - cam.center[2];
    const float vn = sqrtf(vx * vx + vy * vy + vz * vz);
    const float ivn = 1.0f / vn;
    const float dx = vx * ivn, dy = vy * ivn, dz = vz * ivn;
    out.dir[0] = dx; out.dir[1] = dy; out.dir[2] = dz;
    const float* coef = G.colors + i * C * 3;
    float wk[16];
    for (int k = 0; k < C; ++k)
      wk[k] = coef[3 * k] * out.gcol[0] + coef[3 * k + 1] * out.gcol[1] + coef[3 * k + 2] * out.gcol[2];
    float gdir[3];
    sh_basis_vjp(sh_degree_of(C), dx, dy, dz, wk, gdir);
    const float dd = gdir[0] * dx + gdir[1] * dy + gdir[2] * dz;
    out.gp[0] += (gdir[0] - dx * dd) * ivn;
    out.gp[1] += (gdir[1] - dy * dd) * ivn;
    out.gp[2] += (gdir[2] - dz * dd) * ivn;
  }
  return true;
}


// colour-coefficient gradient k, channel ch
__device__ __forceinline__ float color_grad(const Vjp& v, const float* basis, int C, int k,
                                            int ch) {
  return C == 1 ? v.gcol[ch] : basis[k] * v.gcol[ch];
}

__device__ __forceinline__ void block_reduce_pose(float* vals, float* pose_sums) {
  __shared__ float s_red[12][8];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < 12; ++k) {
    float v = vals[k];
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
    if (lane == 0) s_red[k][warp] = v;
  }
  __syncthreads();
  if (threadIdx.x < 12) {
    float v = 0.f;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) v += s_red[threadIdx.x][w];
    atomicAdd(pose_sums + threadIdx.x, v);
  }
}

__global__ void __launch_bounds__(256) preprocess_bwd_kernel(
    tsr_gaussians_t G, tsr_camera_t cam, const float4* __restrict__ rec,
    const int32_t* __restrict__ row_of_source, const float* __restrict__ grad2d,
    float* __restrict__ gpos, float* __restrict__ gls, float* __restrict__ grot,
    float* __restrict__ gop, float* __restrict__ gcol, float* __restrict__ pose_sums,
    int accumulate) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  Vjp v;
  bool vis = false;
  if (i < G.n) vis = vjp_one(G, cam, rec, row_of_source, grad2d, i, v);
  if (i < G.n) {
    if (!vis) {
#pragma unroll
      for (int k = 0; k < 3; ++k) { v.gp[k] = 0.f; v.gls[k] = 0.f; v.gcol[k] = 0.f; }
#pragma unroll
      for (int k = 0; k < 4; ++k) v.gq[k] = 0.f;
      v.go = 0.f;
    }
    const int C = G.sh_coeffs;
    float basis[16];
    if (vis && C > 1) sh_basis(sh_degree_of(C), v.dir[0], v.dir[1], v.dir[2], basis);
    if (accumulate) {
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        gpos[3 * i + k] += v.gp[k];
        gls[3 * i + k] += v.gls[k];
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) grot[4 * i + k] += v.gq[k];
      gop[i] += v.go;
      if (vis)
        for (int k = 0; k < C; ++k)
          for (int ch = 0; ch < 3; ++ch) gcol[(i * C + k) * 3 + ch] += color_grad(v, basis, C, k, ch);
    } else {
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        gpos[3 * i + k] = v.gp[k];
        gls[3 * i + k] = v.gls[k];
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) grot[4 * i + k] = v.gq[k];
      gop[i] = v.go;
      for (int k = 0; k < C; ++k)
        for (int ch = 0; ch < 3; ++ch)
          gcol[(i * C + k) * 3 + ch] = vis ? color_grad(v, basis, C, k, ch) : 0.f;
    }
  }
  if (pose_sums) {
    float pv[12];
#pragma unroll
    for (int k = 0; k < 12; ++k) pv[k] = vis ? v.pose[k] : 0.f;
    block_reduce_pose(pv, pose_sums);
  }
}

// One parameter row: returns 1 when skipped (non-finite gradient).
// Bias corrections enter as reciprocals (one divide per group, not per
// element) and the step uses a fast divide: the update differs from the
// reference's float64 m_hat / (sqrt(v_hat) + eps) by a few FP32 ulp.
template <typename GradFn>
__device__ __forceinline__ int adam_row(const tsr_adam_group_t& G, long long r, GradFn grad,
                                        const float* scal = nullptr, int gk = 0) {
  const int w = G.width;
  bool finite = true;
  for (int k = 0; k < w; ++k) finite &= isfinite(grad(k));
  if (!finite) return 1;
  float* p = G.param + r * w;
  float* m = G.exp_avg + r * w;
  float* v = G.exp_avg_sq + r * w;
  const float lr = scal ? scal[3 * gk] : G.lr;
  const float ibc1 = 1.0f / (scal ? scal[3 * gk + 1] : G.bias_correction1),
              ibc2 = 1.0f / (scal ? scal[3 * gk + 2] : G.bias_correction2);
  float nrm = 0.f;
  for (int k = 0; k < w; ++k) {
    const float gk = grad(k);
    const float mk = kBeta1 * m[k] + kOneMinusBeta1 * gk;
    const float vk = kBeta2 * v[k] + kOneMinusBeta2 * gk * gk;
    m[k] = mk;
    v[k] = vk;
    const float pk = p[k] - __fdividef(lr * (mk * ibc1), sqrtf(vk * ibc2) + kEps);
    p[k] = pk;
    nrm += pk * pk;
  }
  if (G.renormalize) {
    nrm = sqrtf(nrm);
    if (nrm > 0.f) {
      const float inv = 1.0f / nrm;
      for (int k = 0; k < w; ++k) p[k] = p[k] * inv;
    }
  }
  return 0;
}

// scal (nullable): per-step [lr, bias_correction1, bias_correction2] of group
// (gi % scal_period) from device memory -- CUDA-graph replay, where the
// descriptors' by-value scalars are frozen at capture
__global__ void __launch_bounds__(256) adam_kernel(AdamGroups groups,
                                                   unsigned long long* __restrict__ skipped,
                                                   const float* __restrict__ scal,
                                                   int scal_period) {
  const long long total = groups.row_start[groups.n];
  unsigned long long local = 0;
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    int gi = 0;
    while (t >= groups.row_start[gi + 1]) ++gi;
    const tsr_adam_group_t& G = groups.g[gi];
    const long long r = t - groups.row_start[gi];
    const float* g = G.grad + r * G.width;
    local += adam_row(G, r, [&](int k) { return g[k]; }, scal, scal ? gi % scal_period : 0);
  }
  // warp-aggregated skip counter
  for (int d = 16; d > 0; d >>= 1) local += __shfl_xor_sync(0xffffffffu, local, d);
  if ((threadIdx.x & 31) == 0 && local) atomicAdd(skipped, local);
}

__global__ void __launch_bounds__(256) preprocess_bwd_adam_kernel(
    tsr_gaussians_t G, tsr_camera_t cam, const float4* __restrict__ rec,
    const int32_t* __restrict__ row_of_source, const float* __restrict__ grad2d,
    AdamGroups groups, float* __restrict__ pose_sums, unsigned long long* __restrict__ skipped,
    const float* __restrict__ scal, const int32_t* __restrict__ gate,
    int32_t* __restrict__ gated_steps, const float* __restrict__ loss_guard) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const bool diverged = loss_guard && !isfinite(*loss_guard);
  if ((gate && *gate) || diverged) {  // no update (see vjp_adam_sh0_kernel)
    if (i == 0 && gated_steps && !diverged) atomicAdd(gated_steps, 1);
    return;
  }
  Vjp v;
  bool vis = false;
  unsigned long long local = 0;
  if (i < G.n) {
    vis = vjp_one(G, cam, rec, row_of_source, grad2d, i, v);
    const int C = G.sh_coeffs;
    float basis[16];
    if (vis && C > 1) sh_basis(sh_degree_of(C), v.dir[0], v.dir[1], v.dir[2], basis);
    local += adam_row(groups.g[0], i, [&](int k) { return vis ? v.gp[k] : 0.f; }, scal, 0);
    local += adam_row(groups.g[1], i, [&](int k) { return vis ? v.gls[k] : 0.f; }, scal, 1);
    local += adam_row(groups.g[2], i, [&](int k) { return vis ? v.gq[k] : 0.f; }, scal, 2);
    local += adam_row(groups.g[3], i, [&](int k) { return vis ? v.go : 0.f; }, scal, 3);
    local += adam_row(groups.g[4], i, [&](int k) {
      return vis ? color_grad(v, basis, C, k / 3, k % 3) : 0.f;
    }, scal, 4);
  }
  if (pose_sums) {
    float pv[12];
#pragma unroll
    for (int k = 0; k < 12; ++k) pv[k] = vis ? v.pose[k] : 0.f;
    block_reduce_pose(pv, pose_sums);
  }
  for (int d = 16; d > 0; d >>= 1) local += __shfl_xor_sync(0xffffffffu, local, d);
  if ((threadIdx.x & 31) == 0 && local) atomicAdd(skipped, local);
}

// SH degree 0 fast path: every parameter / moment of the Gaussian is loaded
// up front (42 independent loads in flight), the VJP runs on the registers,
// the consumed Grad2D row is zeroed for the next step, and the five Adam
// groups are updated and stored.
#ifndef TSR_VJP_MINB
#define TSR_VJP_MINB 6  // 80 registers: measured 97 us vs 101 us at 7 CTAs/SM (72 registers, more spills)
#endif
// kPose: accumulate the pose sums (pose optimisation); without it the
// twelve per-Gaussian pose terms are dead code (registers for the Adam part)
template <bool kPose>
__global__ void __launch_bounds__(128, TSR_VJP_MINB) vjp_adam_sh0_kernel(
    tsr_camera_t cam, long long n, const float4* __restrict__ rec,
    const int32_t* __restrict__ row_of_source, float* __restrict__ grad2d, AdamGroups groups,
    float* __restrict__ pose_sums, unsigned long long* __restrict__ skipped,
    const float* __restrict__ scal, const int32_t* __restrict__ gate,
    int32_t* __restrict__ gated_steps, const float* __restrict__ loss_guard) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  // a non-finite loss (trainer.py:331-338 raises TrainingDiverged before its
  // Adam step) leaves the parameters untouched; the host raises at its next
  // flush
  const bool diverged = loss_guard && !isfinite(*loss_guard);
  if ((gate && *gate) || diverged) {
    // the step's pair capacity overflowed (K2's sticky flag): its Grad2D
    // comes from truncated tile lists, so the update is skipped -- params
    // and moments untouched, the consumed row zeroed for the next step; the
    // host grows the capacity and redoes the step (TrainStep._poll_status)
    if (i < n) {
      const int row = row_of_source[i];
      if (row >= 0) {
        float* g2p = grad2d + (long long)row * TSR_GRAD2D_FLOATS;
#pragma unroll
        for (int k = 0; k < TSR_GRAD2D_FLOATS; ++k) g2p[k] = 0.f;
      }
    }
    if (i == 0 && gated_steps && !diverged) atomicAdd(gated_steps, 1);
    return;
  }
  bool vis = false;
  unsigned long long local = 0;
  float pose[12];
  if (i < n)
    local = vjp_adam_row_sh0<kPose>(cam, groups, i, row_of_source[i], rec, grad2d, scal, true,
                                    pose, vis);
  if (kPose) {
    float pv[12];
#pragma unroll
    for (int k = 0; k < 12; ++k) pv[k] = vis ? pose[k] : 0.f;
    block_reduce_pose(pv, pose_sums);
  }
  for (int d = 16; d > 0; d >>= 1) local += __shfl_xor_sync(0xffffffffu, local, d);
  if ((threadIdx.x & 31) == 0 && local) atomicAdd(skipped, local);
}

// ---- fused ZeRO-1 update over peer memory (the B200 variant)
// One CTA per (group, 64-row chunk of this rank's shard): the chunk's
// gradient is the sum of the ranks' rows read through peer pointers in rank
// order (bitwise the deterministic fixed-order reduction) with consecutive
// threads on consecutive floats (every peer read is a coalesced 128-byte
// line over NVLink, not a row-strided scalar), Adam runs element-wise on
// the local parameters with this rank's shard moments (rows with a
// non-finite gradient untouched, the quaternion rows renormalised), and the
// updated chunk is stored into every rank's parameter buffer, again
// coalesced -- reduce-scatter + K5 + all-gather as one kernel, no collective
// library.  Rows are staged in shared memory for the row-level parts.
constexpr int kPeerMaxWorld = 8;
constexpr int kPeerMaxWidth = 48;  // colors at SH degree 3
constexpr int kPeerRows = 64;
struct PeerPtrs {
  const float* g[kPeerMaxWorld * TSR_MAX_ADAM_GROUPS];  // [rank * n_groups + group]
  float* p[kPeerMaxWorld * TSR_MAX_ADAM_GROUPS];
};

__global__ void __launch_bounds__(256) zero1_peer_adam_kernel(AdamGroups groups, PeerPtrs pp,
                                                              int world, long long row_begin,
                                                              long long rows,
                                                              unsigned long long* __restrict__ skipped) {
  extern __shared__ float s_peer[];
  const int gi = blockIdx.y, ng = groups.n, tid = threadIdx.x;
  const tsr_adam_group_t& G = groups.g[gi];
  const int w = G.width;
  const long long r0 = (long long)blockIdx.x * kPeerRows;
  if (r0 >= rows) return;
  const int nr = (int)min((long long)kPeerRows, rows - r0), ne = nr * w;
  float* s_g = s_peer;                                   // summed gradients
  float* s_p = s_peer + kPeerRows * kPeerMaxWidth;       // updated parameters
  int* s_ok = reinterpret_cast<int*>(s_peer + 2 * kPeerRows * kPeerMaxWidth);  // finite rows
  const long long f0 = (row_begin + r0) * w;  // flat offset: parameters / gradients
  const long long m0 = r0 * w;                // flat offset: the shard's moments
  if (tid < nr) s_ok[tid] = 1;
  for (int e = tid; e < ne; e += blockDim.x) {
    float acc = pp.g[gi][f0 + e];
    for (int q = 1; q < world; ++q) acc += pp.g[q * ng + gi][f0 + e];
    s_g[e] = acc;
  }
  __syncthreads();
  for (int e = tid; e < ne; e += blockDim.x)
    if (!isfinite(s_g[e])) s_ok[e / w] = 0;
  __syncthreads();
  const float ibc1 = 1.0f / G.bias_correction1, ibc2 = 1.0f / G.bias_correction2;
  float* m = G.exp_avg + m0;
  float* v = G.exp_avg_sq + m0;
  const float* prm = G.param + f0;
  for (int e = tid; e < ne; e += blockDim.x) {
    float pk = prm[e];
    if (s_ok[e / w]) {
      const float gk = s_g[e];
      const float mk = kBeta1 * m[e] + kOneMinusBeta1 * gk;
      const float vk = kBeta2 * v[e] + kOneMinusBeta2 * gk * gk;
      m[e] = mk;
      v[e] = vk;
      pk = pk - __fdividef(G.lr * (mk * ibc1), sqrtf(vk * ibc2) + kEps);
    }
    s_p[e] = pk;
  }
  __syncthreads();
  if (G.renormalize && tid < nr && s_ok[tid]) {  // the row's norm in element order
    float* row = s_p + tid * w;
    float nrm = 0.f;
    for (int k = 0; k < w; ++k) nrm += row[k] * row[k];
    nrm = sqrtf(nrm);
    if (nrm > 0.f) {
      const float inv = 1.0f / nrm;
      for (int k = 0; k < w; ++k) row[k] = row[k] * inv;
    }
  }
  __syncthreads();
  for (int e = tid; e < ne; e += blockDim.x) {  // all-gather by direct stores, own rank included
    const float pv = s_p[e];
    for (int q = 0; q < world; ++q) pp.p[q * ng + gi][f0 + e] = pv;
  }
  unsigned long long local = (tid < nr && !s_ok[tid]) ? 1ull : 0ull;
  for (int d = 16; d > 0; d >>= 1) local += __shfl_xor_sync(0xffffffffu, local, d);
  if ((tid & 31) == 0 && local) atomicAdd(skipped, local);
}

// Adam for the Gaussians K4's fused epilogue does not reach (backward.cu,
// tsr_render_bwd_adam): culled ones and visible rows without any (tile,
// splat) pair -- a zero gradient, a dense update all the same (optim.py:78-82)
// -- and the re-arming of the per-row merge counters for the next step.  A
// row whose count did not complete (a pair-capacity overflow: its pairs past
// the capacity were never stored) has its Grad2D zeroed here; that step's
// update is gated anyway.
__global__ void __launch_bounds__(128, TSR_VJP_MINB) vjp_adam_rest_kernel(
    tsr_camera_t cam, long long n, const float4* __restrict__ rec,
    const int32_t* __restrict__ row_of_source, const int32_t* __restrict__ counts,
    int32_t* __restrict__ row_done, float* __restrict__ grad2d, AdamGroups groups,
    unsigned long long* __restrict__ skipped, const float* __restrict__ scal,
    const int32_t* __restrict__ gate, int32_t* __restrict__ gated_steps,
    const float* __restrict__ loss_guard) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const bool diverged = loss_guard && !isfinite(*loss_guard);
  const bool gated = gate && *gate;
  const bool update = !gated && !diverged;
  unsigned long long local = 0;
  if (i < n) {
    const int row = row_of_source[i];
    bool mine = row < 0;
    if (row >= 0) {
      const int c = counts[row], d = row_done[row];
      row_done[row] = 0;  // re-armed for the next step
      if (c == 0) {
        mine = true;
      } else if (d != c) {
        float* g2p = grad2d + (long long)row * TSR_GRAD2D_FLOATS;
#pragma unroll
        for (int k = 0; k < TSR_GRAD2D_FLOATS; ++k) g2p[k] = 0.f;
      }
    }
    if (mine) {
      bool vis;
      float pose[12];
      local = vjp_adam_row_sh0<false>(cam, groups, i, row, rec, grad2d, scal, update, pose, vis);
    }
  }
  if (i == 0 && gated && gated_steps && !diverged) atomicAdd(gated_steps, 1);
  for (int d = 16; d > 0; d >>= 1) local += __shfl_xor_sync(0xffffffffu, local, d);
  if ((threadIdx.x & 31) == 0 && local) atomicAdd(skipped, local);
}

}  // namespace tsr

using namespace tsr;

extern "C" int tsr_preprocess_bwd(const tsr_gaussians_t* g, const tsr_camera_t* cam,
                                  const float* rec, const int32_t* row_of_source,
                                  const float* grad2d, float* grad_positions,
                                  float* grad_log_scales, float* grad_rotations,
                                  float* grad_opacity_logits, float* grad_colors,
                                  float* pose_sums, int32_t accumulate, void* stream) {
  if (!g || !cam || g->n < 0) return TSR_E_INVALID;
  if (g->n == 0) return TSR_OK;
  int blocks = (int)((g->n + 255) / 256);
  preprocess_bwd_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(
      *g, *cam, (const float4*)rec, row_of_source, grad2d, grad_positions, grad_log_scales,
      grad_rotations, grad_opacity_logits, grad_colors, pose_sums, accumulate);
  TSR_CHECK_LAUNCH();
  return TSR_OK;
}

extern "C" int tsr_adam_step(const tsr_adam_group_t* groups_host, int32_t n_groups,
                             unsigned long long* skipped, void* stream) {
  AdamGroups gs;
  if (!fill_adam_groups(groups_host, n_groups, gs) || !skipped) return TSR_E_INVALID;
  for (int k = 0; k < n_groups; ++k)
    if (!gs.g[k].grad || !gs.g[k].exp_avg || !gs.g[k].exp_avg_sq) return TSR_E_INVALID;
  const long long total = gs.row_start[n_groups];
  if (total == 0) return TSR_OK;
  long long blocks = (total + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  adam_kernel<<<(int)blocks, 256, 0, (cudaStream_t)stream>>>(gs, skipped, nullptr, 1);
  TSR_CHECK_LAUNCH();
  return TSR_OK;
}

extern "C" int tsr_adam_step_dev(const tsr_adam_group_t* groups_host, int32_t n_groups,
                                 const float* group_scalars, int32_t scal_period,
                                 unsigned long long* skipped, void* stream) {
  AdamGroups gs;
  if (!fill_adam_groups(groups_host, n_groups, gs) || !skipped || !group_scalars || scal_period < 1)
    return TSR_E_INVALID;
  for (int k = 0; k < n_groups; ++k)
    if (!gs.g[k].grad || !gs.g[k].exp_avg || !gs.g[k].exp_avg_sq) return TSR_E_INVALID;
  const long long total = gs.row_start[n_groups];
  if (total == 0) return TSR_OK;
  long long blocks = (total + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  adam_kernel<<<(int)blocks, 256, 0, (cudaStream_t)stream>>>(gs, skipped, group_scalars,
                                                             scal_period);
  TSR_CHECK_LAUNCH();
  return TSR_OK;
}

extern "C" int tsr_zero1_peer_adam(const tsr_adam_group_t* groups_host, int32_t n_groups,
                                   int32_t world, const float* const* peer_grads,
                                   float* const* peer_params, int64_t row_begin,
                                   int64_t row_end, unsigned long long* skipped, void* stream) {
  if (!groups_host || !peer_grads || !peer_params || !skipped) return TSR_E_INVALID;
  if (world < 1 || world > kPeerMaxWorld || n_groups < 1 || n_groups > TSR_MAX_ADAM_GROUPS)
    return TSR_E_INVALID;
  if (row_begin < 0 || row_end < row_begin) return TSR_E_INVALID;
  AdamGroups gs;
  if (!fill_adam_groups(groups_host, n_groups, gs)) return TSR_E_INVALID;
  PeerPtrs pp;
  for (int q = 0; q < world; ++q)
    for (int k = 0; k < n_groups; ++k) {
      if (gs.g[k].width > kPeerMaxWidth || !gs.g[k].exp_avg || !gs.g[k].exp_avg_sq)
        return TSR_E_INVALID;
      pp.g[q * n_groups + k] = peer_grads[q * n_groups + k];
      pp.p[q * n_groups + k] = peer_params[q * n_groups + k];
      if (!pp.g[q * n_groups + k] || !pp.p[q * n_groups + k]) return TSR_E_INVALID;
    }
  // every group covers the shard rows [row_begin, row_end)
  const long long rows = row_end - row_begin;
  if (rows == 0) return TSR_OK;
  const size_t smem = (2 * kPeerRows * kPeerMaxWidth + kPeerRows) * sizeof(float);
  const dim3 grid((unsigned)((rows + kPeerRows - 1) / kPeerRows), (unsigned)n_groups);
  zero1_peer_adam_kernel<<<grid, 256, smem, (cudaStream_t)stream>>>(gs, pp, world, row_begin, rows,
                                                                    skipped);
  TSR_CHECK_LAUNCH();
  return TSR_OK;
}

extern "C" int tsr_preprocess_bwd_adam(const tsr_gaussians_t* g, const tsr_camera_t* cam,
                                       const float* rec, const int32_t* row_of_source,
                                       const float* grad2d,
                                       const tsr_adam_group_t* groups_host, float* pose_sums,
                                       unsigned long long* skipped, void* stream) {
  return tsr_preprocess_bwd_adam_ex(g, cam, rec, row_of_source, grad2d, groups_host, nullptr,
                                    pose_sums, skipped, nullptr, nullptr, nullptr, stream);
}

extern "C" int tsr_preprocess_bwd_adam_dev(const tsr_gaussians_t* g, const tsr_camera_t* cam,
                                           const float* rec, const int32_t* row_of_source,
                                           const float* grad2d,
                                           const tsr_adam_group_t* groups_host,
                                           const float* group_scalars, float* pose_sums,
                                           unsigned long long* skipped, void* stream) {
  return tsr_preprocess_bwd_adam_ex(g, cam, rec, row_of_source, grad2d, groups_host,
                                    group_scalars, pose_sums, skipped, nullptr, nullptr, nullptr, stream);
}

extern "C" int tsr_preprocess_bwd_adam_ex(const tsr_gaussians_t* g, const tsr_camera_t* cam,
                                          const float* rec, const int32_t* row_of_source,
                                          const float* grad2d,
                                          const tsr_adam_group_t* groups_host,
                                          const float* group_scalars, float* pose_sums,
                                          unsigned long long* skipped, const int32_t* gate,
                                          int32_t* gated_steps, const float* loss_guard,
                                          void* stream) {
  AdamGroups gs;
  if (!g || !cam || !fill_adam_groups(groups_host, 5, gs) || !skipped) return TSR_E_INVALID;
  for (int k = 0; k < 5; ++k)
    if (gs.g[k].rows != g->n || !gs.g[k].exp_avg || !gs.g[k].exp_avg_sq) return TSR_E_INVALID;
  if (gs.g[0].width != 3 || gs.g[1].width != 3 || gs.g[2].width != 4 || gs.g[3].width != 1 ||
      gs.g[4].width != 3 * g->sh_coeffs)
    return TSR_E_INVALID;
  if (g->n == 0) return TSR_OK;
  int blocks = (int)((g->n + 255) / 256);
  if (g->sh_coeffs == 1) {
    // fast path; also zeroes the consumed Grad2D rows for the next step
    auto* k = pose_sums ? vjp_adam_sh0_kernel<true> : vjp_adam_sh0_kernel<false>;
    k<<<(int)((g->n + 127) / 128), 128, 0, (cudaStream_t)stream>>>(
        *cam, g->n, (const float4*)rec, row_of_source, (float*)grad2d, gs, pose_sums, skipped,
        group_scalars, gate, gated_steps, loss_guard);
  } else {
    preprocess_bwd_adam_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(
        *g, *cam, (const float4*)rec, row_of_source, grad2d, gs, pose_sums, skipped,
        group_scalars, gate, gated_steps, loss_guard);
  }
  TSR_CHECK_LAUNCH();
  return TSR_OK;
}

extern "C" const char* tsr_version(void) {
  return "tilesplat_b200 0.1.0 sm_100a";
}

// Launch of vjp_adam_rest_kernel for tsr_render_bwd_adam (backward.cu).
int tsr_launch_vjp_adam_rest(const tsr_camera_t& cam, long long n, const float* rec,
                             const int32_t* row_of_source, const int32_t* counts,
                             int32_t* row_done, float* grad2d, const tsr::AdamGroups& gs,
                             unsigned long long* skipped, const float* scal, const int32_t* gate,
                             int32_t* gated_steps, const float* loss_guard, cudaStream_t s) {
  if (n <= 0) return TSR_OK;
  vjp_adam_rest_kernel<<<(int)((n + 127) / 128), 128, 0, s>>>(
      cam, n, (const float4*)rec, row_of_source, counts, row_done, grad2d, gs, skipped, scal,
      gate, gated_steps, loss_guard);
  TSR_CHECK_LAUNCH();
  return TSR_OK;
}
