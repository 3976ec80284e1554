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

namespace tsr {

struct Vjp {
  float gp[3], gls[3], gq[4], go;
  float gcol[3];           // d colour (for the SH chain)
  float dir[3];            // unit view direction (SH > 0)
  float pose[12];          // J^T G_A + g_pcam p^T (3x3), g_pcam (3)
};

// Per-Gaussian chain on already-loaded parameters (position p, log-scales
// ls, raw quaternion q) and the packed Grad2D row g2.
__device__ __forceinline__ void vjp_core(const tsr_camera_t& cam, float px, float py, float pz,
                                         const float* ls, const float* qv, float4 r0, float4 r1,
                                         const float* g2, Vjp& out);

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

__device__ __forceinline__ void vjp_core(const tsr_camera_t& cam, float px, float py, float pz,
                                         const float* ls, const float* qv, float4 r0, float4 r1,
                                         const float* g2, Vjp& out) {
  const float* R = cam.R;
  const float X = fmaf(R[0], px, fmaf(R[1], py, fmaf(R[2], pz, cam.t[0])));
  const float Y = fmaf(R[3], px, fmaf(R[4], py, fmaf(R[5], pz, cam.t[1])));
  const float Z = fmaf(R[6], px, fmaf(R[7], py, fmaf(R[8], pz, cam.t[2])));
  float qw = qv[0], qx = qv[1], qy = qv[2], qz = qv[3];
  const float qnorm = sqrtf(qw * qw + qx * qx + qy * qy + qz * qz);
  const float iqn = 1.0f / qnorm;
  qw *= iqn; qx *= iqn; qy *= iqn; qz *= iqn;
  float Rq[9];
  Rq[0] = 1.f - 2.f * (qy * qy + qz * qz);
  Rq[1] = 2.f * (qx * qy - qw * qz);
  Rq[2] = 2.f * (qx * qz + qw * qy);
  Rq[3] = 2.f * (qx * qy + qw * qz);
  Rq[4] = 1.f - 2.f * (qx * qx + qz * qz);
  Rq[5] = 2.f * (qy * qz - qw * qx);
  Rq[6] = 2.f * (qx * qz - qw * qy);
  Rq[7] = 2.f * (qy * qz + qw * qx);
  Rq[8] = 1.f - 2.f * (qx * qx + qy * qy);
  const float s[3] = {expf(ls[0]), expf(ls[1]), expf(ls[2])};
  float M[9];
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int k = 0; k < 3; ++k) M[3 * r + k] = Rq[3 * r + k] * s[k];
  float S3[9];
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int k = 0; k < 3; ++k)
      S3[3 * r + k] = M[3 * r] * M[3 * k] + M[3 * r + 1] * M[3 * k + 1] + M[3 * r + 2] * M[3 * k + 2];
  const float iz = 1.0f / Z, iz2 = iz * iz;
  const float fx = cam.fx, fy = cam.fy;
  // J rows: (j00, 0, j02), (0, j11, j12)
  const float j00 = fx * iz, j02 = -fx * X * iz2, j11 = fy * iz, j12 = -fy * Y * iz2;
  float A[6];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    A[k] = j00 * R[k] + j02 * R[6 + k];
    A[3 + k] = j11 * R[3 + k] + j12 * R[6 + k];
  }
  const float ca = r0.z, cb = r0.w, cc = r1.x, o = r1.y;
  const float gm0 = g2[0], gm1 = g2[1];
  const float gb00 = g2[2], gb01 = 0.5f * g2[3], gb11 = g2[4];
  const float gop = g2[5];
  out.gcol[0] = g2[6]; out.gcol[1] = g2[7]; out.gcol[2] = g2[8];
  const float gdep = g2[9];
  // G_Sigma = -C Gbar C  (2x2 symmetric)
  const float t00 = ca * gb00 + cb * gb01, t01 = ca * gb01 + cb * gb11;
  const float t10 = cb * gb00 + cc * gb01, t11 = cb * gb01 + cc * gb11;
  const float G00 = -(t00 * ca + t01 * cb), G01 = -(t00 * cb + t01 * cc);
  const float G10 = -(t10 * ca + t11 * cb), G11 = -(t10 * cb + t11 * cc);
  // AS = A Sigma3 (2x3);  G_A = 2 G_Sigma AS
  float AS[6];
#pragma unroll
  for (int r = 0; r < 2; ++r)
#pragma unroll
    for (int k = 0; k < 3; ++k)
      AS[3 * r + k] = A[3 * r] * S3[k] + A[3 * r + 1] * S3[3 + k] + A[3 * r + 2] * S3[6 + k];
  float GA[6];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    GA[k] = 2.f * (G00 * AS[k] + G01 * AS[3 + k]);
    GA[3 + k] = 2.f * (G10 * AS[k] + G11 * AS[3 + k]);
  }
  // G_Sigma3 = A^T G_Sigma A (3x3)
  float GS3[9];
#pragma unroll
  for (int r = 0; r < 3; ++r) {
    const float u0 = A[r] * G00 + A[3 + r] * G10;
    const float u1 = A[r] * G01 + A[3 + r] * G11;
#pragma unroll
    for (int k = 0; k < 3; ++k) GS3[3 * r + k] = u0 * A[k] + u1 * A[3 + k];
  }
  // G_J = G_A R^T (only the 4 entries J depends on are needed)
  const float GJ00 = GA[0] * R[0] + GA[1] * R[1] + GA[2] * R[2];
  const float GJ02 = GA[0] * R[6] + GA[1] * R[7] + GA[2] * R[8];
  const float GJ11 = GA[3] * R[3] + GA[4] * R[4] + GA[5] * R[5];
  const float GJ12 = GA[3] * R[6] + GA[4] * R[7] + GA[5] * R[8];
  const float iz3 = iz2 * iz;
  const float gx = gm0 * fx * iz - GJ02 * fx * iz2;
  const float gy = gm1 * fy * iz - GJ12 * fy * iz2;
  const float gz = -gm0 * fx * X * iz2 - gm1 * fy * Y * iz2 + gdep - GJ00 * fx * iz2 -
                   GJ11 * fy * iz2 + GJ02 * 2.f * fx * X * iz3 + GJ12 * 2.f * fy * Y * iz3;
  // pose sums: J^T G_A + g_pcam p^T, g_pcam
  const float Jm[6] = {j00, 0.f, j02, 0.f, j11, j12};
  const float gpc[3] = {gx, gy, gz};
  const float pw[3] = {px, py, pz};
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int k = 0; k < 3; ++k)
      out.pose[3 * r + k] = Jm[r] * GA[k] + Jm[3 + r] * GA[3 + k] + gpc[r] * pw[k];
  out.pose[9] = gx; out.pose[10] = gy; out.pose[11] = gz;
  // Sigma3 = M M^T:  G_M = 2 G_Sigma3 M ; G_Rq = G_M diag(s) ; grad s
  float GM[9];
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int k = 0; k < 3; ++k)
      GM[3 * r + k] = 2.f * (GS3[3 * r] * M[k] + GS3[3 * r + 1] * M[3 + k] + GS3[3 * r + 2] * M[6 + k]);
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const float gsk = GM[k] * Rq[k] + GM[3 + k] * Rq[3 + k] + GM[6 + k] * Rq[6 + k];
    out.gls[k] = gsk * s[k];
  }
  float GR[9];
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int k = 0; k < 3; ++k) GR[3 * r + k] = GM[3 * r + k] * s[k];
  // d R / d (w,x,y,z) contracted with G_R (projection.py:213-219)
  const float w = qw, x = qx, y = qy, z = qz;
  const float gw = 2.f * (-z * GR[1] + y * GR[2] + z * GR[3] - x * GR[5] - y * GR[6] + x * GR[7]);
  const float gxq = 2.f * (y * GR[1] + z * GR[2] + y * GR[3] - 2.f * x * GR[4] - w * GR[5] +
                           z * GR[6] + w * GR[7] - 2.f * x * GR[8]);
  const float gyq = 2.f * (-2.f * y * GR[0] + x * GR[1] + w * GR[2] + x * GR[3] + z * GR[5] -
                           w * GR[6] + z * GR[7] - 2.f * y * GR[8]);
  const float gzq = 2.f * (-2.f * z * GR[0] - w * GR[1] + x * GR[2] + w * GR[3] -
                           2.f * z * GR[4] + y * GR[5] + x * GR[6] + y * GR[7]);
  const float dotq = gw * w + gxq * x + gyq * y + gzq * z;
  out.gq[0] = (gw - dotq * w) * iqn;
  out.gq[1] = (gxq - dotq * x) * iqn;
  out.gq[2] = (gyq - dotq * y) * iqn;
  out.gq[3] = (gzq - dotq * z) * iqn;
  // positions: g_pcam @ R_eff
#pragma unroll
  for (int k = 0; k < 3; ++k) out.gp[k] = gx * R[k] + gy * R[3 + k] + gz * R[6 + k];
  out.go = gop * o * (1.f - o);
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

// ------------------------------------------------------------------ Adam --
constexpr float kBeta1 = 0.9f, kBeta2 = 0.999f, kEps = 1e-15f;  // optim.py:12-14
// 1 - beta as the FP32 rounding of the exact decimal (1.f - 0.999f would be
// 0.00099998713, a 1.3e-5 relative bias on every second moment)
constexpr float kOneMinusBeta1 = 0.1f, kOneMinusBeta2 = 0.001f;

struct AdamGroups {
  tsr_adam_group_t g[TSR_MAX_ADAM_GROUPS];
  long long row_start[TSR_MAX_ADAM_GROUPS + 1];
  int n;
};

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

// Adam update of one row held in registers (optim.py:74-88); returns 1 when
// the row is skipped (non-finite gradient: moments and params untouched).
// Per-step scalars of one group: from the descriptor (by value), or from a
// device array [lr, bias_correction1, bias_correction2] x 5 that the host
// rewrites every step (CUDA-graph replay, where kernel arguments are frozen).
struct AdamScal {
  float lr, ibc1, ibc2;
};

__device__ __forceinline__ AdamScal adam_scal(const tsr_adam_group_t& G, const float* dev, int k) {
  if (dev) return {dev[3 * k], 1.0f / dev[3 * k + 1], 1.0f / dev[3 * k + 2]};
  return {G.lr, 1.0f / G.bias_correction1, 1.0f / G.bias_correction2};
}

template <int W>
__device__ __forceinline__ int adam_regs(const tsr_adam_group_t& G, const AdamScal& S,
                                         const float* g, float* p, float* m, float* v) {
  bool finite = true;
#pragma unroll
  for (int k = 0; k < W; ++k) finite &= isfinite(g[k]);
  if (!finite) return 1;
  const float ibc1 = S.ibc1, ibc2 = S.ibc2;
  float nrm = 0.f;
#pragma unroll
  for (int k = 0; k < W; ++k) {
    m[k] = kBeta1 * m[k] + kOneMinusBeta1 * g[k];
    v[k] = kBeta2 * v[k] + kOneMinusBeta2 * g[k] * g[k];
    p[k] = p[k] - __fdividef(S.lr * (m[k] * ibc1), sqrtf(v[k] * ibc2) + kEps);
    nrm += p[k] * p[k];
  }
  if (G.renormalize) {
    nrm = sqrtf(nrm);
    if (nrm > 0.f) {
      const float inv = 1.0f / nrm;
#pragma unroll
      for (int k = 0; k < W; ++k) p[k] = p[k] * inv;
    }
  }
  return 0;
}

template <int W>
__device__ __forceinline__ void load_row(const float* base, long long i, float* out) {
#pragma unroll
  for (int k = 0; k < W; ++k) out[k] = base[i * W + k];
}
template <int W>
__device__ __forceinline__ void store_row(float* base, long long i, const float* in) {
#pragma unroll
  for (int k = 0; k < W; ++k) base[i * W + k] = in[k];
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
  Vjp vj;
  bool vis = false;
  unsigned long long local = 0;
  if (i < n) {
    // two load phases (VJP inputs, then the moments) keep fewer registers
    // live than loading all 42 values up front, so 3 CTAs (24 warps) fit
    const tsr_adam_group_t &G0 = groups.g[0], &G1 = groups.g[1], &G2 = groups.g[2],
                           &G3 = groups.g[3], &G4 = groups.g[4];
    float pp[3], pl[3], pq[4], po[1], pc[3];
    load_row<3>(G0.param, i, pp);
    load_row<3>(G1.param, i, pl);
    load_row<4>(G2.param, i, pq);
    const int row = row_of_source[i];
    float gp[3] = {0.f, 0.f, 0.f}, gl[3] = {0.f, 0.f, 0.f}, gq[4] = {0.f, 0.f, 0.f, 0.f};
    float go[1] = {0.f}, gc[3] = {0.f, 0.f, 0.f};
    if (row >= 0) {
      vis = true;
      float* g2p = grad2d + (long long)row * TSR_GRAD2D_FLOATS;
      float g2[TSR_GRAD2D_FLOATS];
#pragma unroll
      for (int k = 0; k < TSR_GRAD2D_FLOATS; ++k) g2[k] = g2p[k];
      vjp_core(cam, pp[0], pp[1], pp[2], pl, pq, rec[3 * row], rec[3 * row + 1], g2, vj);
#pragma unroll
      for (int k = 0; k < TSR_GRAD2D_FLOATS; ++k) g2p[k] = 0.f;  // ready for the next step
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        gp[k] = vj.gp[k];
        gl[k] = vj.gls[k];
        gc[k] = vj.gcol[k];
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) gq[k] = vj.gq[k];
      go[0] = vj.go;
    }
    float mp[3], ml[3], mq[4], mo[1], mc[3];
    float vp[3], vl[3], vq[4], vo[1], vc[3];
    load_row<3>(G0.exp_avg, i, mp); load_row<3>(G0.exp_avg_sq, i, vp);
    load_row<3>(G1.exp_avg, i, ml); load_row<3>(G1.exp_avg_sq, i, vl);
    load_row<4>(G2.exp_avg, i, mq); load_row<4>(G2.exp_avg_sq, i, vq);
    load_row<1>(G3.param, i, po); load_row<1>(G3.exp_avg, i, mo); load_row<1>(G3.exp_avg_sq, i, vo);
    load_row<3>(G4.param, i, pc); load_row<3>(G4.exp_avg, i, mc); load_row<3>(G4.exp_avg_sq, i, vc);
    const AdamScal S0 = adam_scal(G0, scal, 0), S1 = adam_scal(G1, scal, 1),
                   S2 = adam_scal(G2, scal, 2), S3 = adam_scal(G3, scal, 3),
                   S4 = adam_scal(G4, scal, 4);
    local += adam_regs<3>(G0, S0, gp, pp, mp, vp);
    local += adam_regs<3>(G1, S1, gl, pl, ml, vl);
    local += adam_regs<4>(G2, S2, gq, pq, mq, vq);
    local += adam_regs<1>(G3, S3, go, po, mo, vo);
    local += adam_regs<3>(G4, S4, gc, pc, mc, vc);
    store_row<3>(G0.param, i, pp); store_row<3>(G0.exp_avg, i, mp); store_row<3>(G0.exp_avg_sq, i, vp);
    store_row<3>(G1.param, i, pl); store_row<3>(G1.exp_avg, i, ml); store_row<3>(G1.exp_avg_sq, i, vl);
    store_row<4>(G2.param, i, pq); store_row<4>(G2.exp_avg, i, mq); store_row<4>(G2.exp_avg_sq, i, vq);
    store_row<1>(G3.param, i, po); store_row<1>(G3.exp_avg, i, mo); store_row<1>(G3.exp_avg_sq, i, vo);
    store_row<3>(G4.param, i, pc); store_row<3>(G4.exp_avg, i, mc); store_row<3>(G4.exp_avg_sq, i, vc);
  }
  if (kPose) {
    float pv[12];
#pragma unroll
    for (int k = 0; k < 12; ++k) pv[k] = vis ? vj.pose[k] : 0.f;
    block_reduce_pose(pv, pose_sums);
  }
  for (int d = 16; d > 0; d >>= 1) local += __shfl_xor_sync(0xffffffffu, local, d);
  if ((threadIdx.x & 31) == 0 && local) atomicAdd(skipped, local);
}

// ---- fused ZeRO-1 update over peer memory (the B200 variant)
// One thread per (group, shard row): the gradient row is the sum of the
// ranks' rows read through peer pointers in rank order (bitwise the
// deterministic fixed-order reduction), Adam runs on the local parameter
// row with this rank's shard moments, and the updated row is stored into
// every rank's parameter buffer -- reduce-scatter + K5 + all-gather as one
// kernel, no collective library.
constexpr int kPeerMaxWorld = 8;
constexpr int kPeerMaxWidth = 48;  // colors at SH degree 3
struct PeerPtrs {
  const float* g[kPeerMaxWorld * TSR_MAX_ADAM_GROUPS];  // [rank * n_groups + group]
  float* p[kPeerMaxWorld * TSR_MAX_ADAM_GROUPS];
};

__global__ void __launch_bounds__(256) zero1_peer_adam_kernel(AdamGroups groups, PeerPtrs pp,
                                                              int world, long long row_begin,
                                                              unsigned long long* __restrict__ skipped) {
  const long long total = groups.row_start[groups.n];
  const int ng = groups.n;
  unsigned long long local = 0;
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    int gi = 0;
    while (t >= groups.row_start[gi + 1]) ++gi;
    const tsr_adam_group_t& G = groups.g[gi];
    const long long r = t - groups.row_start[gi];  // shard row (moments)
    const long long row = row_begin + r;           // parameter row
    const int w = G.width;
    float gsum[kPeerMaxWidth];
    bool finite = true;
    for (int k = 0; k < w; ++k) {
      float acc = pp.g[gi][row * w + k];
      for (int q = 1; q < world; ++q) acc += pp.g[q * ng + gi][row * w + k];
      gsum[k] = acc;
      finite &= isfinite(acc);
    }
    if (!finite) {
      ++local;
      continue;
    }
    float* p = G.param + row * w;
    float* m = G.exp_avg + r * w;
    float* v = G.exp_avg_sq + r * w;
    const float ibc1 = 1.0f / G.bias_correction1, ibc2 = 1.0f / G.bias_correction2;
    float nrm = 0.f;
    for (int k = 0; k < w; ++k) {
      const float gk = gsum[k];
      const float mk = kBeta1 * m[k] + kOneMinusBeta1 * gk;
      const float vk = kBeta2 * v[k] + kOneMinusBeta2 * gk * gk;
      m[k] = mk;
      v[k] = vk;
      const float pk = p[k] - __fdividef(G.lr * (mk * ibc1), sqrtf(vk * ibc2) + kEps);
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
    for (int q = 0; q < world; ++q) {  // all-gather by direct peer stores
      float* dst = pp.p[q * ng + gi] + row * w;
      if (dst == p) continue;
      for (int k = 0; k < w; ++k) dst[k] = p[k];
    }
  }
  for (int d = 16; d > 0; d >>= 1) local += __shfl_xor_sync(0xffffffffu, local, d);
  if ((threadIdx.x & 31) == 0 && local) atomicAdd(skipped, local);
}

static bool fill_groups(const tsr_adam_group_t* gh, int n, AdamGroups& out) {
  if (n <= 0 || n > TSR_MAX_ADAM_GROUPS) return false;
  out.n = n;
  out.row_start[0] = 0;
  for (int k = 0; k < n; ++k) {
    if (gh[k].width <= 0 || gh[k].rows < 0 || !gh[k].param) return false;
    out.g[k] = gh[k];
    out.row_start[k + 1] = out.row_start[k] + gh[k].rows;
  }
  return true;
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
  if (!fill_groups(groups_host, n_groups, gs) || !skipped) return TSR_E_INVALID;
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
  if (!fill_groups(groups_host, n_groups, gs) || !skipped || !group_scalars || scal_period < 1)
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
  if (!fill_groups(groups_host, n_groups, gs)) return TSR_E_INVALID;
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
  gs.row_start[0] = 0;
  for (int k = 0; k < n_groups; ++k) gs.row_start[k + 1] = gs.row_start[k] + (row_end - row_begin);
  const long long total = gs.row_start[n_groups];
  if (total == 0) return TSR_OK;
  long long blocks = (total + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  zero1_peer_adam_kernel<<<(int)blocks, 256, 0, (cudaStream_t)stream>>>(gs, pp, world, row_begin,
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
  if (!g || !cam || !fill_groups(groups_host, 5, gs) || !skipped) return TSR_E_INVALID;
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
