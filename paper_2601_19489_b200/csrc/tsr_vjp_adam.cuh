// Per-Gaussian projection VJP and Adam in registers, shared by the fused
// K4b+K5 kernels (vjp_adam.cu) and K4's fused per-row epilogue (backward.cu).
//   project_vjp   projection.py:139-241
//   Adam.step     optim.py:60-88
#pragma once
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


// One Gaussian of the SH-0 training step: its VJP from the packed Grad2D
// row (row >= 0; the row is read from L2 -- other CTAs merged into it with
// atomics -- and zeroed for the next step), then Adam on its five groups
// (update == false: gradient consumed, parameters and moments untouched).
// Returns the number of skipped (non-finite) rows; *vis says whether the
// Gaussian was visible, pose (kPose) receives its pose terms.  kL2: read the
// Grad2D row from L2 (rows merged by other CTAs inside the same kernel).
template <bool kPose, bool kL2 = false>
__device__ __forceinline__ unsigned vjp_adam_row_sh0(const tsr_camera_t& cam,
                                                     const AdamGroups& groups, long long i,
                                                     int row, const float4* __restrict__ rec,
                                                     float* __restrict__ grad2d,
                                                     const float* __restrict__ scal, bool update,
                                                     float* pose, bool& vis) {
  const tsr_adam_group_t &G0 = groups.g[0], &G1 = groups.g[1], &G2 = groups.g[2],
                         &G3 = groups.g[3], &G4 = groups.g[4];
  float pp[3], pl[3], pq[4], po[1], pc[3];
  load_row<3>(G0.param, i, pp);
  load_row<3>(G1.param, i, pl);
  load_row<4>(G2.param, i, pq);
  float gp[3] = {0.f, 0.f, 0.f}, gl[3] = {0.f, 0.f, 0.f}, gq[4] = {0.f, 0.f, 0.f, 0.f};
  float go[1] = {0.f}, gc[3] = {0.f, 0.f, 0.f};
  vis = false;
  if (row >= 0) {
    vis = true;
    float* g2p = grad2d + (long long)row * TSR_GRAD2D_FLOATS;
    float g2[TSR_GRAD2D_FLOATS];
#pragma unroll
    for (int k = 0; k < TSR_GRAD2D_FLOATS; ++k) g2[k] = kL2 ? __ldcg(g2p + k) : g2p[k];
    Vjp vj;
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
    if (kPose) {
#pragma unroll
      for (int k = 0; k < 12; ++k) pose[k] = vj.pose[k];
    }
  }
  if (!update) return 0u;
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
  unsigned skipped = 0;
  skipped += adam_regs<3>(G0, S0, gp, pp, mp, vp);
  skipped += adam_regs<3>(G1, S1, gl, pl, ml, vl);
  skipped += adam_regs<4>(G2, S2, gq, pq, mq, vq);
  skipped += adam_regs<1>(G3, S3, go, po, mo, vo);
  skipped += adam_regs<3>(G4, S4, gc, pc, mc, vc);
  store_row<3>(G0.param, i, pp); store_row<3>(G0.exp_avg, i, mp); store_row<3>(G0.exp_avg_sq, i, vp);
  store_row<3>(G1.param, i, pl); store_row<3>(G1.exp_avg, i, ml); store_row<3>(G1.exp_avg_sq, i, vl);
  store_row<4>(G2.param, i, pq); store_row<4>(G2.exp_avg, i, mq); store_row<4>(G2.exp_avg_sq, i, vq);
  store_row<1>(G3.param, i, po); store_row<1>(G3.exp_avg, i, mo); store_row<1>(G3.exp_avg_sq, i, vo);
  store_row<3>(G4.param, i, pc); store_row<3>(G4.exp_avg, i, mc); store_row<3>(G4.exp_avg_sq, i, vc);
  return skipped;
}

inline bool fill_adam_groups(const tsr_adam_group_t* gh, int n, AdamGroups& out) {
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

// vjp_adam.cu: Adam of the rows K4's fused epilogue does not reach
int tsr_launch_vjp_adam_rest(const tsr_camera_t& cam, long long n, const float* rec,
                             const int32_t* row_of_source, const int32_t* counts,
                             int32_t* row_done, float* grad2d, const tsr::AdamGroups& gs,
                             unsigned long long* skipped, const float* scal, const int32_t* gate,
                             int32_t* gated_steps, const float* loss_guard, cudaStream_t s);
