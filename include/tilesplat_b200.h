/*
 * tilesplat_b200.h -- C-ABI of the B200-native differentiable tile rasterizer.
 *
 * Drop-in boundary for the hot path of the reference package `tilesplat`
 * (/root/reference/pkg/src/tilesplat, pure Python/NumPy).  The reference has
 * no FFI; its boundary is the Python API re-exported by tilesplat/__init__.py:6-20.
 * Each entry point below replaces one reference function (cited file:line).
 * The Python host package `paper_2601_19489_b200` binds these with ctypes and
 * keeps the reference names/signatures.
 *
 * Conventions
 *   - every pointer is a DEVICE pointer unless the name ends in `_host`;
 *   - `stream` is a cudaStream_t passed as void*; every call is stream-ordered,
 *     asynchronous, stateless and re-entrant (no global mutable state);
 *   - the library never allocates or frees caller memory; scratch comes from a
 *     caller-provided workspace sized by the matching *_workspace() query;
 *   - return 0 (TSR_OK) or a TSR_E_* code; the host raises the reference's
 *     exception types from these codes.
 *
 * Data layout in HBM (FP32 unless noted):
 *   raster record  rec[M][12] = {mx, my, a, b, c, opacity, depth, level_t,
 *                                r, g, b, 0}   (48 B, 16-B aligned rows)
 *     = SplatBatch.means2d/conics/opacities/depths/level_t + per-row RGB
 *   keys  [P] int64  = tile << 32 | bits(float32 depth)   (binning.py:137-152)
 *   values[P] int32  = batch row
 *   offsets[T+1] int64 (binning.py:156-157)
 *   grad2d[M][10] = {d_mx, d_my, d_a, d_b, d_c, d_opacity, d_r, d_g, d_b, d_depth}
 */
#ifndef TILESPLAT_B200_H
#define TILESPLAT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TSR_OK 0
#define TSR_E_INVALID 1   /* bad argument (shape, null pointer, limits)   */
#define TSR_E_CUDA 2      /* CUDA launch / runtime error                 */
#define TSR_E_CAPACITY 3  /* output capacity too small (caller retries)   */
#define TSR_E_WORKSPACE 4 /* workspace smaller than *_workspace() says    */

#define TSR_TILE 16
#define TSR_REC_FLOATS 12
#define TSR_GRAD2D_FLOATS 10
#define TSR_CKPT_INTERVAL 32
#define TSR_MAX_GAUSSIANS (1LL << 26)

/* Pinhole camera with the pose delta already folded in
 * (projection.py:73-78, pose.py:100-111). */
typedef struct {
  float fx, fy, cx, cy;
  int32_t width, height;
  float R[9];      /* effective world->camera rotation, row-major            */
  float t[3];      /* effective translation                                   */
  float center[3]; /* camera centre in world coordinates (SH view dirs)       */
  float near_plane;
} tsr_camera_t;

/* GaussianSet (scene.py:50-106) as FP32 SoA device arrays. */
typedef struct {
  const float* positions;      /* (N,3)            */
  const float* log_scales;     /* (N,3)            */
  const float* rotations;      /* (N,4) w,x,y,z    */
  const float* opacity_logits; /* (N,)             */
  const float* colors;         /* (N,C,3) SH coeff */
  int64_t n;
  int32_t sh_coeffs;           /* C = (deg+1)^2, deg <= 3 */
} tsr_gaussians_t;

/* ---------------------------------------------------------------- K1 ----
 * project + _splat_colors + compute_snugboxes + exact per-splat pair count
 * (projection.py:77-136, trainer.py:170-178, binning.py:87-104,166-215).
 * One pass: culled rows are compacted in source order by a single-pass
 * decoupled look-back scan.  Outputs (capacity N rows): rec, source_ids,
 * row_of_source (-1 if culled), counts[M] (pairs per row), depth_bits[M]
 * (f32 depth bits, binning.py:137-139), spans[M] (16-byte compact column
 * walk, see sort.cu), totals[0] = M, totals[1] = P (device).
 * strategy: 0 = bin_sequential column walk, 1 = bin_load_balanced min-q test,
 *           2 = bin_aabb radius rectangle (binning.py:301-325, the bench-tiling baseline)
 * (both yield the same pair multiset). */
size_t tsr_preprocess_workspace(int64_t n);
int tsr_preprocess_fwd(const tsr_gaussians_t* g, const tsr_camera_t* cam, int32_t strategy,
                       float* rec, int32_t* source_ids, int32_t* row_of_source, int32_t* counts,
                       uint32_t* depth_bits, void* spans, int64_t* totals, void* workspace,
                       size_t workspace_bytes, void* stream);

/* Same counts / depth bits / spans for a caller-built batch of m rows
 * (bin_sequential on a make_batch()-style SplatBatch, binning.py:166-215);
 * totals[0] = m, totals[1] = P (device). */
int tsr_count_pairs(const float* rec, int64_t m, int32_t width, int32_t height,
                    int32_t strategy, int32_t* counts, uint32_t* depth_bits, void* spans,
                    int64_t* totals, void* stream);

/* compute_snugboxes (binning.py:87-104): FP64 extents + inclusive tile rect
 * (int32 [tx0,tx1,ty0,ty1]). */
int tsr_snugboxes(const float* rec, int64_t m, int32_t width, int32_t height,
                  double* x_min, double* x_max, double* y_min, double* y_max,
                  int32_t* tile_rect, void* stream);

/* ---------------------------------------------------------------- K2 ----
 * TileIndex (binning.py:137-158) without a 64-bit key sort: stable one-sweep
 * radix sort of rows by depth bits -> rank-major emission of (tile, rank)
 * pairs -> stable one-sweep radix sort by tile -> keys = tile << 32 | depth
 * bits, values = row, offsets[T+1], ckpt_base[T+1] = offsets >> 5 (record r
 * of tile t at ckpt_base[t] + r; the tiles' floor(n_tile / 32) records never
 * overlap, forward.py:139-145).  M and P are read from `totals` on the device; the
 * capacities bound every buffer.  If P > p_cap the pairs are clamped and
 * *overflow (sticky, device int32) is set to 1: the caller re-runs with a
 * larger capacity. */
size_t tsr_index_workspace(int64_t m_cap, int64_t p_cap);
/* tsr_build_index plus what the deterministic merge needs: inv_perm[e] =
 * sorted position of emission index e (P_cap), and per depth rank the batch
 * row, pair count and emission offset (M_cap each). */
int tsr_build_index_det(const float* rec, const uint32_t* depth_bits, const void* spans,
                        const int32_t* counts, const int64_t* totals, int64_t m_cap,
                        int64_t p_cap, int32_t width, int32_t height, int32_t strategy,
                        int64_t* keys, int32_t* values, int64_t* offsets, int64_t* ckpt_base,
                        int32_t* overflow, void* workspace, size_t workspace_bytes,
                        uint32_t* inv_perm, uint32_t* rank_row, uint32_t* rank_count,
                        uint32_t* rank_off, void* stream);
int tsr_build_index(const float* rec, const uint32_t* depth_bits, const void* spans,
                    const int32_t* counts, const int64_t* totals, int64_t m_cap, int64_t p_cap,
                    int32_t width, int32_t height, int32_t strategy, int64_t* keys,
                    int32_t* values, int64_t* offsets, int64_t* ckpt_base, int32_t* overflow,
                    void* workspace, size_t workspace_bytes, void* stream);

/* ---------------------------------------------------------------- K3 ----
 * render (forward.py:87-161). ckpt may be NULL (record_checkpoints=False).
 * Checkpoint record r of tile t holds the (T, Cr, Cg, Cb, D) state after list
 * position 32(r+1)-1, laid out ckpt[((ckpt_base[t]+r)*5 + ch)*256 + local_px];
 * it is written for every pixel that consumed that position. */
int tsr_render_fwd(const float* rec, const int32_t* values, const int64_t* offsets,
                   int32_t width, int32_t height, const float* background_host,
                   float* out_color, float* out_depth, float* out_final_T,
                   int32_t* out_n_contrib, int32_t* out_n_considered,
                   float* ckpt, const int64_t* ckpt_base, void* stream);

/* Same with ckpt_stride 1 (every record, as above) or 2 (only the odd
 * records r = 1, 3, 5, ...: the supergroup starts tsr_render_bwd reads, half
 * the checkpoint traffic; the training step uses this). */
int tsr_render_fwd_ex(const float* rec, const int32_t* values, const int64_t* offsets,
                      int32_t width, int32_t height, const float* background_host,
                      float* out_color, float* out_depth, float* out_final_T,
                      int32_t* out_n_contrib, int32_t* out_n_considered, float* ckpt,
                      const int64_t* ckpt_base, int32_t ckpt_stride, void* stream);

/* K3 scoring mode (forward.py:132-137; density.py:36-76).  Re-renders the
 * view (same outputs as tsr_render_fwd, no checkpoints) and handles every
 * strong contribution (blend with w = T alpha >= 1/255):
 *   mode 1: warp_counts[t*4 + w] = strong contributions of warp w of tile t
 *   mode 2: writes (pixel index, batch row) pairs at warp_base[t*4 + w]
 *           (exclusive scan of mode 1's counts): the reference's
 *           Contributions, in (tile, warp, list position, lane) order
 *   mode 3: row_score[row] += weight for each strong contribution to a pixel
 *           with mask[pixel] != 0 (the fused density scoring pass). */
int tsr_render_score(const float* rec, const int32_t* values, const int64_t* offsets,
                     int32_t width, int32_t height, const float* background_host, int32_t mode,
                     const uint8_t* mask, float weight, float* row_score, int64_t* warp_counts,
                     const int64_t* warp_base, int64_t* out_pixel, int64_t* out_row,
                     float* out_color, float* out_depth, float* out_final_T,
                     int32_t* out_n_contrib, int32_t* out_n_considered, void* stream);

/* Launch order for the per-tile kernels: heavy tiles (list longer than 4x
 * the mean) first in raster order, then the rest in raster order (one CTA;
 * order is (n_tiles + 1,) int32, order[n_tiles] = 0 when there is no heavy
 * tile -- raster order, nothing else written).  tsr_render_fwd_ordered / tsr_render_bwd_ordered
 * take it (NULL: raster order) -- the same outputs, the heavy tiles no longer
 * finish last (C3-lo). */
int tsr_tile_order(const int64_t* offsets, int32_t n_tiles, int32_t* order, void* stream);
int tsr_render_fwd_ordered(const float* rec, const int32_t* values, const int64_t* offsets,
                           int32_t width, int32_t height, const float* background_host,
                           float* out_color, float* out_depth, float* out_final_T,
                           int32_t* out_n_contrib, int32_t* out_n_considered, float* ckpt,
                           const int64_t* ckpt_base, int32_t ckpt_stride,
                           const int32_t* tile_order, void* stream);

/* ---------------------------------------------------------------- K4 ----
 * backward_per_gaussian (backward.py:137-223): a warp owns a supergroup of
 * 64 list positions (two checkpoint groups, lane j the splat pair 2j, 2j+1)
 * and runs a systolic pipeline over the pixels that entered it, restarting
 * from the checkpoint record: lane j takes (T, R) from lane j-1 by one
 * shuffle per step; one merged atomic write per (splat pair, supergroup).
 * grad2d must be zeroed by the caller.  grad_depth / grad_final_T are
 * nullable.  merges (device, u64) counts (splat, tile) merges with the
 * reference's semantics.
 *
 * tsr_render_bwd: one CTA (4 warps) per tile, the warps taking the tile's
 * supergroups.  tsr_render_bwd_ws (the product path): the (tile,
 * supergroup) work units of the whole frame go to a global queue that every
 * warp of a persistent grid drains, each warp compacting its unit's active
 * pixels with their checkpoint state into its own shared-memory records --
 * heavy tiles spread over the whole GPU and no warp idles at a tile's end.
 * It needs a workspace of tsr_render_bwd_workspace(width, height, p_bound)
 * bytes, p_bound >= the pair count (a capacity is fine). */
int tsr_render_bwd_ordered(const float* rec, const int32_t* values, const int64_t* offsets,
                           int32_t width, int32_t height, const float* color, const float* depth,
                           const float* final_T, const int32_t* n_considered, const float* ckpt,
                           const int64_t* ckpt_base, const float* grad_color,
                           const float* grad_depth, const float* grad_final_T, float* grad2d,
                           unsigned long long* merges, const int32_t* tile_order, void* stream);
size_t tsr_render_bwd_workspace(int32_t width, int32_t height, int64_t p_bound);

/* Region-culled K3 + K4 (the training step's pair; replaces the
 * tsr_render_fwd_ordered(ckpt_stride 2) + tsr_render_bwd_ordered pair behind
 * backward_per_gaussian, backward.py:137-223).  tsr_render_fwd_regions is K3
 * writing checkpoint records only at segment starts (every 1024 list
 * positions) plus, per (tile, region), the list positions that blend at >= 1
 * pixel of the region (regions of 8 x region_height pixels, region_height 8
 * or 4; both calls take the same value), and the backward's streams (one
 * per (tile, 1024-position segment, region) with entries), filed as each
 * tile finishes under the bucket of the stream's length:
 *   region_list   tsr_region_list_entries(...) uint32 ((position, row) pairs)
 *   region_seg    tsr_region_seg_entries(...) int32
 *   region_units  tsr_region_unit_entries(...) uint32 (72 length buckets)
 *   region_ctl    tsr_region_ctl_entries() int32 (bucket counts, grab
 *                 counter; zeroed by tsr_render_fwd_regions).
 * tsr_render_bwd_regions streams each region's list past its pixels (one
 * systolic pipeline of 8 (region_height 4) or 16 lanes per stream; a warp's
 * lane groups take streams of near-equal length, longest first) and merges
 * the same Grad2D sums with atomics.
 * p_bound >= the pair count (a capacity is fine). */
int tsr_render_fwd_regions(const float* rec, const int32_t* values, const int64_t* offsets,
                           int32_t width, int32_t height, const float* background_host,
                           float* out_color, float* out_depth, float* out_final_T,
                           int32_t* out_n_contrib, int32_t* out_n_considered, float* ckpt,
                           const int64_t* ckpt_base, uint32_t* region_list, int32_t* region_seg,
                           uint32_t* region_units, int32_t* region_ctl, int32_t region_height,
                           const int32_t* tile_order, void* stream);
size_t tsr_region_list_entries(int32_t width, int32_t height, int64_t p_bound);
size_t tsr_region_seg_entries(int32_t width, int32_t height, int64_t p_bound);
size_t tsr_region_unit_entries(int32_t width, int32_t height, int64_t p_bound);
size_t tsr_region_ctl_entries(void);
int tsr_render_bwd_regions(const float* rec, const int32_t* values, const int64_t* offsets,
                           int32_t width, int32_t height, const float* color, const float* depth,
                           const float* final_T, const int32_t* n_considered, const float* ckpt,
                           const int64_t* ckpt_base, const uint32_t* region_list,
                           const int32_t* region_seg, const uint32_t* region_units,
                           int32_t* region_ctl, const float* grad_color,
                           const float* grad_depth, const float* grad_final_T, float* grad2d,
                           unsigned long long* merges, int32_t region_height, void* stream);
int tsr_render_bwd_ws(const float* rec, const int32_t* values, const int64_t* offsets,
                      int32_t width, int32_t height, const float* color, const float* depth,
                      const float* final_T, const int32_t* n_considered, const float* ckpt,
                      const int64_t* ckpt_base, const float* grad_color,
                      const float* grad_depth, const float* grad_final_T, float* grad2d,
                      unsigned long long* merges, int64_t p_bound, void* workspace,
                      size_t workspace_bytes, void* stream);
int tsr_render_bwd(const float* rec, const int32_t* values, const int64_t* offsets,
                   int32_t width, int32_t height, const float* color,
                   const float* depth, const float* final_T,
                   const int32_t* n_considered, const float* ckpt,
                   const int64_t* ckpt_base, const float* grad_color,
                   const float* grad_depth, const float* grad_final_T,
                   float* grad2d, unsigned long long* merges, void* stream);

/* Deterministic merge (bitwise run-to-run reproducible): K4 writes each
 * processed (splat, tile) pair's 10 scaled sums to slots[pair] (P x 10
 * floats, no atomics; processed[t] = list positions tile t processed), then
 * one thread per depth rank sums its row's slots in emission order into
 * grad2d (overwritten: no zeroing needed), using tsr_build_index_det's
 * outputs.  The row count is m, or *m_dev when m_dev is not NULL and smaller
 * (capacity launches without a host read). */
int tsr_render_bwd_det(const float* rec, const int32_t* values, const int64_t* offsets,
                       int32_t width, int32_t height, const float* color, const float* depth,
                       const float* final_T, const int32_t* n_considered, const float* ckpt,
                       const int64_t* ckpt_base, const float* grad_color,
                       const float* grad_depth, const float* grad_final_T,
                       unsigned long long* merges, float* slots, int32_t* processed,
                       const uint32_t* inv_perm, const uint32_t* rank_row,
                       const uint32_t* rank_count, const uint32_t* rank_off,
                       const int64_t* keys, int64_t m, const int64_t* m_dev, float* grad2d,
                       void* stream);
/* the deterministic merge on the work-unit K4 (same slots/processed contract;
 * processed[] is written by the call) */
int tsr_render_bwd_ws_det(const float* rec, const int32_t* values, const int64_t* offsets,
                          int32_t width, int32_t height, const float* color, const float* depth,
                          const float* final_T, const int32_t* n_considered, const float* ckpt,
                          const int64_t* ckpt_base, const float* grad_color,
                          const float* grad_depth, const float* grad_final_T,
                          unsigned long long* merges, float* slots, int32_t* processed,
                          const uint32_t* inv_perm, const uint32_t* rank_row,
                          const uint32_t* rank_count, const uint32_t* rank_off,
                          const int64_t* keys, int64_t m, const int64_t* m_dev, float* grad2d,
                          int64_t p_bound, void* workspace, size_t workspace_bytes,
                          void* stream);

/* --------------------------------------------------------------- K4b ----
 * project_vjp + SH/colour chain (projection.py:139-241, trainer.py:231-257,
 * scene.py:279-291).  Writes (not accumulates) per-Gaussian gradients for
 * every source row: culled rows get zeros.  pose_sums (device, 12 floats,
 * accumulated) = {sum_rows J^T G_A + g_pcam p^T (3x3 row-major), sum g_pcam}.
 * grad_* are (N,3),(N,3),(N,4),(N,),(N,C,3).  accumulate != 0 adds into them
 * (multi-view gradient accumulation). */
int tsr_preprocess_bwd(const tsr_gaussians_t* g, const tsr_camera_t* cam,
                       const float* rec, const int32_t* row_of_source,
                       const float* grad2d, float* grad_positions,
                       float* grad_log_scales, float* grad_rotations,
                       float* grad_opacity_logits, float* grad_colors,
                       float* pose_sums, int32_t accumulate, void* stream);

/* ---------------------------------------------------------------- K5 ----
 * Adam.step (optim.py:60-88): dense bias-corrected update of every row,
 * non-finite gradient rows skipped (moments and params untouched) and
 * counted into *skipped (device, accumulated), quaternion rows renormalised.
 * lr / bias corrections are precomputed on the host in FP64. */
typedef struct {
  float* param;
  const float* grad;
  float* exp_avg;
  float* exp_avg_sq;
  int64_t rows;
  int32_t width;        /* floats per row */
  int32_t renormalize;  /* 1 for the rotation group */
  float lr;
  float bias_correction1; /* 1 - beta1^t */
  float bias_correction2; /* 1 - beta2^t */
} tsr_adam_group_t;

#define TSR_MAX_ADAM_GROUPS 8
int tsr_adam_step(const tsr_adam_group_t* groups_host, int32_t n_groups,
                  unsigned long long* skipped, void* stream);
/* tsr_adam_step with the per-step scalars from device memory: group k uses
 * group_scalars[3 (k % scal_period) + {0, 1, 2}] = {lr, bias_correction1,
 * bias_correction2} (CUDA-graph replay of the view-parallel step). */
int tsr_adam_step_dev(const tsr_adam_group_t* groups_host, int32_t n_groups,
                      const float* group_scalars, int32_t scal_period,
                      unsigned long long* skipped, void* stream);

/* Fused ZeRO-1 update over peer memory (SURVEY §8(e), B200 variant;
 * replaces the reference's single-process Adam.step, optim.py:60-88, in a
 * G-rank view-parallel step).  For the shard rows [row_begin, row_end) of
 * every group k: g = sum over ranks q = 0..world-1, in rank order, of
 * peer_grads[q * n_groups + k] (full-size (N, width) gradient buffers, device
 * pointers valid in this process: CUDA IPC / peer mappings); Adam on
 * groups[k].param (full-size, local) with groups[k].exp_avg / exp_avg_sq
 * holding ONLY the shard's moments (row 0 = row_begin); the updated row is
 * stored into every peer_params[q * n_groups + k].  groups[k].grad and
 * .rows are ignored.  world <= 8, width <= 48.  The caller orders the ranks:
 * every rank's gradients complete before any launch, every launch complete
 * before the parameters are read again. */
int tsr_zero1_peer_adam(const tsr_adam_group_t* groups_host, int32_t n_groups, int32_t world,
                        const float* const* peer_grads, float* const* peer_params,
                        int64_t row_begin, int64_t row_end, unsigned long long* skipped,
                        void* stream);

/* K4b fused with K5 for the single-view training step: the per-Gaussian
 * gradient never leaves registers.  groups_host[0..4] = positions,
 * log_scales, rotations, opacity_logits, colors (grad pointers ignored).
 * For SH degree 0 the consumed grad2d rows are zeroed in place (the buffer
 * is ready for the next step's K4 without a memset). */
int tsr_preprocess_bwd_adam(const tsr_gaussians_t* g, const tsr_camera_t* cam,
                            const float* rec, const int32_t* row_of_source,
                            const float* grad2d,
                            const tsr_adam_group_t* groups_host,
                            float* pose_sums, unsigned long long* skipped,
                            void* stream);

/* Same, with the per-step scalars read from DEVICE memory when group_scalars
 * is not NULL: [lr, bias_correction1, bias_correction2] for each of the 5
 * groups (the descriptors' own lr / bias corrections are then ignored).  A
 * CUDA graph that captures this launch replays with the scalars the host
 * writes each step (pinned-memory copy node), since kernel arguments are
 * frozen at capture. */
int tsr_preprocess_bwd_adam_dev(const tsr_gaussians_t* g, const tsr_camera_t* cam,
                                const float* rec, const int32_t* row_of_source,
                                const float* grad2d, const tsr_adam_group_t* groups_host,
                                const float* group_scalars, float* pose_sums,
                                unsigned long long* skipped, void* stream);

/* tsr_preprocess_bwd_adam_dev with an overflow gate (nullable): when *gate is
 * non-zero (K2's sticky pair-capacity overflow flag of this step) the update
 * is skipped -- params and moments untouched, consumed Grad2D rows zeroed --
 * and *gated_steps (nullable) is incremented, so the host can grow the
 * capacity and redo exactly the skipped steps.  Training-loop guard, no
 * reference counterpart (the reference has no capacities).  loss_guard
 * (nullable, device scalar): a non-finite loss skips the update too, the
 * reference's divergence guard before Adam (trainer.py:331-338). */
int tsr_preprocess_bwd_adam_ex(const tsr_gaussians_t* g, const tsr_camera_t* cam,
                               const float* rec, const int32_t* row_of_source,
                               const float* grad2d, const tsr_adam_group_t* groups_host,
                               const float* group_scalars, float* pose_sums,
                               unsigned long long* skipped, const int32_t* gate,
                               int32_t* gated_steps, const float* loss_guard, void* stream);

/* K4 with the projection VJP + Adam fused into its tail (SH 0 training step;
 * replaces tsr_render_bwd_ordered + tsr_preprocess_bwd_adam_ex).  Each tile
 * CTA, after its merges, counts its pairs into row_done[row]; the CTA that
 * brings a row to counts[row] (K1's pair count) runs that Gaussian's VJP and
 * Adam update (source_ids maps rows to Gaussians) and zeroes its Grad2D row.
 * A second kernel updates the Gaussians without pairs (culled, or no tile)
 * and re-arms row_done (zero-filled once by the caller).  Adam scalars from
 * group_scalars (device, [lr, bc1, bc2] x 5) when not NULL; gate /
 * gated_steps / loss_guard as in tsr_preprocess_bwd_adam_ex. */
int tsr_render_bwd_adam(const float* rec, const int32_t* values, const int64_t* offsets,
                        int32_t width, int32_t height, const float* color, const float* depth,
                        const float* final_T, const int32_t* n_considered, const float* ckpt,
                        const int64_t* ckpt_base, const float* grad_color,
                        const float* grad_depth, const float* grad_final_T, float* grad2d,
                        unsigned long long* merges, const int32_t* tile_order,
                        const tsr_gaussians_t* g, const tsr_camera_t* cam,
                        const tsr_adam_group_t* groups_host, const float* group_scalars,
                        const int32_t* source_ids, const int32_t* row_of_source,
                        const int32_t* counts, int32_t* row_done, unsigned long long* skipped,
                        const int32_t* gate, int32_t* gated_steps, const float* loss_guard,
                        void* stream);

/* ---------------------------------------------------------- depth chain ----
 * Disparity loss on the normalised render depth and its chain to the raster
 * outputs (losses.py:94-112 + trainer.py:201-214): mask = n_contrib > 0
 * [& valid (u8, nullable)], d = depth / (1 - final_T), L = w mean_mask
 * |1/max(d,eps) - 1/max(prior,eps)|, grad_depth / grad_final_T written for
 * every pixel (zero outside the mask).  The weight is *weight_dev when not
 * NULL (graph replay), else `weight`.  loss_out / total_out (nullable, device
 * scalars): L and *e_photo + L.  workspace: tsr_depth_chain_workspace()
 * bytes, zero-filled once before the first call (it re-arms itself). */
size_t tsr_depth_chain_workspace(void);
int tsr_depth_chain(const float* depth, const float* final_T, const int32_t* n_contrib,
                    const float* prior, const uint8_t* valid, int32_t height, int32_t width,
                    float weight, const float* weight_dev, const float* e_photo, float* loss_out,
                    float* total_out, float* grad_depth, float* grad_final_T, void* workspace,
                    size_t workspace_bytes, void* stream);

/* --------------------------------------------------------------- loss ----
 * Fused photometric objective (losses.py:44-91): E = (1-lam) mean|r-g| +
 * lam (1 - SSIM), 11-tap sigma=1.5 Gaussian window, zero padding.  rendered,
 * gt, grad are (H, W, 3) FP32; out3 (device) = {E, l1, ssim}. */
size_t tsr_photometric_workspace(int32_t height, int32_t width);
int tsr_photometric(const float* rendered, const float* gt, int32_t height, int32_t width,
                    float lam, float* grad, float* out3, void* workspace,
                    size_t workspace_bytes, void* stream);

/* Version / build string (for smoke checks). */
const char* tsr_version(void);

#ifdef __cplusplus
}
#endif
#endif /* TILESPLAT_B200_H */
