// K2: key duplication, stable on-device radix sort, per-tile ranges and the
// checkpoint record bases.
//
//   emission (splat-major)   binning.py:178-221 (sequential) / :262-286 (LB)
//   key = tile<<32 | f32 bits binning.py:137-139,152
//   stable LSD sort          binning.py:142-148  -> ties resolve by emission order
//   offsets (T+1)            binning.py:156-157
//   checkpoint count/tile    forward.py:139-145  (floor(n_tile / 32) records)
#include <cub/device/device_radix_sort.cuh>
#include <cuda_runtime.h>

#include "tsr_common.cuh"

namespace tsr {

__device__ __forceinline__ long long make_key(long long tile, float depth) {
  return (tile << 32) | (long long)__float_as_uint(depth);
}

// Sequential strategy: one thread walks one splat's SnugBox columns.
__global__ void duplicate_sequential_kernel(const float* __restrict__ rec, long long m,
                                            int tiles_x, int tiles_y,
                                            const int64_t* __restrict__ pair_offsets,
                                            int64_t* __restrict__ keys,
                                            int32_t* __restrict__ values) {
  long long row = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= m) return;
  const float* r = rec + row * 12;
  SplatF64 s = load_splat_f64(r);
  SnugRect box = snugbox(s, tiles_x, tiles_y);
  if (box.tx0 > box.tx1 || box.ty0 > box.ty1) return;
  const float depth = r[6];
  long long out = pair_offsets[row];
  for (long long tx = box.tx0; tx <= box.tx1; ++tx) {
    long long ty0, ty1;
    int n = column_rows(s, box, tx, tiles_y, ty0, ty1);
    for (int k = 0; k < n; ++k) {
      keys[out] = make_key((ty0 + k) * tiles_x + tx, depth);
      values[out] = (int32_t)row;
      ++out;
    }
  }
}

// Load-balanced strategy (bin_load_balanced, binning.py:262-286 and the
// paper's load-balanced writing): one warp per splat, the SnugBox candidate
// tiles are dealt round-robin to the 32 lanes (lane = within % 32,
// lane_test_counts binning.py:289-298); each lane runs the exact FP64
// min-q <= t test and hits are compacted with a warp ballot.
__global__ void duplicate_load_balanced_kernel(const float* __restrict__ rec, long long m,
                                               int tiles_x, int tiles_y,
                                               const int64_t* __restrict__ pair_offsets,
                                               int64_t* __restrict__ keys,
                                               int32_t* __restrict__ values) {
  const int lane = threadIdx.x & 31;
  long long row = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (row >= m) return;
  const float* r = rec + row * 12;
  SplatF64 s = load_splat_f64(r);
  SnugRect box = snugbox(s, tiles_x, tiles_y);
  if (box.tx0 > box.tx1 || box.ty0 > box.ty1) return;
  const long long nrows = box.ty1 - box.ty0 + 1;
  const long long ncand = (box.tx1 - box.tx0 + 1) * nrows;
  const float depth = r[6];
  long long out = pair_offsets[row];
  for (long long base = 0; base < ncand; base += 32) {
    long long w = base + lane;
    bool hit = false;
    long long tile = 0;
    if (w < ncand) {
      long long tx = box.tx0 + w / nrows;  // column-major candidate order
      long long ty = box.ty0 + w % nrows;
      double rx0 = dsub((double)(16 * tx), s.mx);
      double ry0 = dsub((double)(16 * ty), s.my);
      hit = min_q_box(s, rx0, dadd(rx0, 16.0), ry0, dadd(ry0, 16.0)) <= s.t;
      tile = ty * tiles_x + tx;
    }
    unsigned ballot = __ballot_sync(0xffffffffu, hit);
    if (hit) {
      long long slot = out + __popc(ballot & ((1u << lane) - 1u));
      keys[slot] = make_key(tile, depth);
      values[slot] = (int32_t)row;
    }
    out += __popc(ballot);
  }
}

// offsets[t] = first sorted index whose tile >= t, for t in [0, T].
__global__ void tile_ranges_kernel(const int64_t* __restrict__ keys, long long p, int n_tiles,
                                   int64_t* __restrict__ offsets) {
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i > p) return;
  long long cur = i < p ? (keys[i] >> 32) : (long long)n_tiles;
  long long prev = i == 0 ? -1 : (keys[i - 1] >> 32);
  for (long long t = prev + 1; t <= cur; ++t) offsets[t] = i;
}

// ckpt_base[t] = sum_{u<t} floor(n_u / 32); ckpt_base[T] = total records.
__global__ void __launch_bounds__(1024) ckpt_base_kernel(const int64_t* __restrict__ offsets,
                                                         int n_tiles,
                                                         int64_t* __restrict__ ckpt_base) {
  __shared__ long long s_warp[32];
  __shared__ long long s_carry;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) s_carry = 0;
  __syncthreads();
  for (int base = 0; base < n_tiles; base += 1024) {
    int t = base + threadIdx.x;
    long long v = t < n_tiles ? (offsets[t + 1] - offsets[t]) / kGroup : 0;
    long long incl = v;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      long long y = __shfl_up_sync(0xffffffffu, incl, d);
      if (lane >= d) incl += y;
    }
    if (lane == 31) s_warp[warp] = incl;
    __syncthreads();
    if (warp == 0) {
      long long w = s_warp[lane], wi = w;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        long long y = __shfl_up_sync(0xffffffffu, wi, d);
        if (lane >= d) wi += y;
      }
      s_warp[lane] = wi - w;
    }
    __syncthreads();
    long long carry = s_carry;
    if (t < n_tiles) ckpt_base[t] = carry + s_warp[warp] + incl - v;
    __syncthreads();
    if (threadIdx.x == 1023) s_carry = carry + s_warp[warp] + incl;
    __syncthreads();
  }
  if (threadIdx.x == 0) ckpt_base[n_tiles] = s_carry;
}

static int key_bits(int n_tiles) {
  int b = 0;
  while ((1 << b) < n_tiles) ++b;
  return 32 + (b == 0 ? 1 : b);
}

}  // namespace tsr

using namespace tsr;

extern "C" int tsr_duplicate_keys(const float* rec, int64_t m, int32_t width, int32_t height,
                                  const int64_t* pair_offsets, int64_t n_pairs,
                                  int32_t strategy, int64_t* keys, int32_t* values,
                                  void* stream) {
  if (m < 0 || width <= 0 || height <= 0 || n_pairs < 0) return TSR_E_INVALID;
  if (m == 0 || n_pairs == 0) return TSR_OK;
  cudaStream_t s = (cudaStream_t)stream;
  const int tx = tiles_of(width), ty = tiles_of(height);
  if (strategy == 1) {
    long long threads = m * 32;
    int blocks = (int)((threads + 255) / 256);
    duplicate_load_balanced_kernel<<<blocks, 256, 0, s>>>(rec, m, tx, ty, pair_offsets, keys,
                                                         values);
  } else {
    int blocks = (int)((m + 127) / 128);
    duplicate_sequential_kernel<<<blocks, 128, 0, s>>>(rec, m, tx, ty, pair_offsets, keys,
                                                      values);
  }
  TSR_CHECK_LAUNCH();
  return TSR_OK;
}

extern "C" size_t tsr_sort_workspace(int64_t n_pairs, int32_t n_tiles) {
  size_t bytes = 0;
  cub::DeviceRadixSort::SortPairs((void*)nullptr, bytes, (const unsigned long long*)nullptr,
                                  (unsigned long long*)nullptr, (const int32_t*)nullptr,
                                  (int32_t*)nullptr, (int64_t)(n_pairs > 0 ? n_pairs : 1), 0,
                                  key_bits(n_tiles));
  return bytes + 256;
}

extern "C" int tsr_sort_pairs(const int64_t* keys_in, int64_t* keys_out,
                              const int32_t* values_in, int32_t* values_out, int64_t n_pairs,
                              int32_t n_tiles, void* workspace, size_t workspace_bytes,
                              void* stream) {
  if (n_pairs < 0 || n_tiles <= 0) return TSR_E_INVALID;
  if (n_pairs == 0) return TSR_OK;
  size_t need = 0;
  cub::DeviceRadixSort::SortPairs((void*)nullptr, need, (const unsigned long long*)keys_in,
                                  (unsigned long long*)keys_out, values_in, values_out,
                                  (int64_t)n_pairs, 0, key_bits(n_tiles), (cudaStream_t)stream);
  if (workspace_bytes < need) return TSR_E_WORKSPACE;
  cudaError_t e = cub::DeviceRadixSort::SortPairs(
      workspace, need, (const unsigned long long*)keys_in, (unsigned long long*)keys_out,
      values_in, values_out, (int64_t)n_pairs, 0, key_bits(n_tiles), (cudaStream_t)stream);
  return e == cudaSuccess ? TSR_OK : TSR_E_CUDA;
}

extern "C" int tsr_tile_ranges(const int64_t* sorted_keys, int64_t n_pairs, int32_t n_tiles,
                               int64_t* offsets, int64_t* ckpt_base, void* stream) {
  if (n_pairs < 0 || n_tiles <= 0) return TSR_E_INVALID;
  cudaStream_t s = (cudaStream_t)stream;
  long long threads = n_pairs + 1;
  int blocks = (int)((threads + 255) / 256);
  tile_ranges_kernel<<<blocks, 256, 0, s>>>(sorted_keys, n_pairs, n_tiles, offsets);
  TSR_CHECK_LAUNCH();
  if (ckpt_base) {
    ckpt_base_kernel<<<1, 1024, 0, s>>>(offsets, n_tiles, ckpt_base);
    TSR_CHECK_LAUNCH();
  }
  return TSR_OK;
}
