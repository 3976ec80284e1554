// K2: depth-sorted per-tile index without a 64-bit key sort.
//
// The reference builds key = tile << 32 | bits(f32 depth) per (tile, splat)
// pair, emitted splat-major, and sorts it with a stable LSD radix sort
// (binning.py:137-158), so ties resolve by emission (= batch row) order.  The
// same order is produced here with far less traffic:
//   1. stable LSD radix sort of the M rows by their 32-bit depth bits
//      (4 x 8-bit passes over 8 B per row)  -> depth rank r of every row;
//      rank order == (depth bits, row) order, exactly the reference's tie rule;
//   2. exclusive scan of pair counts in rank order, then emission of
//      (tile, r) pairs rank-major from K1's compact column spans (no FP64
//      re-walk unless a splat's span did not fit the 16-byte record);
//   3. stable LSD radix sort of the pairs by tile (8-bit digits, 2 passes
//      for up to 65536 tiles)                 -> within a tile, rank order;
//   4. finalize: keys = tile << 32 | depth bits[r], values = row[r], and the
//      per-tile ranges + checkpoint bases.
// Every size (M, P) is read from device memory: the whole pipeline runs
// without a host synchronisation and can be captured in a CUDA graph.  The
// radix passes are the classic three-kernel form (CTA histograms -> one
// decoupled look-back scan -> stable scatter ranked with __match_any_sync).
#include <cuda_runtime.h>

#include "tsr_common.cuh"

namespace tsr {

constexpr int kSB = 256;                 // threads per CTA
constexpr int kSItems = 16;              // items per thread
constexpr int kSTile = kSB * kSItems;    // 4096 items per CTA
constexpr int kBins = 256;               // 8-bit digits

__device__ __forceinline__ long long clamp_n(const long long* n_dev, long long n_cap) {
  const long long n = *n_dev;
  return n < n_cap ? (n > 0 ? n : 0) : n_cap;
}

// ------------------------------------------------------------ scan (u32) --
// Exclusive scan with a decoupled look-back; value(i) = in[gather ? gather[i] : i].
constexpr int kScanItems = 8;
constexpr int kScanTile = kSB * kScanItems;

__device__ __forceinline__ void st_rel(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_rel(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__global__ void __launch_bounds__(kSB) scan_u32_kernel(const uint32_t* __restrict__ in,
                                                       const int32_t* __restrict__ gather,
                                                       uint32_t* __restrict__ out,
                                                       const long long* __restrict__ n_dev,
                                                       long long n_cap,
                                                       unsigned long long* __restrict__ status,
                                                       unsigned int* __restrict__ ticket) {
  __shared__ uint32_t s_warp[kSB / 32];
  __shared__ uint32_t s_prefix;
  __shared__ int s_bid;
  if (threadIdx.x == 0) s_bid = (int)atomicAdd(ticket, 1u);
  __syncthreads();
  const int bid = s_bid;
  const long long n = n_dev ? clamp_n(n_dev, n_cap) : n_cap;
  const long long base = (long long)bid * kScanTile + (long long)threadIdx.x * kScanItems;
  uint32_t v[kScanItems];
  uint32_t sum = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    const long long i = base + k;
    uint32_t x = 0;
    if (i < n) x = in[gather ? (long long)gather[i] : i];
    v[k] = sum;
    sum += x;
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t incl = sum;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t t = __shfl_up_sync(0xffffffffu, incl, d);
    if (lane >= d) incl += t;
  }
  if (lane == 31) s_warp[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    const uint32_t w = lane < kSB / 32 ? s_warp[lane] : 0u;
    uint32_t wi = w;
#pragma unroll
    for (int d = 1; d < kSB / 32; d <<= 1) {
      const uint32_t t = __shfl_up_sync(0xffffffffu, wi, d);
      if (lane >= d) wi += t;
    }
    const uint32_t agg = __shfl_sync(0xffffffffu, wi, kSB / 32 - 1);
    if (lane < kSB / 32) s_warp[lane] = wi - w;
    if (lane == 0) {
      uint32_t excl = 0;
      if (bid == 0) {
        st_rel(&status[0], (2ull << 62) | agg);
      } else {
        st_rel(&status[bid], (1ull << 62) | agg);
        for (int j = bid - 1;; --j) {
          unsigned long long s;
          do {
            s = ld_rel(&status[j]);
          } while ((s >> 62) == 0);
          excl += (uint32_t)(s & 0xffffffffull);
          if ((s >> 62) == 2) break;
        }
        st_rel(&status[bid], (2ull << 62) | (uint32_t)(excl + agg));
      }
      s_prefix = excl;
    }
  }
  __syncthreads();
  const uint32_t off = s_prefix + s_warp[warp] + (incl - sum);
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    const long long i = base + k;
    if (i < n) out[i] = off + v[k];
  }
}

// ------------------------------------------------------------ radix sort --
__global__ void __launch_bounds__(kSB) radix_hist_kernel(const uint32_t* __restrict__ keys,
                                                         const long long* __restrict__ n_dev,
                                                         long long n_cap, int shift, int n_ctas,
                                                         uint32_t* __restrict__ hist) {
  __shared__ uint32_t s_h[kBins];
  s_h[threadIdx.x] = 0;
  __syncthreads();
  const long long n = clamp_n(n_dev, n_cap);
  const long long base = (long long)blockIdx.x * kSTile;
#pragma unroll 4
  for (int k = 0; k < kSItems; ++k) {
    const long long i = base + (long long)k * kSB + threadIdx.x;
    if (i < n) atomicAdd(&s_h[(keys[i] >> shift) & (kBins - 1)], 1u);
  }
  __syncthreads();
  hist[(long long)threadIdx.x * n_ctas + blockIdx.x] = s_h[threadIdx.x];
}

// Stable scatter: warp w owns items [base + 512 w, base + 512 (w+1)), ranked
// round by round with __match_any_sync; per-warp digit counters in shared
// memory are prefixed over warps so CTA-local ranks follow input order.
__global__ void __launch_bounds__(kSB) radix_scatter_kernel(
    const uint32_t* __restrict__ keys_in, const uint32_t* __restrict__ vals_in,
    uint32_t* __restrict__ keys_out, uint32_t* __restrict__ vals_out,
    const long long* __restrict__ n_dev, long long n_cap, int shift, int n_ctas,
    const uint32_t* __restrict__ hist_scan) {
  __shared__ uint32_t s_cnt[kSB / 32][kBins];
  __shared__ uint32_t s_base[kBins];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int w = 0; w < kSB / 32; ++w) s_cnt[w][threadIdx.x] = 0;
  s_base[threadIdx.x] = hist_scan[(long long)threadIdx.x * n_ctas + blockIdx.x];
  __syncthreads();
  const long long n = clamp_n(n_dev, n_cap);
  const long long wbase = (long long)blockIdx.x * kSTile + (long long)warp * (kSItems * 32);
  const unsigned lt = (1u << lane) - 1u;
  uint32_t packed[kSItems];  // digit << 16 | rank within warp (< 512)
#pragma unroll
  for (int r = 0; r < kSItems; ++r) {
    const long long i = wbase + r * 32 + lane;
    const bool valid = i < n;
    const uint32_t d = valid ? (keys_in[i] >> shift) & (kBins - 1) : 0u;
    const unsigned peers = __match_any_sync(0xffffffffu, valid ? d : (kBins + lane));
    const uint32_t before = __popc(peers & lt);
    uint32_t cnt = 0;
    if (valid) cnt = s_cnt[warp][d];
    __syncwarp();
    if (valid && before == 0) s_cnt[warp][d] = cnt + __popc(peers);
    __syncwarp();
    packed[r] = (d << 16) | (cnt + before);
  }
  __syncthreads();
  {
    uint32_t run = 0;
#pragma unroll
    for (int w = 0; w < kSB / 32; ++w) {
      const uint32_t c = s_cnt[w][threadIdx.x];
      s_cnt[w][threadIdx.x] = run;
      run += c;
    }
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < kSItems; ++r) {
    const long long i = wbase + r * 32 + lane;
    if (i < n) {
      const uint32_t d = packed[r] >> 16;
      const uint32_t pos = s_base[d] + s_cnt[warp][d] + (packed[r] & 0xffffu);
      keys_out[pos] = keys_in[i];
      vals_out[pos] = vals_in ? vals_in[i] : (uint32_t)i;
    }
  }
}

// ------------------------------------------------------------- emission --
// Compact column-walk record written by K1 (see preprocess.cu):
//   x = tx0 | ncols << 16,  y = ty_base | overflow << 31,
//   z, w = 8 columns x (row offset 4 bits | nrows 4 bits)
__global__ void __launch_bounds__(kSB) emit_pairs_kernel(
    const float* __restrict__ rec, const uint4* __restrict__ spans,
    const uint32_t* __restrict__ order, const uint32_t* __restrict__ off_rank,
    const long long* __restrict__ totals, long long m_cap, long long p_cap, int tiles_x,
    int tiles_y, int strategy, uint32_t* __restrict__ tile_out, uint32_t* __restrict__ rank_out,
    int* __restrict__ overflow) {
  const long long m = clamp_n(totals, m_cap);
  const long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= m) return;
  if (r == 0 && totals[1] > p_cap && overflow) *overflow = 1;  // sticky
  const uint32_t row = order[r];
  long long out = off_rank[r];
  const uint4 sp = spans[row];
  if (strategy == 0 && !(sp.y >> 31)) {
    const int tx0 = (int)(sp.x & 0xffffu), ncols = (int)(sp.x >> 16);
    const int ty_base = (int)(sp.y & 0xffffu);
    for (int c = 0; c < ncols; ++c) {
      const uint32_t code = ((c < 4 ? sp.z : sp.w) >> (8 * (c & 3))) & 0xffu;
      const int ty0 = ty_base + (int)(code & 15u), nr = (int)(code >> 4);
      for (int k = 0; k < nr; ++k, ++out) {
        if (out < p_cap) {
          tile_out[out] = (uint32_t)((ty0 + k) * tiles_x + tx0 + c);
          rank_out[out] = (uint32_t)r;
        }
      }
    }
    return;
  }
  // exact FP64 re-walk (span overflow, or the load-balanced min-q test)
  SplatF64 s = load_splat_f64(rec + (long long)row * 12);
  SnugRect box = snugbox(s, tiles_x, tiles_y);
  if (box.tx0 > box.tx1 || box.ty0 > box.ty1) return;
  for (long long tx = box.tx0; tx <= box.tx1; ++tx) {
    if (strategy == 1) {
      const double rx0 = dsub((double)(16 * tx), s.mx);
      for (long long ty = box.ty0; ty <= box.ty1; ++ty) {
        const double ry0 = dsub((double)(16 * ty), s.my);
        if (min_q_box(s, rx0, dadd(rx0, 16.0), ry0, dadd(ry0, 16.0)) <= s.t) {
          if (out < p_cap) {
            tile_out[out] = (uint32_t)(ty * tiles_x + tx);
            rank_out[out] = (uint32_t)r;
          }
          ++out;
        }
      }
    } else {
      long long ty0, ty1;
      const int nr = column_rows(s, box, tx, tiles_y, ty0, ty1);
      for (int k = 0; k < nr; ++k, ++out) {
        if (out < p_cap) {
          tile_out[out] = (uint32_t)((ty0 + k) * tiles_x + tx);
          rank_out[out] = (uint32_t)r;
        }
      }
    }
  }
}

// keys/values in the reference's layout + ranges: offsets[t] = first i with tile >= t.
__global__ void __launch_bounds__(kSB) finalize_index_kernel(
    const uint32_t* __restrict__ tiles_sorted, const uint32_t* __restrict__ ranks_sorted,
    const uint32_t* __restrict__ depth_bits_by_rank, const uint32_t* __restrict__ row_by_rank,
    const long long* __restrict__ totals, long long p_cap, int n_tiles,
    int64_t* __restrict__ keys, int32_t* __restrict__ values, int64_t* __restrict__ offsets) {
  const long long p = clamp_n(totals + 1, p_cap);
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i > p) return;
  long long cur = n_tiles;
  if (i < p) {
    const uint32_t t = tiles_sorted[i], r = ranks_sorted[i];
    keys[i] = ((long long)t << 32) | (long long)depth_bits_by_rank[r];
    values[i] = (int32_t)row_by_rank[r];
    cur = t;
  }
  const long long prev = i == 0 ? -1 : (long long)tiles_sorted[i - 1];
  for (long long t = prev + 1; t <= cur; ++t) offsets[t] = i;
}

// ckpt_base[t] = sum_{u<t} floor(n_u / 32); ckpt_base[T] = total records
// (forward.py:139-145: one record per completed 32-entry group).
__global__ void __launch_bounds__(1024) ckpt_base_kernel(const int64_t* __restrict__ offsets,
                                                         int n_tiles,
                                                         int64_t* __restrict__ ckpt_base) {
  __shared__ long long s_warp[32];
  __shared__ long long s_carry;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) s_carry = 0;
  __syncthreads();
  for (int base = 0; base < n_tiles; base += 1024) {
    const int t = base + threadIdx.x;
    const long long v = t < n_tiles ? (offsets[t + 1] - offsets[t]) / kGroup : 0;
    long long incl = v;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const long long y = __shfl_up_sync(0xffffffffu, incl, d);
      if (lane >= d) incl += y;
    }
    if (lane == 31) s_warp[warp] = incl;
    __syncthreads();
    if (warp == 0) {
      const long long w = s_warp[lane];
      long long wi = w;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const long long y = __shfl_up_sync(0xffffffffu, wi, d);
        if (lane >= d) wi += y;
      }
      s_warp[lane] = wi - w;
    }
    __syncthreads();
    const long long carry = s_carry;
    if (t < n_tiles) ckpt_base[t] = carry + s_warp[warp] + incl - v;
    __syncthreads();
    if (threadIdx.x == 1023) s_carry = carry + s_warp[warp] + incl;
    __syncthreads();
  }
  if (threadIdx.x == 0) ckpt_base[n_tiles] = s_carry;
}

// -------------------------------------------------------------- planning --
struct IndexWorkspace {
  uint32_t *dk0, *dv0, *dk1, *dv1;  // depth sort ping-pong (M_cap)
  uint32_t* off_rank;               // M_cap
  uint32_t *tk0, *tv0, *tk1, *tv1;  // tile sort ping-pong (P_cap)
  uint32_t *hist, *hist_scan;       // 256 x max_ctas
  unsigned long long* status;       // look-back status words
  unsigned int* tickets;            // 16 tickets
  size_t bytes;
  long long max_ctas, scan_blocks;
};

static size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

static IndexWorkspace plan(void* base, long long m_cap, long long p_cap) {
  IndexWorkspace w;
  const long long mc = m_cap > 0 ? m_cap : 1, pc = p_cap > 0 ? p_cap : 1;
  w.max_ctas = ((mc > pc ? mc : pc) + kSTile - 1) / kSTile;
  const long long hist_n = (long long)kBins * w.max_ctas;
  const long long scan_n = hist_n > mc ? hist_n : mc;
  w.scan_blocks = (scan_n + kScanTile - 1) / kScanTile;
  char* p = (char*)base;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    char* q = p ? p + off : nullptr;
    off += align256(bytes);
    return q;
  };
  w.dk0 = (uint32_t*)take(4 * mc);
  w.dv0 = (uint32_t*)take(4 * mc);
  w.dk1 = (uint32_t*)take(4 * mc);
  w.dv1 = (uint32_t*)take(4 * mc);
  w.off_rank = (uint32_t*)take(4 * mc);
  w.tk0 = (uint32_t*)take(4 * pc);
  w.tv0 = (uint32_t*)take(4 * pc);
  w.tk1 = (uint32_t*)take(4 * pc);
  w.tv1 = (uint32_t*)take(4 * pc);
  w.hist = (uint32_t*)take(4 * hist_n);
  w.hist_scan = (uint32_t*)take(4 * hist_n);
  // one status region per scan launch (6 radix passes + 1 rank scan)
  w.status = (unsigned long long*)take(8 * (size_t)w.scan_blocks * 8);
  w.tickets = (unsigned int*)take(16 * 4);
  w.bytes = off;
  return w;
}

static int scan_launch(const uint32_t* in, const int32_t* gather, uint32_t* out,
                       const long long* n_dev, long long n_cap, unsigned long long* status,
                       unsigned int* ticket, cudaStream_t s) {
  const long long blocks = (n_cap + kScanTile - 1) / kScanTile;
  if (blocks == 0) return TSR_OK;
  scan_u32_kernel<<<(int)blocks, kSB, 0, s>>>(in, gather, out, n_dev, n_cap, status, ticket);
  TSR_CHECK_LAUNCH();
  return TSR_OK;
}

// One stable radix pass over n (device) <= n_cap items.
static int radix_pass(const uint32_t* kin, const uint32_t* vin, uint32_t* kout, uint32_t* vout,
                      const long long* n_dev, long long n_cap, int shift, IndexWorkspace& w,
                      int slot, cudaStream_t s) {
  const int ctas = (int)((n_cap + kSTile - 1) / kSTile);
  if (ctas == 0) return TSR_OK;
  radix_hist_kernel<<<ctas, kSB, 0, s>>>(kin, n_dev, n_cap, shift, ctas, w.hist);
  TSR_CHECK_LAUNCH();
  int rc = scan_launch(w.hist, nullptr, w.hist_scan, nullptr, (long long)kBins * ctas,
                       w.status + (size_t)slot * w.scan_blocks, w.tickets + slot, s);
  if (rc != TSR_OK) return rc;
  radix_scatter_kernel<<<ctas, kSB, 0, s>>>(kin, vin, kout, vout, n_dev, n_cap, shift, ctas,
                                            w.hist_scan);
  TSR_CHECK_LAUNCH();
  return TSR_OK;
}

}  // namespace tsr

using namespace tsr;

extern "C" size_t tsr_index_workspace(int64_t m_cap, int64_t p_cap) {
  return plan(nullptr, m_cap, p_cap).bytes;
}

extern "C" int tsr_build_index(const float* rec, const uint32_t* depth_bits, const void* spans,
                               const int32_t* counts, const int64_t* totals, int64_t m_cap,
                               int64_t p_cap, int32_t width, int32_t height, int32_t strategy,
                               int64_t* keys, int32_t* values, int64_t* offsets,
                               int64_t* ckpt_base, int32_t* overflow, void* workspace,
                               size_t workspace_bytes, void* stream) {
  if (m_cap < 0 || p_cap < 0 || width <= 0 || height <= 0 || !totals || !offsets)
    return TSR_E_INVALID;
  if (workspace_bytes < tsr_index_workspace(m_cap, p_cap)) return TSR_E_WORKSPACE;
  cudaStream_t s = (cudaStream_t)stream;
  IndexWorkspace w = plan(workspace, m_cap, p_cap);
  const int tx = tiles_of(width), ty = tiles_of(height);
  const int n_tiles = tx * ty;
  const long long* M = (const long long*)totals;
  const long long* P = (const long long*)totals + 1;
  if (cudaMemsetAsync(w.status, 0, 8 * (size_t)w.scan_blocks * 8, s) != cudaSuccess ||
      cudaMemsetAsync(w.tickets, 0, 16 * 4, s) != cudaSuccess)
    return TSR_E_CUDA;
  int rc = TSR_OK;
  // 1. depth ranks: 4 stable 8-bit passes over (depth bits, row)
  if (m_cap > 0) {
    rc = radix_pass(depth_bits, nullptr, w.dk1, w.dv1, M, m_cap, 0, w, 0, s);
    if (!rc) rc = radix_pass(w.dk1, w.dv1, w.dk0, w.dv0, M, m_cap, 8, w, 1, s);
    if (!rc) rc = radix_pass(w.dk0, w.dv0, w.dk1, w.dv1, M, m_cap, 16, w, 2, s);
    if (!rc) rc = radix_pass(w.dk1, w.dv1, w.dk0, w.dv0, M, m_cap, 24, w, 3, s);
    if (rc) return rc;
    // 2. rank-order pair offsets and rank-major emission
    rc = scan_launch((const uint32_t*)counts, (const int32_t*)w.dv0, w.off_rank, M, m_cap,
                     w.status + 4 * (size_t)w.scan_blocks, w.tickets + 4, s);
    if (rc) return rc;
    emit_pairs_kernel<<<(int)((m_cap + kSB - 1) / kSB), kSB, 0, s>>>(
        rec, (const uint4*)spans, w.dv0, w.off_rank, (const long long*)totals, m_cap, p_cap, tx, ty, strategy, w.tk0,
        w.tv0, overflow);
    TSR_CHECK_LAUNCH();
  }
  // 3. stable sort of pairs by tile
  uint32_t *tk = w.tk0, *tv = w.tv0;
  if (p_cap > 0) {
    int slot = 5;
    for (int shift = 0; (n_tiles - 1) >> shift; shift += 8, ++slot) {
      if (slot > 7) return TSR_E_INVALID;
      uint32_t* ko = tk == w.tk0 ? w.tk1 : w.tk0;
      uint32_t* vo = tv == w.tv0 ? w.tv1 : w.tv0;
      rc = radix_pass(tk, tv, ko, vo, P, p_cap, shift, w, slot, s);
      if (rc) return rc;
      tk = ko;
      tv = vo;
    }
  }
  // 4. keys / values / ranges (+ checkpoint bases)
  finalize_index_kernel<<<(int)((p_cap + 1 + kSB - 1) / kSB), kSB, 0, s>>>(
      tk, tv, w.dk0, w.dv0, (const long long*)totals, p_cap, n_tiles, keys, values, offsets);
  TSR_CHECK_LAUNCH();
  if (ckpt_base) {
    ckpt_base_kernel<<<1, 1024, 0, s>>>(offsets, n_tiles, ckpt_base);
    TSR_CHECK_LAUNCH();
  }
  return rc;
}
