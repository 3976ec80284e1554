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
//      (tile | depth bits, row) pairs rank-major from K1's compact column
//      spans (no FP64 re-walk unless a splat's span did not fit the 16-byte
//      record);
//   3. stable LSD radix sort of the pairs by tile (8-bit digits, 2 passes
//      for up to 65536 tiles) -> within a tile, rank order; the last pass
//      writes the final int64 keys (tile << 32 | depth bits) and int32 rows;
//   4. per-tile ranges (boundaries of the sorted keys) + checkpoint bases.
// Every size (M, P) is read from device memory: the whole pipeline runs
// without a host synchronisation and can be captured in a CUDA graph.  The
// radix passes are the classic three-kernel form (CTA histograms -> one
// decoupled look-back scan -> stable scatter ranked with __match_any_sync).
#include <cuda_runtime.h>

#include "tsr_common.cuh"

namespace tsr {

constexpr int kSB = 256;                 // threads per CTA
constexpr int kSItemsMax = 16;           // items per thread (large passes)
constexpr int kSTileMax = kSB * kSItemsMax;
constexpr int kBins = 256;               // 8-bit digits
// M-sized passes (1M rows) use 4 items/thread so ~1000 CTAs keep every SM
// busy; P-sized passes use 8.
__host__ __device__ constexpr int items_for(long long n_cap) {
  return n_cap > (1ll << 22) ? 8 : 4;
}

__device__ __forceinline__ long long clamp_n(const long long* n_dev, long long n_cap) {
  const long long n = *n_dev;
  return n < n_cap ? (n > 0 ? n : 0) : n_cap;
}

// ------------------------------------------------------------ scan (u32) --
// Exclusive scan with a decoupled look-back; value(i) = in[gather ? gather[i] : i].
constexpr int kScanItems = 8;
constexpr int kScanTile = kSB * kScanItems;

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
    const uint32_t excl = (uint32_t)warp_lookback(status, bid, agg);
    if (lane == 0) s_prefix = excl;
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
template <int ITEMS>
__global__ void __launch_bounds__(kSB) radix_hist_kernel(const uint32_t* __restrict__ keys,
                                                         const long long* __restrict__ n_dev,
                                                         long long n_cap, int shift, int n_ctas,
                                                         uint32_t* __restrict__ hist) {
  __shared__ uint32_t s_h[kBins];
  s_h[threadIdx.x] = 0;
  const long long n = clamp_n(n_dev, n_cap);
  const long long base = (long long)blockIdx.x * (kSB * ITEMS);
  uint32_t kk[ITEMS];
#pragma unroll
  for (int k = 0; k < ITEMS; ++k) {  // all loads in flight first
    const long long i = base + (long long)k * kSB + threadIdx.x;
    kk[k] = i < n ? keys[i] : 0xffffffffu;
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < ITEMS; ++k) {
    const long long i = base + (long long)k * kSB + threadIdx.x;
    const bool valid = i < n;
    const uint32_t d = (kk[k] >> shift) & (kBins - 1);
    // skewed digits (e.g. the exponent byte of depths) collapse to one atomic
    const uint32_t d0 = __shfl_sync(0xffffffffu, d, 0);
    if (__all_sync(0xffffffffu, valid && d == d0)) {
      if ((threadIdx.x & 31) == 0) atomicAdd(&s_h[d], 32u);
    } else if (valid) {
      atomicAdd(&s_h[d], 1u);
    }
  }
  __syncthreads();
  hist[(long long)threadIdx.x * n_ctas + blockIdx.x] = s_h[threadIdx.x];
}

// Block-wide exclusive scan helper (256 threads): returns the exclusive
// prefix of v; *total receives the block sum.
template <typename T>
__device__ __forceinline__ T block_excl_scan_256(T v, T* s_w, T* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  T incl = v;
#pragma unroll
  for (int k = 1; k < 32; k <<= 1) {
    const T t = __shfl_up_sync(0xffffffffu, incl, k);
    if (lane >= k) incl += t;
  }
  if (lane == 31) s_w[warp] = incl;
  __syncthreads();
  T pre = 0, tot = 0;
#pragma unroll
  for (int w = 0; w < kSB / 32; ++w) {
    pre += w < warp ? s_w[w] : (T)0;
    tot += s_w[w];
  }
  *total = tot;
  return pre + incl - v;
}

// Per-digit exclusive scan over CTAs (one CTA per digit): hist_scan[d][c] =
// sum_{c' < c} hist[d][c'], digit_total[d] = sum_c hist[d][c].  Each thread
// scans a contiguous run of the row, then one block scan (no loop of
// barriers); the digit prefix is added by the scatter kernel.
constexpr int kRowPerThread = 64;  // rows up to 16384 CTAs (33.5M pairs at 8 items)
__global__ void __launch_bounds__(kSB) radix_digit_scan_kernel(const uint32_t* __restrict__ hist,
                                                               int n_ctas,
                                                               uint32_t* __restrict__ hist_scan,
                                                               uint32_t* __restrict__ digit_total) {
  __shared__ uint32_t s_w[kSB / 32];
  const int d = blockIdx.x;
  const uint32_t* row = hist + (long long)d * n_ctas;
  uint32_t* out = hist_scan + (long long)d * n_ctas;
  const int per = (n_ctas + kSB - 1) / kSB;  // <= kRowPerThread (checked by the host)
  const int c0 = threadIdx.x * per;
  const int c1 = min(c0 + per, n_ctas);
  uint32_t sum = 0;
  for (int c = c0; c < c1; ++c) sum += row[c];
  uint32_t total;
  uint32_t run = block_excl_scan_256(sum, s_w, &total);
  for (int c = c0; c < c1; ++c) {  // second read hits L1
    const uint32_t v = row[c];
    out[c] = run;
    run += v;
  }
  if (threadIdx.x == 0) digit_total[d] = total;
}

// Stable scatter.  Ranking: warp w owns items [base + 32 ITEMS w, ...),
// ranked round by round with __match_any_sync against per-warp digit
// counters; counters are prefixed over warps and digits so the CTA-local
// order is (digit, input position).  The CTA stages keys/values in shared
// memory in that order and writes each digit's run contiguously (coalesced).
// V = uint32_t (depth passes: row) or unsigned long long (tile passes:
// depth bits << 32 | row).  FINAL writes the TileIndex layout instead:
// keys64 = tile << 32 | depth bits, values32 = row.
template <int ITEMS, typename V, bool FINAL>
__global__ void __launch_bounds__(kSB) radix_scatter_kernel(
    const uint32_t* __restrict__ keys_in, const V* __restrict__ vals_in,
    uint32_t* __restrict__ keys_out, V* __restrict__ vals_out, int64_t* __restrict__ keys64,
    int32_t* __restrict__ values32, const long long* __restrict__ n_dev, long long n_cap,
    int shift, int n_ctas, const uint32_t* __restrict__ hist_scan,
    const uint32_t* __restrict__ digit_total) {
  constexpr int kTileN = kSB * ITEMS;
  __shared__ uint32_t s_cnt[kSB / 32][kBins];
  __shared__ uint32_t s_gbase[kBins];  // global start of this CTA's run of digit d
  __shared__ uint32_t s_lbase[kBins];  // CTA-local start of digit d
  __shared__ uint32_t s_wsum[kSB / 32];
  __shared__ uint32_t s_keys[kTileN];
  __shared__ V s_vals[kTileN];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
#pragma unroll
  for (int w = 0; w < kSB / 32; ++w) s_cnt[w][tid] = 0;
  const long long n = clamp_n(n_dev, n_cap);
  const long long cta_base = (long long)blockIdx.x * kTileN;
  if (cta_base >= n) return;  // uniform per CTA
  {
    // exclusive prefix of the digit totals (identical in every CTA)
    const uint32_t v = digit_total[tid];
    uint32_t incl = v;
#pragma unroll
    for (int k = 1; k < 32; k <<= 1) {
      const uint32_t t = __shfl_up_sync(0xffffffffu, incl, k);
      if (lane >= k) incl += t;
    }
    if (lane == 31) s_wsum[warp] = incl;
    __syncthreads();
    uint32_t wpre = 0;
#pragma unroll
    for (int w = 0; w < kSB / 32; ++w) wpre += w < warp ? s_wsum[w] : 0u;
    s_gbase[tid] = wpre + incl - v + hist_scan[(long long)tid * n_ctas + blockIdx.x];
  }
  __syncthreads();
  const long long wbase = cta_base + (long long)warp * (ITEMS * 32);
  const unsigned lt = (1u << lane) - 1u;
  uint32_t key[ITEMS], packed[ITEMS];
  V val[ITEMS];
#pragma unroll
  for (int r = 0; r < ITEMS; ++r) {  // all loads in flight first
    const long long i = wbase + r * 32 + lane;
    key[r] = i < n ? keys_in[i] : 0u;
    val[r] = i < n ? (vals_in ? vals_in[i] : (V)i) : (V)0;
  }
#pragma unroll
  for (int r = 0; r < ITEMS; ++r) {
    const long long i = wbase + r * 32 + lane;
    const bool valid = i < n;
    const uint32_t d = (key[r] >> shift) & (kBins - 1);
    const unsigned peers = __match_any_sync(0xffffffffu, valid ? d : (kBins + lane));
    const uint32_t before = __popc(peers & lt);
    uint32_t cnt = 0;
    if (valid) cnt = s_cnt[warp][d];
    __syncwarp();
    if (valid && before == 0) s_cnt[warp][d] = cnt + __popc(peers);
    __syncwarp();
    packed[r] = valid ? ((d << 16) | (cnt + before)) : 0xffffffffu;
  }
  __syncthreads();
  // digit tid: exclusive prefix over warps, then over digits
  uint32_t run = 0;
#pragma unroll
  for (int w = 0; w < kSB / 32; ++w) {
    const uint32_t c = s_cnt[w][tid];
    s_cnt[w][tid] = run;
    run += c;
  }
  uint32_t incl = run;
#pragma unroll
  for (int k = 1; k < 32; k <<= 1) {
    const uint32_t t = __shfl_up_sync(0xffffffffu, incl, k);
    if (lane >= k) incl += t;
  }
  __syncthreads();  // s_wsum reuse
  if (lane == 31) s_wsum[warp] = incl;
  __syncthreads();
  uint32_t wpre = 0;
#pragma unroll
  for (int w = 0; w < kSB / 32; ++w) wpre += w < warp ? s_wsum[w] : 0u;
  s_lbase[tid] = wpre + incl - run;
  __syncthreads();
#pragma unroll
  for (int r = 0; r < ITEMS; ++r) {
    if (packed[r] != 0xffffffffu) {
      const uint32_t d = packed[r] >> 16;
      const uint32_t local = s_lbase[d] + s_cnt[warp][d] + (packed[r] & 0xffffu);
      s_keys[local] = key[r];
      s_vals[local] = val[r];
    }
  }
  __syncthreads();
  const int cnt_valid = (int)(n - cta_base < kTileN ? n - cta_base : kTileN);
  for (int i = tid; i < cnt_valid; i += kSB) {
    const uint32_t k = s_keys[i];
    const uint32_t d = (k >> shift) & (kBins - 1);
    const uint32_t g = s_gbase[d] + (uint32_t)i - s_lbase[d];
    const V v = s_vals[i];
    if constexpr (FINAL) {
      keys64[g] = ((long long)k << 32) | (long long)(v >> 32);
      values32[g] = (int32_t)(uint32_t)v;
    } else {
      keys_out[g] = k;
      vals_out[g] = v;
    }
  }
}

// ------------------------------------------------------------- emission --
__device__ __forceinline__ void emit_one(long long out, long long p_cap, uint32_t tile,
                                         unsigned long long val, uint32_t* tile_out,
                                         unsigned long long* val_out) {
  if (out < p_cap) {
    tile_out[out] = tile;
    val_out[out] = val;
  }
}

// Rank-major emission.  Compact column-walk record written by K1 (see
// preprocess.cu):  x = tx0 | ncols << 16,  y = ty_base | overflow << 31,
// z, w = 8 columns x (row offset 4 bits | nrows 4 bits).
__global__ void __launch_bounds__(kSB) emit_pairs_kernel(
    const float* __restrict__ rec, const uint4* __restrict__ spans,
    const uint32_t* __restrict__ depth_by_rank, const uint32_t* __restrict__ row_by_rank,
    const uint32_t* __restrict__ off_rank, const long long* __restrict__ totals, long long m_cap,
    long long p_cap, int tiles_x, int tiles_y, int strategy, uint32_t* __restrict__ tile_out,
    unsigned long long* __restrict__ val_out, int* __restrict__ overflow) {
  const long long m = clamp_n(totals, m_cap);
  const long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= m) return;
  if (r == 0 && totals[1] > p_cap && overflow) *overflow = 1;  // sticky
  const uint32_t row = row_by_rank[r];
  const unsigned long long val = ((unsigned long long)depth_by_rank[r] << 32) | row;
  long long out = off_rank[r];
  const uint4 sp = spans[row];
  if (strategy == 0 && !(sp.y >> 31)) {
    const int tx0 = (int)(sp.x & 0xffffu), ncols = (int)(sp.x >> 16);
    const int ty_base = (int)(sp.y & 0xffffu);
    for (int c = 0; c < ncols; ++c) {
      const uint32_t code = ((c < 4 ? sp.z : sp.w) >> (8 * (c & 3))) & 0xffu;
      const int ty0 = ty_base + (int)(code & 15u), nr = (int)(code >> 4);
      for (int k = 0; k < nr; ++k, ++out)
        emit_one(out, p_cap, (uint32_t)((ty0 + k) * tiles_x + tx0 + c), val, tile_out, val_out);
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
        if (min_q_box(s, rx0, dadd(rx0, 16.0), ry0, dadd(ry0, 16.0)) <= s.t)
          emit_one(out++, p_cap, (uint32_t)(ty * tiles_x + tx), val, tile_out, val_out);
      }
    } else {
      long long ty0, ty1;
      const int nr = column_rows(s, box, tx, tiles_y, ty0, ty1);
      for (int k = 0; k < nr; ++k, ++out)
        emit_one(out, p_cap, (uint32_t)((ty0 + k) * tiles_x + tx), val, tile_out, val_out);
    }
  }
}

// offsets[t] = first sorted index whose tile >= t, t in [0, T] (binning.py:156-157).
__global__ void __launch_bounds__(kSB) tile_ranges_kernel(const int64_t* __restrict__ keys,
                                                          const long long* __restrict__ totals,
                                                          long long p_cap, int n_tiles,
                                                          int64_t* __restrict__ offsets) {
  const long long p = clamp_n(totals + 1, p_cap);
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i > p) return;
  const long long cur = i < p ? (keys[i] >> 32) : (long long)n_tiles;
  const long long prev = i == 0 ? -1 : (keys[i - 1] >> 32);
  for (long long t = prev + 1; t <= cur; ++t) offsets[t] = i;
}

// ckpt_base[t] = sum_{u<t} floor(n_u / 32) (forward.py:139-145: one record
// per completed 32-entry group); ckpt_base[T] = total records.  One CTA,
// each thread a contiguous run of tiles (up to 65536 tiles).
constexpr int kTilesPerThread = 64;
__global__ void __launch_bounds__(kSB) ckpt_base_kernel(const int64_t* __restrict__ offsets,
                                                        int n_tiles,
                                                        int64_t* __restrict__ ckpt_base) {
  __shared__ long long s_w[kSB / 32];
  const int per = (n_tiles + kSB - 1) / kSB;
  const int t0 = threadIdx.x * per;
  long long sum = 0;
  for (int k = 0; k < per; ++k) {
    const int t = t0 + k;
    if (t < n_tiles) sum += (offsets[t + 1] - offsets[t]) / kGroup;
  }
  long long total;
  long long run = block_excl_scan_256(sum, s_w, &total);
  for (int k = 0; k < per; ++k) {
    const int t = t0 + k;
    if (t < n_tiles) {
      ckpt_base[t] = run;
      run += (offsets[t + 1] - offsets[t]) / kGroup;
    }
  }
  if (threadIdx.x == 0) ckpt_base[n_tiles] = total;
}

// -------------------------------------------------------------- planning --
struct IndexWorkspace {
  uint32_t *dk0, *dv0, *dk1, *dv1;    // depth sort ping-pong (M_cap)
  uint32_t* off_rank;                 // M_cap
  uint32_t *tk0, *tk1;                // tile keys ping-pong (P_cap)
  unsigned long long *tv0, *tv1;      // depth bits << 32 | row (P_cap)
  uint32_t *hist, *hist_scan;         // 256 x max_ctas
  uint32_t* digit_total;              // 256
  unsigned long long* status;         // rank-scan look-back status words
  unsigned int* tickets;
  size_t bytes;
  long long max_ctas, scan_blocks;
};

constexpr int kMaxTiles = 1 << 16;

static size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

static IndexWorkspace plan(void* base, long long m_cap, long long p_cap) {
  IndexWorkspace w;
  const long long mc = m_cap > 0 ? m_cap : 1, pc = p_cap > 0 ? p_cap : 1;
  const long long ctas_m = (mc + kSB * items_for(mc) - 1) / (kSB * items_for(mc));
  const long long ctas_p = (pc + kSB * items_for(pc) - 1) / (kSB * items_for(pc));
  w.max_ctas = ctas_m > ctas_p ? ctas_m : ctas_p;
  const long long hist_n = (long long)kBins * w.max_ctas;
  w.scan_blocks = (mc + kScanTile - 1) / kScanTile;
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
  w.tk1 = (uint32_t*)take(4 * pc);
  w.tv0 = (unsigned long long*)take(8 * pc);
  w.tv1 = (unsigned long long*)take(8 * pc);
  w.hist = (uint32_t*)take(4 * hist_n);
  w.hist_scan = (uint32_t*)take(4 * hist_n);
  w.digit_total = (uint32_t*)take(4 * kBins);
  w.status = (unsigned long long*)take(8 * (size_t)w.scan_blocks);
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
template <int ITEMS, typename V, bool FINAL>
static int radix_pass_t(const uint32_t* kin, const V* vin, uint32_t* kout, V* vout,
                        int64_t* keys64, int32_t* values32, const long long* n_dev,
                        long long n_cap, int shift, IndexWorkspace& w, cudaStream_t s) {
  const int ctas = (int)((n_cap + kSB * ITEMS - 1) / (kSB * ITEMS));
  if (ctas == 0) return TSR_OK;
  if (ctas > kSB * kRowPerThread) return TSR_E_INVALID;  // > 8.4M pairs per pass
  radix_hist_kernel<ITEMS><<<ctas, kSB, 0, s>>>(kin, n_dev, n_cap, shift, ctas, w.hist);
  TSR_CHECK_LAUNCH();
  radix_digit_scan_kernel<<<kBins, kSB, 0, s>>>(w.hist, ctas, w.hist_scan, w.digit_total);
  TSR_CHECK_LAUNCH();
  radix_scatter_kernel<ITEMS, V, FINAL><<<ctas, kSB, 0, s>>>(
      kin, vin, kout, vout, keys64, values32, n_dev, n_cap, shift, ctas, w.hist_scan,
      w.digit_total);
  TSR_CHECK_LAUNCH();
  return TSR_OK;
}

template <typename V, bool FINAL>
static int radix_pass(const uint32_t* kin, const V* vin, uint32_t* kout, V* vout,
                      int64_t* keys64, int32_t* values32, const long long* n_dev,
                      long long n_cap, int shift, IndexWorkspace& w, cudaStream_t s) {
  return items_for(n_cap) == 8
             ? radix_pass_t<8, V, FINAL>(kin, vin, kout, vout, keys64, values32, n_dev, n_cap,
                                         shift, w, s)
             : radix_pass_t<4, V, FINAL>(kin, vin, kout, vout, keys64, values32, n_dev, n_cap,
                                         shift, w, s);
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
  if (n_tiles > kMaxTiles) return TSR_E_INVALID;
  const long long* M = (const long long*)totals;
  const long long* P = (const long long*)totals + 1;
  if (cudaMemsetAsync(w.status, 0, 8 * (size_t)w.scan_blocks, s) != cudaSuccess ||
      cudaMemsetAsync(w.tickets, 0, 16 * 4, s) != cudaSuccess)
    return TSR_E_CUDA;
  int rc = TSR_OK;
  uint32_t* no_k = nullptr;
  if (m_cap > 0) {
    // 1. depth ranks: 4 stable 8-bit passes over (depth bits, row)
    rc = radix_pass<uint32_t, false>(depth_bits, nullptr, w.dk1, w.dv1, nullptr, nullptr, M,
                                     m_cap, 0, w, s);
    if (!rc) rc = radix_pass<uint32_t, false>(w.dk1, w.dv1, w.dk0, w.dv0, nullptr, nullptr, M,
                                              m_cap, 8, w, s);
    if (!rc) rc = radix_pass<uint32_t, false>(w.dk0, w.dv0, w.dk1, w.dv1, nullptr, nullptr, M,
                                              m_cap, 16, w, s);
    if (!rc) rc = radix_pass<uint32_t, false>(w.dk1, w.dv1, w.dk0, w.dv0, nullptr, nullptr, M,
                                              m_cap, 24, w, s);
    if (rc) return rc;
    // 2. rank-order pair offsets and rank-major emission
    rc = scan_launch((const uint32_t*)counts, (const int32_t*)w.dv0, w.off_rank, M, m_cap,
                     w.status, w.tickets, s);
    if (rc) return rc;
    emit_pairs_kernel<<<(int)((m_cap + kSB - 1) / kSB), kSB, 0, s>>>(
        rec, (const uint4*)spans, w.dk0, w.dv0, w.off_rank, M, m_cap, p_cap, tx, ty, strategy,
        w.tk0, w.tv0, overflow);
    TSR_CHECK_LAUNCH();
  }
  // 3. stable sort of the pairs by tile; the last pass writes keys/values
  if (p_cap > 0) {
    int passes = 0;
    while ((n_tiles - 1) >> (8 * passes)) ++passes;
    if (passes == 0) passes = 1;
    uint32_t* tk = w.tk0;
    unsigned long long* tv = w.tv0;
    for (int q = 0; q < passes; ++q) {
      uint32_t* ko = tk == w.tk0 ? w.tk1 : w.tk0;
      unsigned long long* vo = tv == w.tv0 ? w.tv1 : w.tv0;
      if (q == passes - 1)
        rc = radix_pass<unsigned long long, true>(tk, tv, no_k, nullptr, keys, values, P, p_cap,
                                                  8 * q, w, s);
      else
        rc = radix_pass<unsigned long long, false>(tk, tv, ko, vo, nullptr, nullptr, P, p_cap,
                                                   8 * q, w, s);
      if (rc) return rc;
      tk = ko;
      tv = vo;
    }
  }
  // 4. per-tile ranges + checkpoint bases
  tile_ranges_kernel<<<(int)((p_cap + 1 + kSB - 1) / kSB), kSB, 0, s>>>(
      keys, (const long long*)totals, p_cap, n_tiles, offsets);
  TSR_CHECK_LAUNCH();
  if (ckpt_base) {
    ckpt_base_kernel<<<1, kSB, 0, s>>>(offsets, n_tiles, ckpt_base);
    TSR_CHECK_LAUNCH();
  }
  return rc;
}
