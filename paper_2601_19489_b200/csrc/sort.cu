// K2: depth-sorted per-tile index without a 64-bit key sort.
//
// The reference builds key = tile << 32 | bits(f32 depth) per (tile, splat)
// pair, emitted splat-major, and sorts it with a stable LSD radix sort
// (binning.py:137-158), so ties resolve by emission (= batch row) order.  The
// same order is produced here with far less traffic:
//   1. stable LSD radix sort of the M rows by their 32-bit depth bits (8-bit
//      digits; byte 0 always, bytes 1-3 unless the first pass's count phase
//      finds them the same for every row -- e.g. the exponent byte; 2,560-
//      item sub-tiles) -> depth rank of every row; rank order == (depth
//      bits, row) order, exactly the reference's tie rule;
//   2. rank-major emission of (tile, row) pairs -- 4-byte tile keys -- from
//      K1's compact column spans (written by both SnugBox strategies; rows
//      whose span did not fit the 16-byte record re-walk in FP64), staged
//      in shared memory so every CTA stores its contiguous output range
//      coalesced;
//   3. stable LSD radix sort of the pairs by the tile bits only (1-2 passes
//      of ~half the tile bits each, 2,048-item sub-tiles): within a tile,
//      rank order.  The last pass writes the final int64 keys tile << 32 |
//      depth bits of the row and the int32 rows;
//   4. per-tile ranges from the boundaries of the sorted keys; checkpoint
//      bases ckpt_base[t] = offsets[t] >> 5 (record r of tile t lives at
//      ckpt_base[t] + r: floor((O + n) / 32) - floor(O / 32) >= floor(n / 32),
//      so the tiles' record ranges never overlap and the total is <= P / 32).
//
// B200 shape: the whole index build is ONE persistent cooperative kernel (all
// CTAs co-resident, 3 per SM) whose phases are separated by grid barriers.
// At C2 sizes (1M rows, 4.4M pairs) every phase is latency-bound, so the
// multi-kernel form (3 launches per radix pass) or a decoupled look-back
// over ~1000 CTAs costs far more than the bytes.  A radix pass here is:
//   count   each CTA histograms its contiguous slice (warp-aggregated smem
//           atomics) -> cnt[cta][digit];                      grid barrier
//   scan    CTA d scans digit column d over the CTAs -> colscan; grid barrier
//   scatter each CTA re-reads its slice (L2-resident) in 2048-item sub-tiles,
//           ranks them stably with a ballot multi-split, stages them digit-sorted
//           in shared memory and stores each digit run coalesced at
//           digit_start + colscan + running offset;           grid barrier
// Every size (M, P) is read from device memory: nothing synchronises with
// the host, and the call is one memset + one launch.
#include <cuda_runtime.h>

#include "tsr_common.cuh"

namespace tsr {

#ifndef TSR_K2_RANGE_ITEMS
#define TSR_K2_RANGE_ITEMS 8  // boundary tests per thread in flight in the ranges phase
#endif
#ifndef TSR_K2_CTAS
#define TSR_K2_CTAS 3  // CTAs per SM (co-resident: cooperative launch)
#endif
constexpr int kSB = 256;                 // threads per CTA
constexpr int kBins = 256;               // 8-bit digits
#ifndef TSR_K2_PAIR_ITEMS
#define TSR_K2_PAIR_ITEMS 8
#endif
constexpr int kItems = TSR_K2_PAIR_ITEMS;  // items per thread per sub-tile (pair passes)
constexpr int kSub = kSB * kItems;       // 2048-item sub-tiles
#ifndef TSR_K2_DEPTH_ITEMS
#define TSR_K2_DEPTH_ITEMS 10
#endif
constexpr int kDepthItems = TSR_K2_DEPTH_ITEMS;  // the 4-byte depth passes: 2560-item sub-tiles (8/12/16 measured slower)
constexpr int kEmitPer = 2;              // ranks per thread per emission block
constexpr int kEmitRanks = kSB * kEmitPer;
constexpr int kStage = 4096;             // staged pairs per emission window
constexpr int kDynSmem = 49152;          // staging: 4096 x (u64 key, u32 row)
static_assert((kSB / 32) * sizeof(LbWarp) <= kDynSmem, "LB re-walk scratch in the staging area");
constexpr int kMaxGrid = 2048;
constexpr int kMaxBarriers = 32;
constexpr int kMaxTiles = 1 << 16;
constexpr uint32_t kNoPair = ~0u;

struct IndexArgs {
  const float* rec;
  const uint32_t* depth_bits;
  const uint4* spans;
  const int32_t* counts;
  const long long* totals;
  long long m_cap, p_cap;
  int tiles_x, tiles_y, n_tiles, strategy, tile_bits;
  int64_t* keys;
  int32_t* values;
  int64_t* offsets;
  int64_t* ckpt_base;
  int* overflow;
  uint32_t *dk0, *dv0, *dk1, *dv1;   // depth sort ping-pong (M_cap)
  uint32_t *pk0, *pk1;               // pair tile keys ping-pong (P_cap)
  uint32_t *pv0, *pv1;               // pair values (row) ping-pong (P_cap)
  uint32_t* cnt;                     // kMaxGrid x 256 per-CTA digit counts
  uint32_t* colscan;                 // kMaxGrid x 256 exclusive prefix over CTAs
  uint32_t* dtotal;                  // 256 digit totals of the current pass
  unsigned long long* ptot;          // kMaxGrid emitted pairs per CTA
  uint32_t* rank_cnt;                // M_cap pair count per rank
  uint4* rank_span;                  // M_cap column-span record per rank
  // deterministic-merge outputs (nullable; see tsr_build_index_det):
  uint32_t* inv_perm;                // P_cap: sorted position of each emission index
  uint32_t* out_rank_row;            // M_cap: batch row of each depth rank
  uint32_t* out_rank_count;          // M_cap: pairs of each rank
  uint32_t* out_rank_off;            // M_cap: emission offset of each rank
  // zeroed by the per-call memset:
  uint32_t* hist4;                   // [0] OR of the depth keys, [1] OR of their complements
  unsigned int* bar;                 // kMaxBarriers arrival counters
};

struct SortSmem {
  uint32_t cnt[kSB / 32][kBins];  // per-warp digit counters
  uint32_t run[kBins];            // running global offset of each digit
  uint32_t lbase[kBins];          // sub-tile-local start of each digit
  uint32_t h[4][kBins];           // histograms
  uint32_t w32[kSB / 32];
  unsigned long long w64[kSB / 32];
  int skip[4];
};

__device__ __forceinline__ long long clamp_ll(long long n, long long cap) {
  return n < cap ? (n > 0 ? n : 0) : cap;
}

// Grid barrier: all CTAs are co-resident (cooperative launch); counter b is
// used once per call (zeroed by the memset), so no sense reversal is needed.
#ifdef TSR_K2_TRACE
// instrumented build only (tools/k2_trace.py): CTA 0 stamps every barrier
__device__ unsigned long long tsr_k2_trace_buf[128];
__device__ unsigned long long tsr_k2_arrive_buf[2048 * 32];  // [cta][barrier] arrival stamps
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define TSR_TRACE_AT(i)                                                        \
  do {                                                                         \
    if (blockIdx.x == 0 && threadIdx.x == 0) tsr_k2_trace_buf[i] = gtimer(); \
  } while (0)
#define TSR_TRACE_SUB(call, i)                                                     \
  do {                                                                             \
    if (blockIdx.x == 0 && threadIdx.x == 0 && base == lo)                          \
      tsr_k2_trace_buf[64 + 6 * ((call) % 10) + (i)] = gtimer();                   \
  } while (0)
#else
#define TSR_TRACE_AT(i) \
  do {                 \
  } while (0)
#define TSR_TRACE_SUB(call, i) \
  do {                        \
  } while (0)
#endif

// Release-add on arrival (cumulative over the CTA's writes, ordered by the
// bar.sync before it), relaxed polling, and one acquire load once the count
// is complete -- no SC fence (MEMBAR.SC) on either side.
__device__ __forceinline__ void grid_barrier(unsigned int* ctr, unsigned int n_ctas) {
  __syncthreads();
  if (threadIdx.x == 0) {
#ifdef TSR_K2_TRACE
    tsr_k2_arrive_buf[blockIdx.x * 32 + (((uintptr_t)ctr & 127) >> 2)] = gtimer();
#endif
#ifdef TSR_K2_SC_BARRIER
    __threadfence();
    atomicAdd(ctr, 1u);
#else
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(ctr) : "memory");
#endif
    unsigned int v;
    // relaxed polling (an acquire load per poll would invalidate L1 under
    // the co-resident CTA)
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
    while (v < n_ctas) {
#ifndef TSR_K2_SPIN
      __nanosleep(20);
#endif
      asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
    }
#ifdef TSR_K2_SC_BARRIER
    __threadfence();
#else
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
#endif
#ifdef TSR_K2_TRACE
    if (blockIdx.x == 0) tsr_k2_trace_buf[1 + (((uintptr_t)ctr & 127) >> 2)] = gtimer();  // bar is 256-B aligned
#endif
  }
  __syncthreads();
}

// Block-wide exclusive scan (256 threads); *total receives the block sum.
template <typename T>
__device__ __forceinline__ T block_excl_scan(T v, T* s_w, T* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  T incl = v;
#pragma unroll
  for (int k = 1; k < 32; k <<= 1) {
    const T t = __shfl_up_sync(0xffffffffu, incl, k);
    if (lane >= k) incl += t;
  }
  __syncthreads();  // s_w may still be read by a previous call
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

// Lanes of the warp holding the same 8-bit digit (ballot multi-split: one
// ballot per digit bit).  __match_any_sync is emulated in software on this
// part (a BREV loop per distinct value) and shared-memory atomics cost
// ~2 cycles per lane, so ranking and counting use ballots plus one
// non-atomic update per distinct digit.  All 32 lanes must call.
__device__ __forceinline__ unsigned digit_peers(uint32_t d, int bits, unsigned valid_mask) {
  unsigned m = valid_mask;
#pragma unroll
  for (int b = 0; b < 8; ++b) {
    if (b >= bits) break;  // uniform
    const bool bit = (d >> b) & 1u;
    const unsigned bal = __ballot_sync(0xffffffffu, bit);
    m &= bit ? bal : ~bal;
  }
  return m;
}

// Warp-aggregated shared-memory histogram increment for counting (no order
// needed): a digit shared by the whole warp (skewed bytes) costs one atomic.
__device__ __forceinline__ void hist_add(uint32_t* h, uint32_t d, bool valid) {
  const uint32_t d0 = __shfl_sync(0xffffffffu, d, 0);
  if (__all_sync(0xffffffffu, valid && d == d0)) {
    if ((threadIdx.x & 31) == 0) atomicAdd(&h[d0], 32u);
  } else if (valid) {
    atomicAdd(&h[d], 1u);
  }
}

__device__ __forceinline__ void slice(long long n, int bid, int G, long long& lo, long long& hi) {
  lo = n * bid / G;
  hi = n * (bid + 1) / G;
}

template <typename K>
__device__ __forceinline__ uint32_t digit_of(K k, int shift, uint32_t mask) {
  return (uint32_t)(k >> shift) & mask;
}

// ---- radix pass, phase 1: per-CTA digit histogram of the slice
// or_bits (first depth pass only): OR of the keys and OR of their
// complements (= ~AND) into or_bits[0..1], one atomic pair per warp -- which
// depth bytes are the same for every row (those passes are skipped)
template <typename K, int kI>
__device__ void count_phase(const K* __restrict__ kin, long long lo, long long hi, int shift,
                            uint32_t mask, uint32_t* __restrict__ cnt_out, SortSmem& sm,
                            uint32_t* __restrict__ or_bits = nullptr) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  sm.h[0][tid] = 0;
  __syncthreads();
  uint32_t o = 0u, no = 0u;
  for (long long base = lo; base < hi; base += (kSB * kI)) {
    const long long wb = base + (long long)warp * (32 * kI);
    K k[kI];
#pragma unroll
    for (int r = 0; r < kI; ++r) {
      const long long i = wb + r * 32 + lane;
      k[r] = i < hi ? kin[i] : (K)0;
    }
#pragma unroll
    for (int r = 0; r < kI; ++r) {
      const bool valid = wb + r * 32 + lane < hi;
      hist_add(sm.h[0], digit_of(k[r], shift, mask), valid);
      if (or_bits && valid) {
        o |= (uint32_t)k[r];
        no |= ~(uint32_t)k[r];
      }
    }
  }
  if (or_bits) {
    for (int d = 16; d > 0; d >>= 1) {
      o |= __shfl_xor_sync(0xffffffffu, o, d);
      no |= __shfl_xor_sync(0xffffffffu, no, d);
    }
    if (lane == 0 && (o | no)) {
      atomicOr(&or_bits[0], o);
      atomicOr(&or_bits[1], no);
    }
  }
  __syncthreads();
  cnt_out[tid] = sm.h[0][tid];
}

// ---- radix pass, phase 2: CTA d scans digit column d over the G CTAs
__device__ void colscan_phase(const uint32_t* __restrict__ cnt, uint32_t* __restrict__ colscan,
                              uint32_t* __restrict__ dtotal, int G, SortSmem& sm) {
  const int per = (G + kSB - 1) / kSB;
  for (int d = blockIdx.x; d < kBins; d += gridDim.x) {
    const int c0 = threadIdx.x * per;
    uint32_t v[kMaxGrid / kSB];
    uint32_t sum = 0;
#pragma unroll
    for (int j = 0; j < kMaxGrid / kSB; ++j) {
      const int c = c0 + j;
      v[j] = (j < per && c < G) ? cnt[(long long)c * kBins + d] : 0u;
      sum += v[j];
    }
    uint32_t total;
    uint32_t run = block_excl_scan(sum, sm.w32, &total);
#pragma unroll
    for (int j = 0; j < kMaxGrid / kSB; ++j) {
      const int c = c0 + j;
      if (j < per && c < G) colscan[(long long)c * kBins + d] = run;
      run += v[j];
    }
    if (threadIdx.x == 0) dtotal[d] = total;
  }
}

// ---- radix pass, phase 3: stable scatter of the slice.
// K = u32 depth bits (values: rows; vin == nullptr -> value = index) or
// u64 pair keys tile << 32 | depth bits (values: rows).
template <typename K, int kI, typename KO = K>
__device__ void scatter_phase(const K* __restrict__ kin, const uint32_t* __restrict__ vin,
                              KO* __restrict__ kout, uint32_t* __restrict__ vout, long long lo,
                              long long hi, int shift, int bits,
                              const uint32_t* __restrict__ colscan_row,
                              const uint32_t* __restrict__ dtotal, SortSmem& sm,
                              unsigned char* dyn, const uint32_t* __restrict__ gather = nullptr,
                              uint32_t* __restrict__ inv = nullptr, int call = 0,
                              const uint32_t* __restrict__ depth_of_row = nullptr) {
  constexpr bool kVals = true;
  K* s_keys = reinterpret_cast<K*>(dyn);
  uint32_t* s_vals = reinterpret_cast<uint32_t*>(dyn + (kSB * kI) * sizeof(K));
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const unsigned lt = (1u << lane) - 1u;
  const uint32_t mask = (1u << bits) - 1u;
  {
    uint32_t total;
    const uint32_t dstart = block_excl_scan(dtotal[tid], sm.w32, &total);
    sm.run[tid] = dstart + colscan_row[tid];
  }
  // the sub-tile's items are loaded one sub-tile ahead: the next sub-tile's
  // loads are issued once this one's items are staged in shared memory, so
  // they overlap the staged read-back and the global stores
  K key[kI];
  uint32_t val[kI];
  auto load_items = [&](long long b) {
    const long long wb = b + (long long)warp * (32 * kI);
#pragma unroll
    for (int r = 0; r < kI; ++r) {  // all loads in flight first
      const long long i = wb + r * 32 + lane;
      key[r] = i < hi ? kin[i] : (K)0;
      if (kVals) val[r] = i < hi ? (vin ? vin[i] : (uint32_t)i) : 0u;
    }
  };
  if (lo < hi) load_items(lo);
  for (long long base = lo; base < hi; base += (kSB * kI)) {
#pragma unroll
    for (int w = 0; w < kSB / 32; ++w) sm.cnt[w][tid] = 0;
    __syncthreads();
    const long long wb = base + (long long)warp * (32 * kI);
    uint32_t packed[kI];
    TSR_TRACE_SUB(call, 0);
#pragma unroll
    for (int r = 0; r < kI; ++r) {
      const bool valid = wb + r * 32 + lane < hi;
      const uint32_t d = digit_of(key[r], shift, mask);
      const unsigned peers = digit_peers(d, bits, __ballot_sync(0xffffffffu, valid));
      const uint32_t before = __popc(peers & lt);
      uint32_t c = 0;
      if (valid) c = sm.cnt[warp][d];
      __syncwarp();
      if (valid && before == 0) sm.cnt[warp][d] = c + __popc(peers);
      __syncwarp();
      packed[r] = valid ? ((d << 16) | (c + before)) : 0xffffffffu;
    }
    TSR_TRACE_SUB(call, 1);
    __syncthreads();
    // digit tid: exclusive prefix over warps (input order), sub-tile total
    uint32_t tot = 0;
#pragma unroll
    for (int w = 0; w < kSB / 32; ++w) {
      const uint32_t c = sm.cnt[w][tid];
      sm.cnt[w][tid] = tot;
      tot += c;
    }
    uint32_t dummy;
    sm.lbase[tid] = block_excl_scan(tot, sm.w32, &dummy);
    __syncthreads();
    TSR_TRACE_SUB(call, 2);
#pragma unroll
    for (int r = 0; r < kI; ++r) {
      if (packed[r] != 0xffffffffu) {
        const uint32_t d = packed[r] >> 16;
        const uint32_t local = sm.lbase[d] + sm.cnt[warp][d] + (packed[r] & 0xffffu);
        s_keys[local] = key[r];
        if (kVals) s_vals[local] = val[r];
      }
    }
    __syncthreads();
    TSR_TRACE_SUB(call, 3);
    if (base + (kSB * kI) < hi) load_items(base + (kSB * kI));
    const int n_here = (int)(hi - base < (kSB * kI) ? hi - base : (kSB * kI));
    {
      // all kI items of the thread in flight at once (the det-mode
      // gathers are random loads)
      K k[kI];
      uint32_t v[kI], g[kI];
#pragma unroll
      for (int r = 0; r < kI; ++r) {
        const int i = tid + r * kSB;
        k[r] = i < n_here ? s_keys[i] : (K)0;
        v[r] = i < n_here ? s_vals[i] : 0u;
        const uint32_t d = digit_of(k[r], shift, mask);
        g[r] = sm.run[d] + (uint32_t)i - sm.lbase[d];
      }
      uint32_t gv[kI];
#pragma unroll
      for (int r = 0; r < kI; ++r)
        gv[r] = (gather && tid + r * kSB < n_here) ? gather[v[r]] : v[r];
      // the last tile pass writes the reference's keys: tile << 32 | depth
      // bits of the row (random 4-byte reads of an L2-resident array)
      KO ko[kI];
#pragma unroll
      for (int r = 0; r < kI; ++r) {
        if constexpr (sizeof(KO) > sizeof(K))
          ko[r] = tid + r * kSB < n_here
                      ? ((KO)k[r] << 32) | (KO)depth_of_row[gv[r]] : (KO)0;
        else
          ko[r] = k[r];
      }
#pragma unroll
      for (int r = 0; r < kI; ++r) {
        if (tid + r * kSB >= n_here) continue;
        kout[g[r]] = ko[r];
        vout[g[r]] = gv[r];
        if (gather) inv[v[r]] = g[r];  // values carry emission indices: inverse permutation
      }
    }
    __syncthreads();
    TSR_TRACE_SUB(call, 4);
    sm.run[tid] += tot;
  }
#ifdef TSR_K2_TRACE
  if (blockIdx.x == 0 && threadIdx.x == 0) tsr_k2_trace_buf[64 + 6 * (call % 10) + 5] = gtimer();
#endif
}

// ---- one full radix pass (3 phases, 3 grid barriers)
template <typename K, int kI = kItems, typename KO = K>
__device__ void radix_pass(const IndexArgs& a, int& nb, const K* kin, const uint32_t* vin,
                           KO* kout, uint32_t* vout, long long n, int shift, int bits,
                           SortSmem& sm, unsigned char* dyn,
                           const uint32_t* gather = nullptr, uint32_t* inv = nullptr,
                           const uint32_t* depth_of_row = nullptr,
                           uint32_t* or_bits = nullptr) {
  const int G = gridDim.x, bid = blockIdx.x;
  long long lo, hi;
  slice(n, bid, G, lo, hi);
  count_phase<K, kI>(kin, lo, hi, shift, (1u << bits) - 1u, a.cnt + (long long)bid * kBins, sm,
                     or_bits);
  grid_barrier(a.bar + nb++, G);
  colscan_phase(a.cnt, a.colscan, a.dtotal, G, sm);
  grid_barrier(a.bar + nb++, G);
  scatter_phase<K, kI, KO>(kin, vin, kout, vout, lo, hi, shift, bits,
                           a.colscan + (long long)bid * kBins, a.dtotal, sm, dyn, gather, inv,
                           nb / 3, depth_of_row);
  grid_barrier(a.bar + nb++, G);
}

// ---- emission.  Compact column-walk record written by K1 (preprocess.cu):
//   x = tx0 | ncols << 16,  y = ty_base | overflow << 31,
//   z, w = 8 columns x (row offset 4 bits | nrows 4 bits).
__device__ __forceinline__ uint32_t rank_row(const uint32_t* row_by_rank, long long r) {
  return row_by_rank ? row_by_rank[r] : (uint32_t)r;
}

// kLB: the instantiation for the load-balanced strategy (its warp-
// cooperative re-walk); the others never hold its registers
template <bool kLB>
__device__ void emit_phase(const IndexArgs& a, long long rlo, long long rhi, long long O,
                           long long p_cap,
                           const uint32_t* __restrict__ row_by_rank, SortSmem& sm,
                           unsigned char* dyn) {
  uint32_t* s_stage = reinterpret_cast<uint32_t*>(dyn);  // tile of each staged pair
  uint32_t* s_sval = reinterpret_cast<uint32_t*>(dyn + kStage * sizeof(uint32_t));
  const int tid = threadIdx.x;
  const int tiles_x = a.tiles_x, tiles_y = a.tiles_y, strategy = a.strategy;
  uint32_t* __restrict__ pairs = a.pk0;
  uint32_t* __restrict__ pair_rows = a.pv0;
  for (long long r0 = rlo; r0 < rhi; r0 += kEmitRanks) {
    uint32_t row[kEmitPer], cnt[kEmitPer], off[kEmitPer];
    uint4 sp[kEmitPer];
    uint32_t sum = 0;
#pragma unroll
    for (int k = 0; k < kEmitPer; ++k) {
      const long long r = r0 + kEmitPer * tid + k;
      cnt[k] = 0;
      sp[k] = make_uint4(0u, 0u, 0u, 0u);
      if (r < rhi) {
        cnt[k] = a.rank_cnt[r];
        sp[k] = a.rank_span[r];
      }
      row[k] = r < rhi ? rank_row(row_by_rank, r) : 0u;
      sum += cnt[k];
    }
    if (r0 == rlo) TSR_TRACE_AT(40);
    uint32_t total;
    uint32_t run = block_excl_scan(sum, sm.w32, &total);
    if (r0 == rlo) TSR_TRACE_AT(41);
#pragma unroll
    for (int k = 0; k < kEmitPer; ++k) {
      off[k] = run;
      run += cnt[k];
    }
    if (a.out_rank_row) {
#pragma unroll
      for (int k = 0; k < kEmitPer; ++k) {
        const long long r = r0 + kEmitPer * tid + k;
        if (r < rhi) {
          // clamp to the pair capacity: on overflow (P > p_cap) the pairs
          // past p_cap were never stored, and the reducer must not read
          // their inverse permutation (sticky overflow flag, grow, retry)
          const long long e0 = O + (long long)off[k];
          const long long room = a.p_cap - e0;
          a.out_rank_row[r] = rank_row(row_by_rank, r);
          a.out_rank_count[r] =
              room <= 0 ? 0u : (uint32_t)min((long long)cnt[k], room);
          a.out_rank_off[r] = (uint32_t)min(e0, a.p_cap);
        }
      }
    }
    for (uint32_t w0 = 0; w0 < total; w0 += kStage) {
      const uint32_t w1 = min(total, w0 + (uint32_t)kStage);
#pragma unroll
      for (int k = 0; k < kEmitPer; ++k) {
        const uint32_t lo = off[k], hi = off[k] + cnt[k];
        if (hi <= w0 || lo >= w1) continue;
        if (sp[k].y >> 31) {  // written by the FP64 re-walk below
          for (uint32_t p = max(lo, w0); p < min(hi, w1); ++p) s_stage[p - w0] = kNoPair;
          continue;
        }
        // one flat loop over the rank's pairs (column-major, K1's order);
        // (column, row-in-column) advance incrementally
        const uint32_t rowk = row[k];
        const uint32_t tx0 = sp[k].x & 0xffffu, ty_base = sp[k].y & 0xffffu;
        unsigned long long codes = ((unsigned long long)sp[k].w << 32) | sp[k].z;
        uint32_t c = 0, code = (uint32_t)codes & 0xffu;
        while ((code >> 4) == 0u && c < 7u) {
          codes >>= 8;
          code = (uint32_t)codes & 0xffu;
          ++c;
        }
        uint32_t t = (ty_base + (code & 15u)) * (uint32_t)tiles_x + tx0 + c, q = 0;
#pragma unroll 1
        for (uint32_t p = lo; p < hi; ++p) {
          if (p >= w0 && p < w1) {
            s_stage[p - w0] = t;
            s_sval[p - w0] = rowk;
          }
          t += (uint32_t)tiles_x;
          if (++q == (code >> 4) && p + 1 < hi) {  // next non-empty column
            q = 0;
            do {
              codes >>= 8;
              code = (uint32_t)codes & 0xffu;
              ++c;
            } while ((code >> 4) == 0u && c < 7u);
            t = (ty_base + (code & 15u)) * (uint32_t)tiles_x + tx0 + c;
          }
        }
      }
      __syncthreads();
      if (r0 == rlo && w0 == 0) TSR_TRACE_AT(45);
      for (uint32_t j = tid; j < w1 - w0; j += kSB) {
        const uint32_t v = s_stage[j];
        const long long g = O + w0 + j;
        if (v != kNoPair && g < p_cap) {
          pairs[g] = v;
          pair_rows[g] = s_sval[j];
        }
      }
      __syncthreads();
      if (r0 == rlo && w0 == 0) TSR_TRACE_AT(46);
    }
    if (r0 == rlo) TSR_TRACE_AT(42);
    // exact FP64 re-walk of the rows whose span record overflowed
    if (kLB) {
      // load-balanced strategy: the warp-cooperative round-robin min-q walk
      // (bin_load_balanced, binning.py:262-298), writing each splat's passing
      // tiles at its emission offset; the staging area is free here
      LbWarp* lbw = reinterpret_cast<LbWarp*>(dyn) + (threadIdx.x >> 5);
#pragma unroll
      for (int k = 0; k < kEmitPer; ++k) {
        const long long r = r0 + kEmitPer * tid + k;
        const bool v = r < rhi && (sp[k].y >> 31) && cnt[k] != 0;
        SplatF64 s{};
        if (v) s = load_splat_f64(a.rec + (long long)row[k] * 12);
        warp_emit_lb(s, v, tiles_x, tiles_y, row[k], O + off[k], p_cap, pairs,
                     pair_rows, *lbw);
      }
    }
#pragma unroll
    for (int k = 0; k < kEmitPer; ++k) {
      if (strategy == 1 || !(sp[k].y >> 31) || cnt[k] == 0) continue;
      long long out = O + off[k];
      SplatF64 s = load_splat_f64(a.rec + (long long)row[k] * 12);
      if (strategy == 2) {  // bin_aabb rectangle, column-major
        long long tx0, tx1, ty0, ty1;
        aabb_rect(s, tiles_x, tiles_y, tx0, tx1, ty0, ty1);
        for (long long tx = tx0; tx <= tx1; ++tx)
          for (long long ty = ty0; ty <= ty1; ++ty, ++out)
            if (out < p_cap) {
              pairs[out] = (uint32_t)(ty * tiles_x + tx);
              pair_rows[out] = row[k];
            }
        continue;
      }
      SnugRect box = snugbox(s, tiles_x, tiles_y);
      if (box.tx0 > box.tx1 || box.ty0 > box.ty1) continue;
      for (long long tx = box.tx0; tx <= box.tx1; ++tx) {
        if (strategy == 1) {
          const double rx0 = dsub((double)(16 * tx), s.mx);
          for (long long ty = box.ty0; ty <= box.ty1; ++ty) {
            const double ry0 = dsub((double)(16 * ty), s.my);
            if (min_q_box(s, rx0, dadd(rx0, 16.0), ry0, dadd(ry0, 16.0)) <= s.t) {
              if (out < p_cap) {
                pairs[out] = (uint32_t)(ty * tiles_x + tx);
                pair_rows[out] = row[k];
              }
              ++out;
            }
          }
        } else {
          long long ty0, ty1;
          const int nr = column_rows(s, box, tx, tiles_y, ty0, ty1);
          for (int q = 0; q < nr; ++q, ++out)
            if (out < p_cap) {
              pairs[out] = (uint32_t)((ty0 + q) * tiles_x + tx);
              pair_rows[out] = row[k];
            }
        }
      }
    }
    if (r0 == rlo) TSR_TRACE_AT(43);
    O += total;
  }
  TSR_TRACE_AT(44);
}

// ---- the persistent index kernel
template <bool kLB>
__global__ void __launch_bounds__(kSB, TSR_K2_CTAS) build_index_kernel(IndexArgs a) {
  __shared__ SortSmem sm;
  extern __shared__ __align__(16) unsigned char dyn[];
  const int G = gridDim.x, bid = blockIdx.x, tid = threadIdx.x;
  int nb = 0;
  const long long m = clamp_ll(a.totals[0], a.m_cap);
#ifdef TSR_K2_TRACE
  if (bid == 0 && tid == 0) tsr_k2_trace_buf[0] = gtimer();
#endif

  // ---- 1. depth ranks
  // byte 0 (the mantissa's low byte) is sorted unconditionally -- a
  // constant digit makes the stable pass the identity -- and its count phase
  // finds which of bytes 1-3 are the same for every row (no separate pass
  // over the keys, no extra barrier); those passes are skipped
  const uint32_t* dkey = a.depth_bits;
  const uint32_t* drow = nullptr;  // identity
  {
    uint32_t* ko[2] = {a.dk0, a.dk1};
    uint32_t* vo[2] = {a.dv0, a.dv1};
    radix_pass<uint32_t, kDepthItems>(a, nb, dkey, drow, ko[0], vo[0], m, 0, 8, sm, dyn, nullptr,
                                      nullptr, nullptr, a.hist4);
    dkey = ko[0];
    drow = vo[0];
    // byte q is constant iff no bit of it is 1 in some row and 0 in another
    const uint32_t var = a.hist4[0] & a.hist4[1];
    int par = 1;
    for (int q = 1; q < 4; ++q) {
      if (m == 0 || ((var >> (8 * q)) & 255u) == 0u) continue;  // CTA-uniform
      radix_pass<uint32_t, kDepthItems>(a, nb, dkey, drow, ko[par], vo[par], m, 8 * q, 8, sm, dyn);
      dkey = ko[par];
      drow = vo[par];
      par ^= 1;
    }
  }

  // ---- 2. rank-major emission
  long long rlo, rhi;
  slice(m, bid, G, rlo, rhi);
  {
    // gather each rank's span record once (its pair count follows from the
    // nibbles; K1's count only for re-walked rows) and store both in rank
    // order, so the emission reads them coalesced
    uint32_t sum = 0;
    for (long long r0 = rlo + tid; r0 < rhi; r0 += 4 * kSB) {
      uint32_t row[4];
      uint4 sp[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const long long r = r0 + j * kSB;
        row[j] = r < rhi ? rank_row(drow, r) : 0u;
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) sp[j] = r0 + j * kSB < rhi ? a.spans[row[j]] : make_uint4(0, 0, 0, 0);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const long long r = r0 + j * kSB;
        if (r >= rhi) continue;
        uint32_t c;
        if (sp[j].y >> 31) {
          c = (uint32_t)a.counts[row[j]];
        } else {
          // sum of the 8 nrows nibbles (high nibble of each byte)
          const uint32_t hz = (sp[j].z >> 4) & 0x0f0f0f0fu, hw = (sp[j].w >> 4) & 0x0f0f0f0fu;
          c = ((hz + hw) * 0x01010101u) >> 24;
        }
        a.rank_cnt[r] = c;
        a.rank_span[r] = sp[j];
        sum += c;
      }
    }
    unsigned long long total;
    block_excl_scan((unsigned long long)sum, sm.w64, &total);
    if (tid == 0) a.ptot[bid] = total;
  }
  grid_barrier(a.bar + nb++, G);
  long long O, P;
  {
    unsigned long long before = 0, all = 0;
    for (int c = tid; c < G; c += kSB) {
      const unsigned long long v = a.ptot[c];
      all += v;
      if (c < bid) before += v;
    }
    unsigned long long t0, t1;
    block_excl_scan(before, sm.w64, &t0);
    block_excl_scan(all, sm.w64, &t1);
    O = (long long)t0;
    P = (long long)t1;
  }
  if (bid == 0 && tid == 0 && P > a.p_cap && a.overflow) *a.overflow = 1;  // sticky
  emit_phase<kLB>(a, rlo, rhi, O, a.p_cap, drow, sm, dyn);
  grid_barrier(a.bar + nb++, G);

  // ---- 3. stable sort of the pairs by tile; the last pass writes keys/values
  const long long np = clamp_ll(P, a.p_cap);
  unsigned long long* keys_out = reinterpret_cast<unsigned long long*>(a.keys);
  uint32_t* vals_out = reinterpret_cast<uint32_t*>(a.values);
  // deterministic-merge mode: the passes carry emission indices (vin ==
  // nullptr: value = input index) and the last one gathers the rows and
  // writes the inverse permutation
  const bool det = a.inv_perm != nullptr;
  const uint32_t* v0 = det ? nullptr : a.pv0;
  const uint32_t* gat = det ? a.pv0 : nullptr;
  if (a.tile_bits > 8) {  // two passes of ~half the tile bits each
    const int b1 = (a.tile_bits + 1) / 2, b2 = a.tile_bits - b1;
    radix_pass<uint32_t>(a, nb, a.pk0, v0, a.pk1, a.pv1, np, 0, b1, sm, dyn);
    radix_pass<uint32_t, kItems, unsigned long long>(a, nb, a.pk1, a.pv1, keys_out, vals_out, np,
                                                     b1, b2, sm, dyn, gat, a.inv_perm,
                                                     a.depth_bits);
  } else {
    radix_pass<uint32_t, kItems, unsigned long long>(a, nb, a.pk0, v0, keys_out, vals_out, np, 0,
                                                     a.tile_bits, sm, dyn, gat, a.inv_perm,
                                                     a.depth_bits);
  }

  // ---- 4. per-tile ranges (binning.py:156-157) + checkpoint bases
  // 8 boundary tests per thread in flight per round (independent loads)
  const int* khi = reinterpret_cast<const int*>(a.keys) + 1;  // tile = high word
  constexpr int kR = TSR_K2_RANGE_ITEMS;
  for (long long i0 = (long long)bid * kSB * kR + tid; i0 <= np; i0 += (long long)G * kSB * kR) {
    int cur[kR], prev[kR];
#pragma unroll
    for (int r = 0; r < kR; ++r) {
      const long long i = i0 + (long long)r * kSB;
      cur[r] = i < np ? khi[2 * i] : a.n_tiles;
      prev[r] = (i == 0 || i > np) ? -1 : khi[2 * (i - 1)];
    }
#pragma unroll
    for (int r = 0; r < kR; ++r) {
      const long long i = i0 + (long long)r * kSB;
      if (i > np) continue;
      for (long long t = (long long)prev[r] + 1; t <= cur[r]; ++t) {
        a.offsets[t] = i;
        if (a.ckpt_base) a.ckpt_base[t] = i >> 5;
      }
    }
  }
  TSR_TRACE_AT(47);
}

// -------------------------------------------------------------- planning --
static size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

struct Plan {
  size_t bytes, ctl_off, ctl_bytes;
  size_t dk0, dv0, dk1, dv1, pk0, pk1, pv0, pv1, cnt, colscan, dtotal, ptot, rank_cnt, rank_span, hist4,
      bar;
};

static Plan plan(long long m_cap, long long p_cap) {
  Plan p;
  const long long mc = m_cap > 0 ? m_cap : 1, pc = p_cap > 0 ? p_cap : 1;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    const size_t q = off;
    off += align256(bytes);
    return q;
  };
  p.dk0 = take(4 * mc);
  p.dv0 = take(4 * mc);
  p.dk1 = take(4 * mc);
  p.dv1 = take(4 * mc);
  p.pk0 = take(4 * pc);
  p.pk1 = take(4 * pc);
  p.pv0 = take(4 * pc);
  p.pv1 = take(4 * pc);
  p.cnt = take(4 * (size_t)kMaxGrid * kBins);
  p.colscan = take(4 * (size_t)kMaxGrid * kBins);
  p.dtotal = take(4 * kBins);
  p.ptot = take(8 * (size_t)kMaxGrid);
  p.rank_cnt = take(4 * mc);
  p.rank_span = take(16 * mc);
  p.ctl_off = off;
  p.hist4 = take(4 * 4 * kBins);
  p.bar = take(4 * kMaxBarriers);
  p.ctl_bytes = off - p.ctl_off;
  p.bytes = off;
  return p;
}

}  // namespace tsr

using namespace tsr;

#ifdef TSR_K2_TRACE
extern "C" int tsr_k2_trace_read(unsigned long long* host, unsigned int* bar_base) {
  if (bar_base)  // the per-CTA arrival stamps [2048][32]
    return cudaMemcpyFromSymbol(host, tsr_k2_arrive_buf, sizeof(tsr_k2_arrive_buf)) == cudaSuccess ? 0 : 2;
  return cudaMemcpyFromSymbol(host, tsr_k2_trace_buf, sizeof(tsr_k2_trace_buf)) == cudaSuccess ? 0 : 2;
}
#endif

extern "C" size_t tsr_index_workspace(int64_t m_cap, int64_t p_cap) {
  return plan(m_cap, p_cap).bytes;
}

static int build_index_impl(const float* rec, const uint32_t* depth_bits, const void* spans,
                            const int32_t* counts, const int64_t* totals, int64_t m_cap,
                            int64_t p_cap, int32_t width, int32_t height, int32_t strategy,
                            int64_t* keys, int32_t* values, int64_t* offsets,
                            int64_t* ckpt_base, int32_t* overflow, void* workspace,
                            size_t workspace_bytes, uint32_t* inv_perm, uint32_t* rank_row_out,
                            uint32_t* rank_count_out, uint32_t* rank_off_out, void* stream) {
  if (m_cap < 0 || p_cap < 0 || width <= 0 || height <= 0 || !totals || !offsets)
    return TSR_E_INVALID;
  if (p_cap >= (1ll << 32) || m_cap >= (1ll << 32)) return TSR_E_INVALID;  // u32 offsets
  if (workspace_bytes < tsr_index_workspace(m_cap, p_cap) || !workspace) return TSR_E_WORKSPACE;
  cudaStream_t s = (cudaStream_t)stream;
  const Plan pl = plan(m_cap, p_cap);
  char* w = (char*)workspace;
  IndexArgs a;
  a.rec = rec;
  a.depth_bits = depth_bits;
  a.spans = (const uint4*)spans;
  a.counts = counts;
  a.totals = (const long long*)totals;
  a.m_cap = m_cap;
  a.p_cap = p_cap;
  a.tiles_x = tiles_of(width);
  a.tiles_y = tiles_of(height);
  a.n_tiles = a.tiles_x * a.tiles_y;
  if (a.n_tiles > kMaxTiles) return TSR_E_INVALID;
  a.strategy = strategy;
  a.tile_bits = 1;
  while ((1 << a.tile_bits) < a.n_tiles) ++a.tile_bits;  // <= 16
  a.keys = keys;
  a.values = values;
  a.offsets = offsets;
  a.ckpt_base = ckpt_base;
  a.overflow = overflow;
  a.dk0 = (uint32_t*)(w + pl.dk0);
  a.dv0 = (uint32_t*)(w + pl.dv0);
  a.dk1 = (uint32_t*)(w + pl.dk1);
  a.dv1 = (uint32_t*)(w + pl.dv1);
  a.pk0 = (uint32_t*)(w + pl.pk0);
  a.pk1 = (uint32_t*)(w + pl.pk1);
  a.pv0 = (uint32_t*)(w + pl.pv0);
  a.pv1 = (uint32_t*)(w + pl.pv1);
  a.cnt = (uint32_t*)(w + pl.cnt);
  a.colscan = (uint32_t*)(w + pl.colscan);
  a.dtotal = (uint32_t*)(w + pl.dtotal);
  a.ptot = (unsigned long long*)(w + pl.ptot);
  a.rank_cnt = (uint32_t*)(w + pl.rank_cnt);
  a.inv_perm = inv_perm;
  a.out_rank_row = rank_row_out;
  a.out_rank_count = rank_count_out;
  a.out_rank_off = rank_off_out;
  a.rank_span = (uint4*)(w + pl.rank_span);
  a.hist4 = (uint32_t*)(w + pl.hist4);
  a.bar = (unsigned int*)(w + pl.bar);

  auto* kern = a.strategy == 1 ? build_index_kernel<true> : build_index_kernel<false>;
  int dev = 0, sms = 0, per_sm = 0;
  if (cudaGetDevice(&dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess ||
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kDynSmem) !=
          cudaSuccess ||
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kSB, kDynSmem) != cudaSuccess)
    return TSR_E_CUDA;
  int grid = sms * (per_sm < TSR_K2_CTAS ? per_sm : TSR_K2_CTAS);
  // small problems: fewer CTAs (each grid barrier costs ~ one arrival per
  // CTA, and a slice of a few hundred items cannot use a whole CTA)
  const long long work = (p_cap > m_cap ? p_cap : m_cap) / 4096 + 8;
  if (work < grid) grid = (int)work;
  if (grid > kMaxGrid) grid = kMaxGrid;
  if (grid < 1) return TSR_E_CUDA;
  if (cudaMemsetAsync(w + pl.ctl_off, 0, pl.ctl_bytes, s) != cudaSuccess) return TSR_E_CUDA;
  void* args[] = {&a};
  if (cudaLaunchCooperativeKernel((const void*)kern, dim3(grid), dim3(kSB), args,
                                  kDynSmem, s) != cudaSuccess)
    return TSR_E_CUDA;
  return TSR_OK;
}

extern "C" int tsr_build_index(const float* rec, const uint32_t* depth_bits, const void* spans,
                               const int32_t* counts, const int64_t* totals, int64_t m_cap,
                               int64_t p_cap, int32_t width, int32_t height, int32_t strategy,
                               int64_t* keys, int32_t* values, int64_t* offsets,
                               int64_t* ckpt_base, int32_t* overflow, void* workspace,
                               size_t workspace_bytes, void* stream) {
  return build_index_impl(rec, depth_bits, spans, counts, totals, m_cap, p_cap, width, height,
                          strategy, keys, values, offsets, ckpt_base, overflow, workspace,
                          workspace_bytes, nullptr, nullptr, nullptr, nullptr, stream);
}

extern "C" int tsr_build_index_det(const float* rec, const uint32_t* depth_bits,
                                   const void* spans, const int32_t* counts,
                                   const int64_t* totals, int64_t m_cap, int64_t p_cap,
                                   int32_t width, int32_t height, int32_t strategy,
                                   int64_t* keys, int32_t* values, int64_t* offsets,
                                   int64_t* ckpt_base, int32_t* overflow, void* workspace,
                                   size_t workspace_bytes, uint32_t* inv_perm,
                                   uint32_t* rank_row, uint32_t* rank_count, uint32_t* rank_off,
                                   void* stream) {
  if (!inv_perm || !rank_row || !rank_count || !rank_off) return TSR_E_INVALID;
  return build_index_impl(rec, depth_bits, spans, counts, totals, m_cap, p_cap, width, height,
                          strategy, keys, values, offsets, ckpt_base, overflow, workspace,
                          workspace_bytes, inv_perm, rank_row, rank_count, rank_off, stream);
}
