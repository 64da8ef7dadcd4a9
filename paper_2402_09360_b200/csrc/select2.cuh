// select2.cuh — grid-wide exact top-k' candidate selection (sm_100a).
//
// Same contract as topk_select (linalg.hpp:157-176): the k' largest scores,
// ties by ascending index, returned as indices in ascending order. The key
// order (common.cuh make_key) makes that an exact order statistic on 64-bit
// unsigned keys, so the selection is: find T = the k'-th largest key, emit
// every key >= T in index order.
//
// Scores sit in L2 right after the proxy kernel, so the cost is latency and
// per-SM issue, not bytes. The pipeline keeps every pass short and spreads
// the wide ones over the whole GPU:
//   S1 sel_pivot_kernel  (1 CTA / query)  sample 2048 keys (a stride
//        permutation of 4-key blocks), pick two sample order statistics that
//        bracket rank k' with ~4 sigma margin -> pivots lo <= T <= hi.
//        n <= 8192: exact T from the whole row, and the same CTA
//        emits the candidates (one launch total).
//   S2 sel_window_kernel (C CTAs / query) count keys > hi, append keys in
//        [lo, hi] to a window buffer (warp-aggregated global atomics); the
//        last CTA of the query (ticket) takes the (k' - above)-th largest
//        key of the window -> T. A bracket miss or window overflow falls
//        back to an exact select over the full row in that CTA (correct,
//        slow, counted in `status`).
//   S3 sel_emit_kernel   (C CTAs / query) count keys >= T per chunk, chunk
//        offsets by decoupled look-back over chunk aggregates (dynamic chunk
//        ids make the wait order safe), ordered write.
// The in-CTA order statistic (block_range_select) bins the current key
// range [lo, hi] into 16 equal sub-ranges by shift, counts with packed
// 4-bit register counters (no shared-memory atomics) and __reduce_add_sync,
// and narrows to the bin holding rank r; <= 64 survivors finish in one warp.
// Each pass shrinks the key range >= 8x; a uniform window of W keys needs
// about log16(W / 64) passes.
//
// Counters (qc, agg) live in a context-owned zeroed buffer; the last CTA of
// each kernel and query restores them to zero, so a CUDA graph replays the
// pipeline without re-initialisation.
#pragma once
#include "common.cuh"
#include "fastsel.cuh"

namespace hire_dev {

constexpr int kSel2Threads = 512;
constexpr int kSel2Kpt = 16;                                  // keys per thread in registers
constexpr int kSel2Exact = kSel2Threads * kSel2Kpt;           // rows <= this: exact in S1
constexpr int kSel2SampleKpt = 4;
constexpr int kSel2Sample = kSel2Threads * kSel2SampleKpt;    // 2048 sampled keys
constexpr int kSel2WinRegs = kSel2Threads * kSel2Kpt;         // window handled in registers
constexpr int kSel2Qc = 8;                                    // u32 counters per query

constexpr int kRsCompact = 1024;  // survivors moved to registers after a pass

struct RangeScratch {
  unsigned cnt[2][32][16];    // per-pass-parity, per-warp bin counts (packed: words 0..7)
  unsigned red[2][32];
  uint64_t ckeys[kRsCompact]; // compacted survivors
  uint64_t small[32];
  uint64_t result;
  int small_n;
  int scan[40];
#ifdef HIRE_RS_STATS
  int passes;
  long long st[16];
#endif
};

// ---- key sources ------------------------------------------------------
// each(f) calls f(key, j) for every key this thread owns; j is the
// per-thread ordinal (a compile-time constant for register sources).
__device__ __forceinline__ void widen_bins(unsigned a, unsigned b, unsigned (&w)[8]);

template <int KPT>
struct RegKeys {
  static constexpr int kFixed = KPT;
  uint64_t k[KPT];
  template <class F>
  __device__ __forceinline__ void each(F f) const {
#pragma unroll
    for (int j = 0; j < KPT; ++j) f(k[j], j);
  }
  // 16-bin histogram of value words in [lo, lo + range], branch-free:
  // 16 x 4-bit counters per 64-bit accumulator, one accumulator per 15 keys.
  __device__ __forceinline__ void count_value_bins(unsigned lo, unsigned range, int sh,
                                                   unsigned (&w)[8]) const {
    constexpr int NA = (KPT + 14) / 15;
    uint64_t acc[NA];
#pragma unroll
    for (int a = 0; a < NA; ++a) acc[a] = 0;
#pragma unroll
    for (int j = 0; j < KPT; ++j) {
      const unsigned d = static_cast<unsigned>(k[j] >> 32) - lo;
      const unsigned sft = (d >> sh) << 2;
      acc[j % NA] += d <= range ? (1ull << sft) : 0ull;
    }
#pragma unroll
    for (int a = 0; a < NA; ++a) widen_bins(static_cast<unsigned>(acc[a]), static_cast<unsigned>(acc[a] >> 32), w);
  }
};

struct RowKeys {  // a full score row in global memory (fallback path)
  static constexpr int kFixed = 0;
  const float* s;
  uint32_t n;
  template <class F>
  __device__ __forceinline__ void each(F f) const {
    int j = 0;
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) f(make_key(__ldcg(s + i), i), j++);
  }
};

struct ArrayKeys {  // keys in global memory written by other CTAs of this kernel
  static constexpr int kFixed = 0;
  const uint64_t* k;
  uint32_t n;
  template <class F>
  __device__ __forceinline__ void each(F f) const {
    int j = 0;
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x)
      f(static_cast<uint64_t>(__ldcg(reinterpret_cast<const unsigned long long*>(k) + i)), j++);
  }
};

// Nibble counters (8 bins x 4 bits per word) -> 16-bit pairs, added into
// w[m] = bin 2m (low half) | bin 2m+1 (high half).
__device__ __forceinline__ void widen_bins(unsigned a, unsigned b, unsigned (&w)[8]) {
#pragma unroll
  for (int m = 0; m < 4; ++m) {
    w[m] += ((a >> (8 * m)) & 0xFu) | (((a >> (8 * m + 4)) & 0xFu) << 16);
    w[m + 4] += ((b >> (8 * m)) & 0xFu) | (((b >> (8 * m + 4)) & 0xFu) << 16);
  }
}

// Barrier over the first NT threads (named barrier 1): the block select may
// run on a subset of a larger CTA.
template <int NT>
__device__ __forceinline__ void rs_sync() {
  asm volatile("bar.sync 1, %0;" ::"n"(NT) : "memory");
}

struct RangeState {
  int phase;            // 0: value word; 1: index word among keys with value word vstar
  unsigned vstar, lo, hi;
  long long rr, cnt;    // rank within [lo, hi], keys in [lo, hi]
  int par;              // count-buffer parity
  long long above;      // keys above the current range
  int bracket;          // 0 exact; 1 lower bound, 2 upper bound of the rank-rr key
  long long stop;       // bracket: stop once the bound's side holds <= stop keys
};

// Projected word of key k for the current phase, and whether it takes part.
__device__ __forceinline__ bool rs_project(const RangeState& st, uint64_t k, unsigned* x) {
  const unsigned hi32 = static_cast<unsigned>(k >> 32);
  *x = st.phase == 0 ? hi32 : static_cast<unsigned>(k);
  return k != 0 && (st.phase == 0 || hi32 == st.vstar);
}

// Block min / max of the projected words -> st.lo, st.hi (block-uniform).
template <int NT, class Src>
__device__ __forceinline__ void rs_minmax(const Src& src, RangeState& st, RangeScratch* rs) {
  constexpr int NW = NT / 32;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  unsigned mn = 0xFFFFFFFFu, mx = 0u;
  src.each([&](uint64_t k, int) {
    unsigned x;
    const bool ok = rs_project(st, k, &x);
    mn = ok ? min(mn, x) : mn;
    mx = ok ? max(mx, x) : mx;
  });
  __syncwarp();
  mn = __reduce_min_sync(0xffffffffu, mn);
  mx = __reduce_max_sync(0xffffffffu, mx);
  if (lane == 0) {
    rs->red[0][wid] = mn;
    rs->red[1][wid] = mx;
  }
  rs_sync<NT>();
  mn = lane < NW ? rs->red[0][lane] : 0xFFFFFFFFu;
  mx = lane < NW ? rs->red[1][lane] : 0u;
  __syncwarp();
  st.lo = __reduce_min_sync(0xffffffffu, mn);
  st.hi = __reduce_max_sync(0xffffffffu, mx);
  rs_sync<NT>();  // red[] may be rewritten by the next minmax
}

// The pass loop: 16-way splits of [lo, hi] until <= 32 keys remain, then
// a direct rank. After the first pass that leaves <= kRsCompact keys, the
// survivors are compacted into registers (2 per thread) and the loop
// continues on those.
template <int NT, class Src>
__device__ uint64_t rs_loop(const Src& src, RangeState st, RangeScratch* rs) {
  constexpr int NW = NT / 32;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (;;) {
    if (st.lo == st.hi) {
      if (st.phase == 1) return (static_cast<uint64_t>(st.vstar) << 32) | st.lo;  // index words are unique
      if (st.cnt > 32) {  // > 32 keys share one value word: select on the index word
        st.phase = 1;
        st.vstar = st.lo;
        rs_minmax<NT>(src, st, rs);
        continue;
      }
    }
    if (st.cnt <= 32) break;
    const unsigned lo = st.lo, hi = st.hi, range = hi - lo;
    int sh = 32 - __clz(range) - 4;
    if (sh < 0) sh = 0;  // (range >> sh) <= 15
    const int pp = st.par;
    if constexpr (Src::kFixed > 0) {
      unsigned w[8];
#pragma unroll
      for (int m = 0; m < 8; ++m) w[m] = 0;
      if (st.phase == 0 && lo != 0) {
        // common case: value words; padding (word 0) wraps outside [lo, hi]
        src.count_value_bins(lo, range, sh, w);
      } else {
        unsigned a = 0, b = 0;
        src.each([&](uint64_t k, int j) {
          unsigned x;
          const bool ok = rs_project(st, k, &x);
          const unsigned dlt = x - lo;
          const unsigned bin = dlt >> sh;
          const unsigned inc = (ok && dlt <= range) ? (1u << ((bin & 7u) << 2)) : 0u;
          a += (bin & 8u) ? 0u : inc;
          b += (bin & 8u) ? inc : 0u;
          if (j % 15 == 14) {  // nibbles hold <= 15
            widen_bins(a, b, w);
            a = 0;
            b = 0;
          }
        });
        widen_bins(a, b, w);
      }
      __syncwarp();
      // transposed butterfly over the 8 packed words: lane L ends with
      // word (L & 7) = bins 2(L&7), 2(L&7)+1 summed over the warp
      unsigned a4[4], a2[2];
      {
        const bool h = lane & 4;
#pragma unroll
        for (int m = 0; m < 4; ++m)
          a4[m] = (h ? w[m + 4] : w[m]) + __shfl_xor_sync(0xffffffffu, h ? w[m] : w[m + 4], 4);
      }
      {
        const bool h = lane & 2;
#pragma unroll
        for (int m = 0; m < 2; ++m)
          a2[m] = (h ? a4[m + 2] : a4[m]) + __shfl_xor_sync(0xffffffffu, h ? a4[m] : a4[m + 2], 2);
      }
      const bool h1 = lane & 1;
      unsigned mine = (h1 ? a2[1] : a2[0]) + __shfl_xor_sync(0xffffffffu, h1 ? a2[0] : a2[1], 1);
      mine += __shfl_xor_sync(0xffffffffu, mine, 8);
      mine += __shfl_xor_sync(0xffffffffu, mine, 16);
      if (lane < 8) rs->cnt[pp][wid][lane] = mine;
    } else {
      // streaming sources (unbounded keys per thread): 32-bit counters
      unsigned u[16];
#pragma unroll
      for (int m = 0; m < 16; ++m) u[m] = 0;
      src.each([&](uint64_t k, int) {
        unsigned x;
        const bool ok = rs_project(st, k, &x);
        const unsigned dlt = x - lo;
        const unsigned bin = (ok && dlt <= range) ? (dlt >> sh) : 16u;
#pragma unroll
        for (int m = 0; m < 16; ++m) u[m] += bin == static_cast<unsigned>(m) ? 1u : 0u;
      });
      __syncwarp();
#pragma unroll
      for (int m = 0; m < 16; ++m) u[m] = __reduce_add_sync(0xffffffffu, u[m]);
      if (lane < 16) {
        unsigned mine = 0;
#pragma unroll
        for (int m = 0; m < 16; ++m) mine = lane == m ? u[m] : mine;
        rs->cnt[pp][wid][lane] = mine;
      }
    }
#ifdef HIRE_RS_STATS
    if (threadIdx.x == 0) { rs->passes++; rs->st[2 + min(rs->passes, 6)] = clock64(); }
#endif
    rs_sync<NT>();
    // every warp: lane j < 16 totals bin j over the warps, then the same decision
    auto bin_count = [&](int v, int j) -> unsigned {
      if constexpr (Src::kFixed > 0) {
        const unsigned wd = rs->cnt[pp][v][j >> 1];
        return (j & 1) ? (wd >> 16) : (wd & 0xFFFFu);
      } else {
        return rs->cnt[pp][v][j];
      }
    };
    unsigned tot = 0;
    if (lane < 16) {
#pragma unroll
      for (int v = 0; v < NW; ++v) tot += bin_count(v, lane);
    }
    st.par ^= 1;
    __syncwarp();
    unsigned cum = tot;  // cum_j = keys in bins >= j
#pragma unroll
    for (int o = 1; o < 16; o <<= 1) {
      const unsigned t = __shfl_down_sync(0xffffffffu, cum, o);
      if (lane + o < 16) cum += t;
    }
    const unsigned bal = __ballot_sync(0xffffffffu, lane < 16 && static_cast<long long>(cum) >= st.rr);
    const int bs = 31 - __clz(bal & 0xFFFFu);
    const unsigned cum_next = __shfl_sync(0xffffffffu, cum, bs + 1);
    const unsigned tb = __shfl_sync(0xffffffffu, tot, bs);
    const unsigned nlo = lo + (static_cast<unsigned>(bs) << sh);
    const unsigned span = (1u << sh) - 1u;  // sh <= 28
    st.hi = (hi - nlo > span) ? nlo + span : hi;
    st.lo = nlo;
    st.rr -= static_cast<long long>(cum_next);
    st.cnt = tb;
    st.above += static_cast<long long>(cum_next);
    if (st.bracket == 1 && st.above + st.cnt <= st.stop) {
      // every key >= this bound ranks within the first above + cnt
      return st.phase == 0 ? (static_cast<uint64_t>(st.lo) << 32) : ((static_cast<uint64_t>(st.vstar) << 32) | st.lo);
    }
    if (st.bracket == 2 && st.cnt <= st.stop) {
      // exactly `above` keys lie above this bound
      return st.phase == 0 ? ((static_cast<uint64_t>(st.hi) << 32) | 0xFFFFFFFFull)
                           : ((static_cast<uint64_t>(st.vstar) << 32) | st.hi);
    }
    // survivors per thread after compaction: a quarter of the keys per
    // thread, bounded by the shared staging buffer
    constexpr int CK0 = Src::kFixed / 4 > 2 ? Src::kFixed / 4 : 2;
    constexpr int CK = CK0 < kRsCompact / NT ? CK0 : kRsCompact / NT;
    if constexpr (Src::kFixed > CK && CK >= 2) {
      if (st.cnt > 32 && st.cnt <= CK * NT && st.lo != st.hi) {
        // compact the survivors (this warp's slice starts after the
        // lower warps' counts of bin bs), continue on 2 keys per thread
        unsigned wc = lane < NW ? bin_count(lane, bs) : 0u;
        unsigned incl = wc;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const unsigned t = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += t;
        }
        unsigned pos = __shfl_sync(0xffffffffu, incl - wc, wid);
        const unsigned clo = st.lo, chi = st.hi;
        src.each([&](uint64_t k, int) {
          unsigned x;
          const bool in = rs_project(st, k, &x) && x - clo <= chi - clo;
          const unsigned bl = __ballot_sync(0xffffffffu, in);
          if (in) rs->ckeys[pos + __popc(bl & ((1u << lane) - 1u))] = k;
          pos += __popc(bl);
        });
        rs_sync<NT>();
        RegKeys<CK> c;
        const int t = threadIdx.x;
#pragma unroll
        for (int j = 0; j < CK; ++j) c.k[j] = t + j * NT < st.cnt ? rs->ckeys[t + j * NT] : 0ull;
        return rs_loop<NT>(c, st, rs);
      }
    }
  }
  // <= 32 keys left in the range: gather, rank each against the others
#ifdef HIRE_RS_STATS
  if (threadIdx.x == 0) rs->st[10] = clock64();
#endif
  const unsigned lo = st.lo, hi = st.hi;
  src.each([&](uint64_t k, int) {
    unsigned x;
    const bool in = rs_project(st, k, &x) && x - lo <= hi - lo;
    if (in) {
      const int p = atomicAdd(&rs->small_n, 1);
      if (p < 32) rs->small[p] = k;
    }
  });
  rs_sync<NT>();
#ifdef HIRE_RS_STATS
  if (threadIdx.x == 0) rs->st[11] = clock64();
#endif
  if (threadIdx.x < 32) {
    const int m = min(rs->small_n, 32);
    if (threadIdx.x < m) {
      const uint64_t mine = rs->small[threadIdx.x];
      int g = 0;
      for (int j = 0; j < m; ++j) g += rs->small[j] > mine ? 1 : 0;
      if (g == st.rr - 1) rs->result = mine;
    }
  }
  rs_sync<NT>();
#ifdef HIRE_RS_STATS
  if (threadIdx.x == 0) rs->st[12] = clock64();
#endif
  return rs->result;
}

// r-th largest (1-based) key among the non-zero keys of `src` (n_in of
// them over the block, 1 <= r <= n_in). Block-uniform result.
//
// Phase A narrows a range of the value word (key >> 32) by 16-way splits;
// if more than 32 keys share the final value word (ties), phase B does the
// same on the index word of those keys; <= 32 survivors are ranked
// directly. Counting is 32/64-bit register arithmetic (no shared atomics);
// each pass costs one barrier: every warp reads all warps' bin counts and
// takes the same decision, and the count buffers alternate by pass parity.
template <int NT, class Src>
__device__ uint64_t block_range_select(const Src& src, long long n_in, long long r, RangeScratch* rs,
                                       int bracket = 0, long long stop = 0) {
  RangeState st;
  st.phase = 0;
  st.vstar = 0;
  st.rr = r;
  st.cnt = n_in;
  st.par = 0;
  st.above = 0;
  st.bracket = bracket;
  st.stop = stop;
  if (threadIdx.x == 0) rs->small_n = 0;
  rs_minmax<NT>(src, st, rs);
#ifdef HIRE_RS_STATS
  if (threadIdx.x == 0) rs->st[0] = clock64();
#endif
  return rs_loop<NT>(src, st, rs);
}

// Block exclusive scan (NT <= 1024) of one int per thread.
template <int NT>
__device__ __forceinline__ int block_scan_excl(int v, int* s_tmp, int* total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int n = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += n;
  }
  if (lane == 31) s_tmp[w] = inc;
  __syncthreads();
  if (w == 0) {
    int t = lane < NT / 32 ? s_tmp[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int n = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= o) t += n;
    }
    if (lane < NT / 32) s_tmp[lane] = t;
    if (lane == NT / 32 - 1) s_tmp[NT / 32] = t;
  }
  __syncthreads();
  const int before = w > 0 ? s_tmp[w - 1] : 0;
  *total = s_tmp[NT / 32];
  __syncthreads();
  return before + inc - v;
}

__device__ __forceinline__ void st_release_u32(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// ---------------------------------------------------------------------
// S1 (small rows, n <= kSel2Exact). One CTA per query: exact T over the
// whole row and the ordered emit -> cand.
// ---------------------------------------------------------------------
template <int NT, int KPT>
__global__ void __launch_bounds__(NT) sel_exact_kernel(
    const float* __restrict__ scores, int64_t stride, uint32_t n, uint32_t K,
    uint32_t* __restrict__ cand, int64_t cand_stride) {
  __shared__ RangeScratch rs;
  hire_dev::griddep_wait();
  hire_dev::griddep_launch();
  KTrace kt_(kKtPivot);
  const int b = blockIdx.x;
  const float* row = scores + b * stride;
  // blocked layout: thread t owns indices [t*KPT, t*KPT+KPT) -> ordered emit
  RegKeys<KPT> src;
  const uint32_t i0 = threadIdx.x * KPT;
  if ((reinterpret_cast<uintptr_t>(row) & 15) == 0 && i0 + KPT <= n) {
#pragma unroll
    for (int j = 0; j < KPT; j += 4) {
      const float4 v = *reinterpret_cast<const float4*>(row + i0 + j);
      src.k[j] = make_key(v.x, i0 + j);
      src.k[j + 1] = make_key(v.y, i0 + j + 1);
      src.k[j + 2] = make_key(v.z, i0 + j + 2);
      src.k[j + 3] = make_key(v.w, i0 + j + 3);
    }
  } else {
#pragma unroll
    for (int j = 0; j < KPT; ++j) {
      const uint32_t i = i0 + j;
      src.k[j] = i < n ? make_key(row[i], i) : 0ull;
    }
  }
  const uint64_t T = block_range_select<NT>(src, n, K, &rs);
  int c = 0;
#pragma unroll
  for (int j = 0; j < KPT; ++j) c += src.k[j] >= T ? 1 : 0;
  int total;
  int pos = block_scan_excl<NT>(c, rs.scan, &total);
  uint32_t* out = cand + b * cand_stride;
#pragma unroll
  for (int j = 0; j < KPT; ++j)
    if (src.k[j] >= T) out[pos++] = i0 + j;
}

#if HIRE_EXPERIMENTS
// ---------------------------------------------------------------------
// Mid-size rows (kSel2Exact < n <= kSmemRowMax): one 1024-thread CTA per
// query holds the whole score row in shared memory; T = the K-th largest
// key by block_fast_select over the shared-memory row; ordered emit with
// warp-owned contiguous slices (count pass -> warp prefix -> write pass).
// One launch instead of the grid-wide pivot / window / window-select / emit.
// ---------------------------------------------------------------------
constexpr int kSmemRowMax = 49152;  // 192 KB of fp32 scores

__global__ void __launch_bounds__(1024, 1) sel_smem_kernel(
    const float* __restrict__ scores, int64_t stride, uint32_t n, uint32_t K,
    uint32_t* __restrict__ cand, int64_t cand_stride) {
  constexpr int NT = 1024, NW = NT / 32;
  __shared__ FastSelScratch fss;
  __shared__ unsigned s_wc[NW];
  extern __shared__ __align__(16) unsigned char row_smem[];
  float* sr = reinterpret_cast<float*>(row_smem);
  hire_dev::griddep_wait();
  hire_dev::griddep_launch();
  KTrace kt_(kKtPivot);
  const int b = blockIdx.x;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const float* row = scores + b * stride;
  if ((reinterpret_cast<uintptr_t>(row) & 15) == 0 && (n & 3) == 0) {
    block_copy_tf<8, float4>(reinterpret_cast<float4*>(sr), static_cast<int>(n / 4),
                             [&](int i) { return __ldcg(reinterpret_cast<const float4*>(row) + i); });
  } else {
    block_copy_tf<8, float>(sr, static_cast<int>(n), [&](int i) { return __ldcg(row + i); });
  }
  __syncthreads();
  const uint64_t dummy[1] = {0ull};
  const uint64_t T = block_fast_select<NT, 1>(dummy, K, &fss, nullptr, sr, n);
  // warp w owns [w*span, (w+1)*span), 32 elements per step (lane = element)
  const uint32_t span = ((n + NW - 1) / NW + 31) / 32 * 32;
  const uint32_t w0 = wid * span, w1 = min(n, w0 + span);
  unsigned c = 0;
  for (uint32_t i0 = w0; i0 < w1; i0 += 32) {
    const uint32_t i = i0 + lane;
    c += __popc(__ballot_sync(0xffffffffu, i < w1 && make_key(sr[i], i) >= T));
  }
  if (lane == 0) s_wc[wid] = c;
  __syncthreads();
  unsigned pos = 0;
  for (int v = 0; v < wid; ++v) pos += s_wc[v];
  uint32_t* out = cand + b * cand_stride;
  for (uint32_t i0 = w0; i0 < w1; i0 += 32) {
    const uint32_t i = i0 + lane;
    const bool in = i < w1 && make_key(sr[i], i) >= T;
    const unsigned bal = __ballot_sync(0xffffffffu, in);
    if (in) out[pos + __popc(bal & ((1u << lane) - 1u))] = i;
    pos += __popc(bal);
  }
}

#endif  // HIRE_EXPERIMENTS

// ---------------------------------------------------------------------
// S1 (large rows). One 128-thread CTA per query: 2048 sampled keys (512
// blocks of 4 consecutive rows, block ids s * perm mod nblk), pivots from
// two sample order statistics -> piv[b] = {lo, hi}.
// ---------------------------------------------------------------------
constexpr int kPivThreads = 128;

constexpr int kWinBins = 256;  // window histogram bins (value-word sub-ranges of [lo, top])
constexpr int kWinGroups = 8;  // chunk groups with their own histogram (bounds same-address atomics)
constexpr int kBinCap = 32;    // keys kept per (group, bin) list

template <int NT>
__global__ void __launch_bounds__(NT) sel_pivot_kernel(
    const float* __restrict__ scores, int64_t stride, uint32_t n, uint32_t K, uint32_t perm,
    uint64_t* __restrict__ piv, unsigned* __restrict__ gh, int exact_lo) {
  constexpr int KPT = kSel2Sample / NT;
  static_assert(KPT % 4 == 0, "the sample is loaded in 4-key blocks per thread (NT <= 512)");
  __shared__ RangeScratch rs;
  __shared__ unsigned s_top;
  hire_dev::griddep_wait();
  hire_dev::griddep_launch();
  KTrace kt_(kKtPivot);
  const int b = blockIdx.x;
  const float* row = scores + b * stride;
  for (int t = threadIdx.x; t < kWinBins * kWinGroups; t += NT) gh[b * kWinBins * kWinGroups + t] = 0u;
  RegKeys<KPT> src;
  const uint32_t nblk = n >> 2;
#pragma unroll
  for (int q = 0; q < KPT / 4; ++q) {
    const uint32_t sidx = threadIdx.x + q * NT;
    const uint32_t i = static_cast<uint32_t>((static_cast<uint64_t>(sidx) * perm) % nblk) * 4;
#pragma unroll
    for (int e = 0; e < 4; ++e) src.k[4 * q + e] = make_key(row[i + e], i + e);
  }
  {  // sample maximum value word: the top of the bin range when hi is open
    unsigned mx = 0;
#pragma unroll
    for (int j = 0; j < KPT; ++j) mx = max(mx, static_cast<unsigned>(src.k[j] >> 32));
    mx = __reduce_max_sync(0xffffffffu, mx);
    if (threadIdx.x == 0) s_top = 0;
    __syncthreads();
    if ((threadIdx.x & 31) == 0) atomicMax(&s_top, mx);
  }
  const double S = kSel2Sample;
  const double p = static_cast<double>(K) / static_cast<double>(n);
  const double mu = p * S, sd = sqrt(S * p * (1.0 - p));
  const long long r_hi = static_cast<long long>(floor(mu - 4.0 * sd - 1.0));
  const long long r_lo = static_cast<long long>(ceil(mu + 4.0 * sd + 1.0));
  // bounds, not exact order statistics: lo <= key(r_lo) with at most
  // 2 r_lo + 16 sample keys above it; hi >= key(r_hi) with fewer than r_hi above
  // exact_lo (the list path, sel_wlist_kernel): only lo, as the exact
  // sample order statistic, so the listed keys stay near r_lo/S * n
  const uint64_t hi = (r_hi >= 1 && !exact_lo) ? block_range_select<NT>(src, kSel2Sample, r_hi, &rs, 2, 16) : ~0ull;
  const uint64_t lo = r_lo <= kSel2Sample
                          ? (exact_lo ? block_range_select<NT>(src, kSel2Sample, r_lo, &rs)
                                      : block_range_select<NT>(src, kSel2Sample, r_lo, &rs, 1, 2 * r_lo + 16))
                          : 1ull;
  if (threadIdx.x == 0) {
    const unsigned vlo = static_cast<unsigned>(lo >> 32);
    const unsigned vtop = max(vlo, r_hi >= 1 ? static_cast<unsigned>(hi >> 32) : s_top);
    const int bits = 32 - __clz(vtop - vlo);  // range < 2^bits
    const int sh = bits > 8 ? bits - 8 : 0;
    piv[4 * b] = lo;
    piv[4 * b + 1] = hi;
    piv[4 * b + 2] = static_cast<uint64_t>(vlo) | (static_cast<uint64_t>(sh) << 32);
  }
}

__device__ __forceinline__ unsigned win_bin(uint64_t k, unsigned vlo, int sh) {
  return min(static_cast<unsigned>(kWinBins - 1), (static_cast<unsigned>(k >> 32) - vlo) >> sh);
}

// ---------------------------------------------------------------------
// S2. grid (C, B), 256 threads. Chunk c of query b: count keys > hi and
// collect the keys in [lo, hi] into its own window segment
// win[b][c*seg ...]; per-chunk counts go to cnt[b][0][c] (above) and
// cnt[b][1][c] (window, may exceed seg = overflow). Loads are issued 8 per
// thread before use. No global atomics: same-address atomics from many
// CTAs serialise at L2 (~27 cycles each). Also clears the chunk's emit
// aggregate agg[b][c] for S3.
// ---------------------------------------------------------------------
constexpr int kWinThreads = 256;
#ifndef HIRE_SCAN_BATCH
#define HIRE_SCAN_BATCH 8
#endif
constexpr int kScanBatch = HIRE_SCAN_BATCH;  // score loads in flight per thread (S2 / S3)

__global__ void __launch_bounds__(kWinThreads) sel_window_kernel(
    const float* __restrict__ scores, int64_t stride, uint32_t n, const uint64_t* __restrict__ piv,
    uint64_t* __restrict__ win, uint32_t seg, unsigned* __restrict__ cnt, unsigned* __restrict__ agg,
    unsigned* __restrict__ gh, uint64_t* __restrict__ lists) {
  constexpr int NT = kWinThreads, U = kScanBatch, STAGE = 1024;
  __shared__ unsigned s_above, s_wn;
  __shared__ uint64_t s_win[STAGE];
  hire_dev::griddep_wait();
  hire_dev::LateTrigger late_trigger_;
  KTrace kt_(kKtWindow);
  const int b = blockIdx.y, C = gridDim.x, c = blockIdx.x;
  const int lane = threadIdx.x & 31;
  const float* row = scores + b * stride;
  uint64_t* w = win + (static_cast<int64_t>(b) * C + c) * seg;
  const uint64_t base_n = n / C, extra = n % C;
  const uint32_t first = static_cast<uint32_t>(c * base_n + (static_cast<uint64_t>(c) < extra ? c : extra));
  const uint32_t width = static_cast<uint32_t>(base_n + (static_cast<uint64_t>(c) < extra ? 1 : 0));
  const uint64_t lo = piv[4 * b], hi = piv[4 * b + 1], bp = piv[4 * b + 2];
  const unsigned vlo = static_cast<unsigned>(bp);
  const int bsh = static_cast<int>(bp >> 32);
  unsigned* ghg = gh + (static_cast<int64_t>(b) * kWinGroups + c % kWinGroups) * kWinBins;
  uint64_t* lsg = lists + (static_cast<int64_t>(b) * kWinGroups + c % kWinGroups) * kWinBins * kBinCap;
  if (threadIdx.x == 0) {
    s_above = 0;
    s_wn = 0;
    agg[static_cast<int64_t>(b) * C + c] = 0u;
  }
  __syncthreads();
  // window keys of the chunk -> shared stage; bin bookkeeping afterwards,
  // all threads at once (one global round trip instead of one per key)
  auto to_bin_list = [&](uint64_t k) {
    const unsigned bin = win_bin(k, vlo, bsh);
    const unsigned lp = atomicAdd(&ghg[bin], 1u);
    if (lp < kBinCap) lsg[bin * kBinCap + lp] = k;
  };
  unsigned above = 0;
  const uint32_t end = first + width;
  for (uint32_t i0 = first; i0 < end; i0 += NT * U) {
    float v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t i = i0 + u * NT + threadIdx.x;
      v[u] = i < end ? row[i] : 0.0f;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t i = i0 + u * NT + threadIdx.x;
      const bool valid = i < end;
      const uint64_t k = valid ? make_key(v[u], i) : 0ull;
      above += (valid && k > hi) ? 1u : 0u;
      const bool inw = valid && k >= lo && k <= hi;
      const unsigned bal = __ballot_sync(0xffffffffu, inw);
      if (bal) {
        unsigned base = 0;
        const int leader = __ffs(bal) - 1;
        if (lane == leader) base = atomicAdd(&s_wn, static_cast<unsigned>(__popc(bal)));
        base = __shfl_sync(0xffffffffu, base, leader);
        const unsigned pos = base + __popc(bal & ((1u << lane) - 1u));
        if (inw) {
          if (pos < STAGE) {
            s_win[pos] = k;
          } else {  // stage full: bookkeeping in place
            if (pos < seg) w[pos] = k;
            to_bin_list(k);
          }
        }
      }
    }
  }
  above = __reduce_add_sync(0xffffffffu, above);
  if (lane == 0 && above) atomicAdd(&s_above, above);
  __syncthreads();
  const unsigned staged = min(s_wn, static_cast<unsigned>(STAGE));
  for (unsigned t = threadIdx.x; t < staged; t += NT) {
    const uint64_t k = s_win[t];
    if (t < seg) w[t] = k;
    to_bin_list(k);
  }
  if (threadIdx.x == 0) {
    unsigned* cq = cnt + static_cast<int64_t>(b) * 2 * C;
    cq[c] = s_above;
    cq[C + c] = s_wn;
  }
}

// ---------------------------------------------------------------------
// S2' (list path). grid (C, B), 256 threads: every key >= lo of chunk c is
// appended to query b's list (warp-aggregated atomics on cnt[b]; list order
// is irrelevant — sel_fin_kernel selects T and emits through a row bitmap).
// Replaces window + window-select + emit with one scan and the finisher.
// ---------------------------------------------------------------------
__global__ void __launch_bounds__(kWinThreads) sel_wlist_kernel(
    const float* __restrict__ scores, int64_t stride, uint32_t n, const uint64_t* __restrict__ piv,
    unsigned* __restrict__ cnt, uint64_t* __restrict__ lists, int cap) {
  constexpr int NT = kWinThreads, U = kScanBatch, STAGE = 1024;
  // keys are staged per CTA and reserved with ONE global atomic per CTA:
  // same-address atomics from many CTAs serialise at L2
  __shared__ uint64_t s_keys[STAGE];
  __shared__ unsigned s_n, s_base;
  hire_dev::griddep_wait();
  hire_dev::LateTrigger late_trigger_;
  KTrace kt_(kKtWindow);
  const int b = blockIdx.y, C = gridDim.x, c = blockIdx.x;
  const int lane = threadIdx.x & 31;
  const float* row = scores + b * stride;
  const uint64_t base_n = n / C, extra = n % C;
  const uint32_t first = static_cast<uint32_t>(c * base_n + (static_cast<uint64_t>(c) < extra ? c : extra));
  const uint32_t end = first + static_cast<uint32_t>(base_n + (static_cast<uint64_t>(c) < extra ? 1 : 0));
  const uint64_t lo = piv[4 * b];
  uint64_t* L = lists + static_cast<int64_t>(b) * cap;
  if (threadIdx.x == 0) s_n = 0;
  __syncthreads();
  for (uint32_t i0 = first; i0 < end; i0 += NT * U) {
    float v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t i = i0 + u * NT + threadIdx.x;
      v[u] = i < end ? row[i] : 0.0f;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t i = i0 + u * NT + threadIdx.x;
      const uint64_t k = make_key(v[u], i);
      const bool in = i < end && k >= lo;
      const unsigned bal = __ballot_sync(0xffffffffu, in);
      if (bal) {
        const int leader = __ffs(bal) - 1;
        unsigned base = 0;
        if (lane == leader) base = atomicAdd(&s_n, static_cast<unsigned>(__popc(bal)));
        base = __shfl_sync(0xffffffffu, base, leader);
        const unsigned pos = base + __popc(bal & ((1u << lane) - 1u));
        if (in && pos < static_cast<unsigned>(STAGE)) s_keys[pos] = k;
        if (base + __popc(bal) > static_cast<unsigned>(STAGE)) {  // stage full: straight to the list
          const bool ovf = in && pos >= static_cast<unsigned>(STAGE);
          const unsigned ob = __ballot_sync(0xffffffffu, ovf);
          const int ol = __ffs(ob) - 1;
          unsigned gb = 0;
          if (lane == ol) gb = atomicAdd(cnt + b, static_cast<unsigned>(__popc(ob)));
          gb = __shfl_sync(0xffffffffu, gb, ol);
          const unsigned gp = gb + __popc(ob & ((1u << lane) - 1u));
          if (ovf && gp < static_cast<unsigned>(cap)) L[gp] = k;
        }
      }
    }
  }
  __syncthreads();
  const unsigned staged = min(s_n, static_cast<unsigned>(STAGE));
  if (threadIdx.x == 0) s_base = staged ? atomicAdd(cnt + b, staged) : 0u;
  __syncthreads();
  for (unsigned t = threadIdx.x; t < staged; t += NT)
    if (s_base + t < static_cast<unsigned>(cap)) L[s_base + t] = s_keys[t];
}

// ---------------------------------------------------------------------
// S12 (stream path): sample bound + list scan in ONE launch. grid (C, B),
// 256 threads. The score row is cut into 128-key granules (512 B, one float4
// per lane); chunk c owns granules g = c (mod C), a systematic sample of the
// whole row. The first CTA of a query to arrive (a ticket: atomicAdd on
// ticket[b], zero at rest) is the query's sampler, so it is running before
// any CTA that waits on it, whatever the dispatch order. The sampler's first
// 4096 keys (16 per thread) are the sample: tau <= the sample's rank-r_s key
// (r_s ~ k'/n * 4096 + margin, chosen on the host so that P[tau > T] ~ 1e-7
// for exchangeable rows; r_s <= 128, larger ranks take the pivot + list
// kernels): tau = the r_s-th largest of the 256 per-thread sample maxima
// (r_s distinct threads hold a key >= it; a warp bitonic sort of the maxima,
// then a rank by binary search over the 8 sorted lists — two barriers).
// tau, stripped of its index part, is published with an
// atomic on qtau[b]; the other CTAs of the query have their first two batches
// of loads in flight while they poll it. Every key >= tau of a chunk is staged
// in shared memory (seg slots) and appended to the query's compact list with
// one reservation atomic per CTA on qcnt[b] (bit 31: a stage or the list
// overflowed, or the bound never arrived).
// qcnt / qtau are zero at rest (cleared by sel_fin_kernel), which takes T =
// the k'-th largest listed key and accepts it when T >= tau (then every key
// >= T of the row is listed, so T is exact); otherwise it selects over the
// whole row.
// ---------------------------------------------------------------------
constexpr int kStrThreads = 256;
constexpr int kStrKpt = 16;
constexpr int kStrSample = kStrThreads * kStrKpt;  // 4096
constexpr int kStrSegMax = 1024;                   // keys staged per CTA
constexpr int kStrMaxChunks = 64;
constexpr int kStrFastRank = 128;                  // r_s up to this: bound from the per-thread maxima

__device__ __forceinline__ unsigned long long ld_relaxed_gpu_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ uint64_t shfl_xor_u64(uint64_t v, int m) {
  return static_cast<uint64_t>(__shfl_xor_sync(0xffffffffu, static_cast<unsigned long long>(v), m));
}

// r-th largest (1-based, r <= 256) of one key per thread over a 256-thread
// CTA; s_sorted: [8][32] u64. Keys are unique or 0 (padding, ranks last).
__device__ __forceinline__ uint64_t block256_rank_of_maxima(uint64_t x, int r, uint64_t* s_sorted, uint64_t* s_res) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int k = 2; k <= 32; k <<= 1) {
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
      const uint64_t o = shfl_xor_u64(x, j);
      const bool keep_max = ((lane & j) == 0) == ((lane & k) == 0);
      x = keep_max ? (x > o ? x : o) : (x < o ? x : o);
    }
  }
  s_sorted[wid * 32 + lane] = x;  // descending by lane
  if (threadIdx.x == 0) *s_res = 0ull;
  __syncthreads();
  int rank = lane;  // own list: keys above x
#pragma unroll
  for (int w = 0; w < 8; ++w) {  // (unrolled: the 7 searches are independent; rolled measured 0.6 us slower)
    if (w == wid) continue;
    const uint64_t* a = s_sorted + w * 32;
    int pos = 0;
#pragma unroll
    for (int step = 16; step > 0; step >>= 1)
      if (a[pos + step - 1] > x) pos += step;
    if (a[pos] > x) ++pos;
    rank += pos;
  }
  if (x != 0ull && rank == r - 1) *s_res = x;
  __syncthreads();
  return *s_res;
}

__global__ void __launch_bounds__(kStrThreads, 4) sel_stream_kernel(
    const float* __restrict__ scores, int64_t stride, uint32_t n, uint32_t r_s, uint32_t seg,
    unsigned* __restrict__ qcnt, unsigned long long* __restrict__ qtau, uint64_t* __restrict__ lists,
    int64_t list_stride, unsigned* __restrict__ ticket) {
  constexpr int NT = kStrThreads, NW = NT / 32, U = kStrKpt / 4;
  __shared__ uint64_t s_sorted[NT];
  __shared__ uint64_t s_keys[kStrSegMax];
  __shared__ unsigned s_n, s_base;
  __shared__ uint64_t s_res;
  __shared__ int s_ticket;
  hire_dev::griddep_wait();
  KTrace kt_(kKtWindow);
  const int b = blockIdx.y, C = gridDim.x, c = blockIdx.x;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  bool dbg = g_ktrace && threadIdx.x == 0 && b == 0;
  const float* row = scores + b * stride;
  const uint32_t G = (n + 127u) >> 7;
  // granule q of this warp's sequence: g = c + C * (wid + NW * q)
  auto gran = [&](uint32_t q) -> uint32_t { return static_cast<uint32_t>(c) + static_cast<uint32_t>(C) * (wid + NW * q); };
  auto load4 = [&](uint32_t g) -> float4 {
    const uint32_t i = (g << 7) + (lane << 2);
    if (g < G && i + 3 < n) return *reinterpret_cast<const float4*>(row + i);
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (g < G) {
      if (i < n) v.x = row[i];
      if (i + 1 < n) v.y = row[i + 1];
      if (i + 2 < n) v.z = row[i + 2];
    }
    return v;
  };
  // the ticket goes out ahead of the loads: its round trip would otherwise
  // queue behind the CTA's 32 KB of score loads in the SM's memory pipe (ncu:
  // 10 % of the kernel's warp time at the role barrier below)
  unsigned my_ticket = 0u;
  if (threadIdx.x == 0) my_ticket = atomicAdd(ticket + b, 1u);
  float4 v0[U], v1[U];
#pragma unroll
  for (int u = 0; u < U; ++u) v0[u] = load4(gran(u));
#pragma unroll
  for (int u = 0; u < U; ++u) v1[u] = load4(gran(U + u));
  // element e of granule g held by this lane
  auto idx_of = [&](uint32_t g, int e) -> uint32_t { return (g << 7) + (lane << 2) + e; };
  auto elem = [](const float4& v, int e) -> float { return e == 0 ? v.x : e == 1 ? v.y : e == 2 ? v.z : v.w; };
  // the loads are in flight; now the role: the first CTA of the query to
  // arrive samples (its own chunk), the others wait for its bound
  if (threadIdx.x == 0) {
    const unsigned t = my_ticket;
    if (t == static_cast<unsigned>(C) - 1u) ticket[b] = 0u;  // every CTA of the query arrived: back to zero
    s_ticket = static_cast<int>(t);
    s_n = 0;
  }
  __syncthreads();
  const bool sampler = s_ticket == 0;
  dbg = dbg && sampler;
  if (dbg) g_ktrace[70] = gtimer();
  uint64_t tau = 1ull;  // fewer sample keys than the rank: list every key
  bool late = false;    // the bound never arrived (the sampler always runs first: bounded wait all the same)
  if (sampler) {
    // valid sample keys: the chunk's first NW * U granules, all full but
    // possibly the row's last one
    long long n_in = 0;
    if (static_cast<uint32_t>(c) < G) {
      const uint32_t own = (G - 1u - c) / C + 1u;  // granules of this chunk
      const uint32_t ns = min(own, static_cast<uint32_t>(NW * U));
      n_in = static_cast<long long>(ns) * 128;
      const uint32_t tail = n & 127u;
      if (tail && (G - 1u - c) % C == 0u && (G - 1u - c) / C < static_cast<uint32_t>(NW * U)) n_in -= 128 - tail;
    }
    if (dbg) g_ktrace[71] = gtimer() + (v0[0].x == 77.125f);
    if (n_in >= static_cast<long long>(r_s)) {
      // this thread's largest sample key: the maximum value, lowest index on ties
      float best = 0.0f;
      uint32_t bi = 0xFFFFFFFFu;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t g = gran(u);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const uint32_t i = idx_of(g, e);
          const float v = elem(v0[u], e);
          const bool ok = g < G && i < n;
          if (ok && (bi == 0xFFFFFFFFu || v > best)) {
            best = v;
            bi = i;
          }
        }
      }
      const uint64_t mx = bi == 0xFFFFFFFFu ? 0ull : make_key(best, bi);
      tau = block256_rank_of_maxima(mx, static_cast<int>(r_s), s_sorted, &s_res);
    }
    // drop the index part: every key with tau's value word is listed, and the
    // scan needs only a float compare
    tau = (tau >> 32) << 32;
    if (tau == 0ull) tau = 1ull;  // (also: fewer than r_s threads held a valid key)
    if (threadIdx.x == 0) atomicExch(qtau + b, static_cast<unsigned long long>(tau));  // performed at L2
  } else {
    if (threadIdx.x == 0) {
      unsigned long long t = 0ull;
      const unsigned long long t0 = gtimer();
      while ((t = ld_relaxed_gpu_u64(qtau + b)) == 0ull) {
        if (gtimer() - t0 > 20000000ull) break;  // 20 ms
        __nanosleep(64);
      }
      s_res = t;
    }
    __syncthreads();
    tau = s_res;
    if (tau == 0ull) {
      late = true;
      tau = ~0ull;  // the finisher falls back
    }
  }
  if (dbg) g_ktrace[72] = gtimer() + (tau == 77ull);
  // keys >= tau -> the CTA's stage. tau carries no index part, so for real
  // scores key >= tau <=> !(x < tv) (NaN is listed too: harmless, the finisher
  // checks T >= tau). The streaming loop only records hits, one bit per key,
  // 64 keys (16 granules) per lane at a time; a block's hits are then written
  // with one warp scan and one shared atomic per warp, their values re-read
  // by index (L1).
  const float tv = key_value(tau);
  uint64_t mask = 0ull;
  auto hits4 = [&](const float4& v, uint32_t g) -> unsigned {
    if (g >= G) return 0u;
    unsigned h = (!(v.x < tv) ? 1u : 0u) | (!(v.y < tv) ? 2u : 0u) | (!(v.z < tv) ? 4u : 0u) | (!(v.w < tv) ? 8u : 0u);
    if ((g << 7) + 128u > n) {  // the row's last, partial granule
      const uint32_t i = idx_of(g, 0);
      h &= i + 3 < n ? 15u : i + 2 < n ? 7u : i + 1 < n ? 3u : i < n ? 1u : 0u;
    }
    return h;
  };
  auto flush = [&](uint32_t qbase) {  // hits of granules qbase .. qbase + 15 of this warp's sequence
    const int cn = __popcll(mask);
    if (__any_sync(0xffffffffu, cn != 0)) {
      int inc = cn;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += t;
      }
      unsigned base = 0;
      if (lane == 31) base = atomicAdd(&s_n, static_cast<unsigned>(inc));
      base = __shfl_sync(0xffffffffu, base, 31);
      unsigned pos = base + static_cast<unsigned>(inc - cn);
      while (mask) {
        const int p = __ffsll(static_cast<long long>(mask)) - 1;
        mask &= mask - 1ull;
        const uint32_t i = idx_of(gran(qbase + (p >> 2)), p & 3);
        if (pos < seg) s_keys[pos] = make_key(row[i], i);
        ++pos;
      }
    }
    mask = 0ull;
  };
#pragma unroll
  for (int u = 0; u < U; ++u) mask |= static_cast<uint64_t>(hits4(v0[u], gran(u))) << (4 * u);
  // the rest of the CTA's granules, one batch of loads ahead
  uint32_t qb = 0;  // first granule of the current 16-granule block
  for (uint32_t q0 = U; gran(q0) < G; q0 += U) {  // warp-uniform bound: gran() depends on wid and q only
    if (q0 - qb == 16u) {
      flush(qb);
      qb = q0;
    }
    float4 cur[U];
#pragma unroll
    for (int u = 0; u < U; ++u) cur[u] = v1[u];
#pragma unroll
    for (int u = 0; u < U; ++u) v1[u] = load4(gran(q0 + U + u));
#pragma unroll
    for (int u = 0; u < U; ++u) mask |= static_cast<uint64_t>(hits4(cur[u], gran(q0 + u))) << (4 * (q0 - qb + u));
  }
  flush(qb);
  hire_dev::griddep_launch();  // late: the finisher's 1024-thread CTAs must not take SMs from this grid
  __syncthreads();
  if (dbg) g_ktrace[73] = gtimer();
  // one reservation per CTA in the query's compact list (bit 31 of the count:
  // the finisher falls back — stage or list overflow, or the bound never came)
  const unsigned total = s_n;
  if (threadIdx.x == 0) {
    unsigned base = 0xFFFFFFFFu;
    if (total > seg || late) {
      atomicOr(qcnt + b, 0x80000000u);
    } else if (total) {
      base = atomicAdd(qcnt + b, total) & 0x7FFFFFFFu;
      if (base + total > static_cast<unsigned>(list_stride)) {
        atomicOr(qcnt + b, 0x80000000u);
        base = 0xFFFFFFFFu;
      }
    }
    s_base = base;
  }
  __syncthreads();
  const unsigned base = s_base;
  if (base != 0xFFFFFFFFu) {
    uint64_t* L = lists + static_cast<int64_t>(b) * list_stride + base;
    for (unsigned t = threadIdx.x; t < total; t += NT) L[t] = s_keys[t];
  }
  if (dbg) g_ktrace[74] = gtimer();
}

// ---------------------------------------------------------------------
// S2b. One 256-thread CTA per query: window counts -> r = K - above; the
// window keys are pulled from the chunk segments (position -> chunk by
// binary search over the prefix counts) and the r-th largest is T.
// Overflow (a chunk past its segment) or a bracket miss falls back to an
// exact select over the full row (correct, slow, counted in status).
// ---------------------------------------------------------------------
constexpr int kWselThreads = 256;
constexpr int kWselMaxChunks = 1024;

template <int NT, int KPT>
__device__ __forceinline__ uint64_t window_select(const uint64_t* w, const unsigned* s_pre, int C,
                                                  uint32_t seg, long long wn, long long r, RangeScratch* rs) {
  RegKeys<KPT> src;
#pragma unroll
  for (int j = 0; j < KPT; ++j) {
    const long long i = threadIdx.x + j * NT;
    uint64_t k = 0;
    if (i < wn) {
      int lo = 0, hi = C - 1;  // last chunk with s_pre[c] <= i
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (s_pre[mid] <= static_cast<unsigned>(i)) lo = mid;
        else hi = mid - 1;
      }
      k = w[static_cast<int64_t>(lo) * seg + (i - s_pre[lo])];
    }
    src.k[j] = k;
  }
  return block_range_select<NT>(src, wn, r, rs);
}

__global__ void __launch_bounds__(kWselThreads) sel_wselect_kernel(
    const float* __restrict__ scores, int64_t stride, uint32_t n, uint32_t K, int C,
    const uint64_t* __restrict__ piv, const uint64_t* __restrict__ win, uint32_t seg,
    const unsigned* __restrict__ cnt, const unsigned* __restrict__ gh, const uint64_t* __restrict__ lists,
    uint64_t* __restrict__ thr, int* __restrict__ status) {
  constexpr int NT = kWselThreads, NW = NT / 32;
  static_assert(NT == kWinBins, "one thread per window bin");
  __shared__ RangeScratch rs;
  __shared__ unsigned s_pre[kWselMaxChunks];
  __shared__ int s_scan[40];
  __shared__ long long s_red[NW];
  __shared__ uint64_t s_T;
  __shared__ long long s_r2;
  __shared__ int s_bstar, s_m, s_bad;
  hire_dev::griddep_wait();
  hire_dev::griddep_launch();
  KTrace kt_(kKtWindowSel);
  const int b = blockIdx.x;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const unsigned* cq = cnt + static_cast<int64_t>(b) * 2 * C;
  const uint64_t* w = win + static_cast<int64_t>(b) * C * seg;
  const uint64_t bp = piv[4 * b + 2];
  const unsigned vlo = static_cast<unsigned>(bp);
  const int bsh = static_cast<int>(bp >> 32);
  const bool dbg = g_ktrace && threadIdx.x == 0 && b == 0;
  if (dbg) g_ktrace[45] = gtimer();
  // chunk counts: keys above hi, window prefix
  long long above_l = 0;
  int over = 0;
  unsigned wsum = 0;
  for (int c0 = 0; c0 < C; c0 += NT) {
    const int c = c0 + threadIdx.x;
    unsigned wc = 0;
    if (c < C) {
      above_l += cq[c];
      wc = cq[C + c];
      over |= wc > seg;
    }
    int tot;
    const int ex = block_scan_excl<NT>(static_cast<int>(wc), s_scan, &tot);
    if (c < C) s_pre[c] = wsum + ex;
    wsum += tot;
  }
  {
    long long a = above_l;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
    if (lane == 0) s_red[wid] = a;
  }
  over = __syncthreads_or(over);
  long long above_t = 0;
#pragma unroll
  for (int v = 0; v < NW; ++v) above_t += s_red[v];
  const long long wn = wsum;
  const long long r = static_cast<long long>(K) - above_t;
  const bool ok = !over && r >= 1 && r <= wn;
  if (dbg) g_ktrace[46] = gtimer();
  if (ok) {
    // bin holding rank r: suffix sums over the 256 window bins
    const int t = threadIdx.x;
    unsigned hb = 0, hmax = 0;  // reversed: t = 0 is the top bin
#pragma unroll
    for (int g = 0; g < kWinGroups; ++g) {
      const unsigned v = gh[(static_cast<int64_t>(b) * kWinGroups + g) * kWinBins + (kWinBins - 1 - t)];
      hb += v;
      hmax = max(hmax, v);
    }
    int tot;
    const int ex = block_scan_excl<NT>(static_cast<int>(hb), s_scan, &tot);
    const long long above_bin = ex, incl = ex + static_cast<long long>(hb);
    if (threadIdx.x == 0) s_bad = 1;
    __syncthreads();
    if (above_bin < r && incl >= r) {
      s_bstar = kWinBins - 1 - t;
      s_r2 = r - above_bin;
      s_m = static_cast<int>(hb);
      s_bad = hmax > kBinCap ? 2 : 0;  // 2: the bin's lists overflowed
    }
    if (threadIdx.x == 0) rs.small_n = 0;
    __syncthreads();
  }
  const int bad = ok ? s_bad : 1;
  if (dbg) { g_ktrace[47] = gtimer(); g_ktrace[50] = ok ? s_m : 99999; }
  if (!bad && s_m <= kRsCompact) {
    // the bin's keys: its kWinGroups lists, one thread per list slot
    const unsigned bstar = static_cast<unsigned>(s_bstar);
    if (threadIdx.x < kWinGroups * kBinCap) {
      const int g = threadIdx.x / kBinCap, j = threadIdx.x % kBinCap;
      const unsigned cntg = gh[(static_cast<int64_t>(b) * kWinGroups + g) * kWinBins + bstar];
      if (static_cast<unsigned>(j) < cntg) {
        const uint64_t k = lists[((static_cast<int64_t>(b) * kWinGroups + g) * kWinBins + bstar) * kBinCap + j];
        const int p = atomicAdd(&rs.small_n, 1);
        if (p < kRsCompact) rs.ckeys[p] = k;
      }
    }
    __syncthreads();
    if (dbg) g_ktrace[48] = gtimer();
    const int m = s_m;
    const long long r2 = s_r2;
    uint64_t T;
    if (m <= 32) {
      if (threadIdx.x < m) {
        const uint64_t mine = rs.ckeys[threadIdx.x];
        int g = 0;
        for (int j = 0; j < m; ++j) g += rs.ckeys[j] > mine ? 1 : 0;
        if (g == r2 - 1) s_T = mine;
      }
      __syncthreads();
      T = s_T;
    } else {
      RegKeys<4> src;  // m <= 1024 = 4 * 256
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int i = threadIdx.x + j * NT;
        src.k[j] = i < m ? rs.ckeys[i] : 0ull;
      }
      __syncthreads();  // ckeys is reused by the select's compaction
      T = block_range_select<NT>(src, m, r2, &rs);
    }
    if (threadIdx.x == 0) thr[b] = T;
    if (dbg) g_ktrace[49] = gtimer();
    return;
  }
  // general path: select over the whole window (or the full row)
  uint64_t T;
  if (ok && wn <= 4096) {
    T = window_select<NT, 16>(w, s_pre, C, seg, wn, r, &rs);
  } else if (ok && wn <= 8192) {
    T = window_select<NT, 32>(w, s_pre, C, seg, wn, r, &rs);
  } else {
    if (threadIdx.x == 0 && status) atomicAdd(status, 1);
    RowKeys src{scores + b * stride, n};
    T = block_range_select<NT>(src, n, K, &rs);
  }
  if (threadIdx.x == 0) thr[b] = T;
}

// ---------------------------------------------------------------------
// S3. grid (C, B), 256 threads. Ordered emit of keys >= thr[b]. Chunk c
// publishes agg[b][c] = count | 0x80000000 (cleared by S2) and sums the
// aggregates of chunks < c (decoupled look-back over aggregates only). A
// CTA's chunk id is a ticket (atomicAdd on ticket[b], zero at rest): lower
// chunks belong to CTAs that started earlier, so the waits resolve whatever
// the dispatch order or residency (MPS, green contexts, preemption). Each warp
// owns a contiguous segment; loads are batched 8 groups of 32 per warp,
// ballots kept in shared memory for the write pass.
// ---------------------------------------------------------------------
constexpr int kEmitThreads = 256;
constexpr int kEmitBallots = 4096;  // u32 ballots kept in smem (131072 keys)

__global__ void __launch_bounds__(kEmitThreads) sel_emit_kernel(
    const float* __restrict__ scores, int64_t stride, uint32_t n, const uint64_t* __restrict__ thr,
    unsigned* __restrict__ agg, uint32_t* __restrict__ cand, int64_t cand_stride, unsigned* __restrict__ ticket) {
  constexpr int NT = kEmitThreads, NW = NT / 32, U = kScanBatch;
  __shared__ unsigned s_bal[kEmitBallots];
  __shared__ int s_scan[40];
  __shared__ unsigned s_pre[NW];
  __shared__ int s_chunk;
  hire_dev::griddep_wait();
  hire_dev::griddep_launch();
  KTrace kt_(kKtEmit);
  const int b = blockIdx.y, C = gridDim.x;
  if (threadIdx.x == 0) {
    const unsigned t = atomicAdd(ticket + b, 1u);
    if (t == static_cast<unsigned>(C) - 1u) ticket[b] = 0u;  // every chunk claimed: back to zero
    s_chunk = static_cast<int>(t);
  }
  __syncthreads();
  const int c = s_chunk;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (g_ktrace && threadIdx.x == 0 && b == 0 && c == C - 1) g_ktrace[39] = gtimer();
  if (g_ktrace && threadIdx.x == 0 && b == 0) atomicMax(&g_ktrace[43], gtimer());
  unsigned* ag = agg + static_cast<int64_t>(b) * C;
  const float* row = scores + b * stride;
  const uint64_t base_n = n / C, extra = n % C;
  const uint32_t first = static_cast<uint32_t>(c * base_n + (static_cast<uint64_t>(c) < extra ? static_cast<uint64_t>(c) : extra));
  const uint32_t width = static_cast<uint32_t>(base_n + (static_cast<uint64_t>(c) < extra ? 1 : 0));
  const uint32_t end = first + width;
  const uint64_t T = thr[b];
  const uint32_t groups = (width + 31) / 32;
  const uint32_t gpw = (groups + NW - 1) / NW;
  const uint32_t g0 = wid * gpw, g1 = min(groups, g0 + gpw);
  const bool keep = gpw * NW <= kEmitBallots;
  int cnt = 0;
  for (uint32_t gb = g0; gb < g1; gb += U) {
    float v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t i = first + (gb + u) * 32 + lane;
      v[u] = (gb + u < g1 && i < end) ? row[i] : 0.0f;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t g = gb + u;
      const uint32_t i = first + g * 32 + lane;
      const bool s = g < g1 && i < end && make_key(v[u], i) >= T;
      const unsigned bal = __ballot_sync(0xffffffffu, s);
      if (keep && lane == 0 && g < g1) s_bal[g] = bal;
      cnt += __popc(bal);
    }
  }
  const bool dbg = g_ktrace && threadIdx.x == 0 && b == 0 && c == C - 1;
  if (dbg) g_ktrace[40] = gtimer();
  int total;
  const int wbase = block_scan_excl<NT>(lane == 0 ? cnt : 0, s_scan, &total);
  if (dbg) g_ktrace[41] = gtimer();
  // the flag word carries the count itself: no data is published behind it,
  // so relaxed accesses suffice (no MEMBAR / L1 invalidate per probe)
  if (threadIdx.x == 0) atomicExch(&ag[c], static_cast<unsigned>(total) | 0x80000000u);  // performed at L2
  if (g_ktrace && threadIdx.x == 0 && b == 0) atomicMax(&g_ktrace[44], gtimer());
  unsigned pre = 0;
  for (int t = threadIdx.x; t < c; t += NT) {
    unsigned v;
    while (!((v = ld_relaxed_gpu(&ag[t])) & 0x80000000u)) {}
    pre += v & 0x7FFFFFFFu;
  }
  pre = __reduce_add_sync(0xffffffffu, pre);
  if (lane == 0) s_pre[wid] = pre;
  __syncthreads();
  unsigned cbase = 0;
#pragma unroll
  for (int v = 0; v < NW; ++v) cbase += s_pre[v];
  if (dbg) g_ktrace[42] = gtimer();
  uint32_t* out = cand + b * cand_stride;
  unsigned pos = cbase + __shfl_sync(0xffffffffu, wbase, 0);
  for (uint32_t g = g0; g < g1; ++g) {
    const uint32_t i = first + g * 32 + lane;
    unsigned bal;
    if (keep) {
      bal = s_bal[g];
    } else {
      const bool s = i < end && make_key(row[i], i) >= T;
      bal = __ballot_sync(0xffffffffu, s);
    }
    if ((bal >> lane) & 1u) out[pos + __popc(bal & ((1u << lane) - 1u))] = i;
    pos += __popc(bal);
  }
}

// ---------------------------------------------------------------------
// Final selection over an explicit pool (<= 32 * 512 keys) per query, one
// CTA per query: keys in registers (blocked layout), T by
// block_range_select, then
//   out_mode 0 RANK  : the K keys sorted by rank (+ softmax probabilities)
//   out_mode 1 INDEX : the K keys in pool order
//   out_mode 2 KEYS  : the K keys in pool order, padded with 0 to out_stride
// Pool entry i of query b: see final_select_kernel (select.cuh).
// ---------------------------------------------------------------------
constexpr int kFinal2Max = 32 * kSel2Threads;

template <int NT, int KPT>
__global__ void __launch_bounds__(NT) final2_kernel(
    const float* __restrict__ vals, int64_t vs, const uint32_t* __restrict__ idx, int64_t is,
    const uint64_t* __restrict__ src_keys, int n_per, int64_t part_stride, int n, int K,
    int out_mode, uint32_t* __restrict__ out_idx, float* __restrict__ out_val,
    float* __restrict__ out_prob, uint64_t* __restrict__ out_keys, int64_t out_stride, int fast_sel) {
  __shared__ union {
    RangeScratch rs;
    FastSelScratch fss;
  } u_;
  RangeScratch& rs = u_.rs;
  __shared__ double s_red[NT / 32];
  __shared__ int s_scan[40];
  extern __shared__ __align__(16) unsigned char smem_f2[];
  uint64_t* s_sel = reinterpret_cast<uint64_t*>(smem_f2);
  hire_dev::griddep_wait();
  hire_dev::griddep_launch();
  KTrace kt_(kKtFinal);
  const int b = blockIdx.x;
  if (g_ktrace && threadIdx.x == 0) atomicMax(&g_ktrace[82], gtimer());  // latest CTA start
  RegKeys<KPT> src;
  const int i0 = threadIdx.x * KPT;
#pragma unroll
  for (int j = 0; j < KPT; ++j) {
    const int i = i0 + j;
    uint64_t k = 0;
    if (i < n) {
      k = src_keys ? src_keys[static_cast<int64_t>(i / n_per) * part_stride + static_cast<int64_t>(b) * n_per + i % n_per]
                   : make_key(vals[b * vs + i], idx[b * is + i]);
    }
    src.k[j] = k;
  }
  int nv = 0;
#pragma unroll
  for (int j = 0; j < KPT; ++j) nv += src.k[j] != 0;
  nv = __reduce_add_sync(0xffffffffu, nv);
  if ((threadIdx.x & 31) == 0) s_scan[threadIdx.x >> 5] = nv;
  __syncthreads();
  int n_valid = 0;
#pragma unroll
  for (int v = 0; v < NT / 32; ++v) n_valid += s_scan[v];
  __syncthreads();
  const int Kq = min(K, n_valid);
  const bool dbg = g_ktrace && threadIdx.x == 0 && b == 0;
  if (dbg) g_ktrace[76] = gtimer();
  // K >= pool: everything is selected (no order statistic needed)
  // the K-th largest key: histogram select (fastsel.cuh, ~8 barriers whatever
  // the rank) or 16-way range splits (one barrier per split)
  uint64_t T;
  if (Kq >= n_valid) T = 1ull;
  else if (Kq < 1) T = ~0ull;
  else if (fast_sel) {
    T = block_fast_select<NT, KPT>(src.k, Kq, &u_.fss);
    __syncthreads();  // the scratch union changes hands
  } else T = block_range_select<NT>(src, n_valid, Kq, &rs);
  int c = 0;
#pragma unroll
  for (int j = 0; j < KPT; ++j) c += (src.k[j] && src.k[j] >= T) ? 1 : 0;
  int total;
  if (dbg) g_ktrace[77] = gtimer() + (T == 12345ull);
  int pos = block_scan_excl<NT>(c, s_scan, &total);
  if (out_mode == 1) {
#pragma unroll
    for (int j = 0; j < KPT; ++j)
      if (src.k[j] && src.k[j] >= T) {
        out_idx[b * out_stride + pos] = key_index(src.k[j]);
        out_val[b * out_stride + pos] = key_value(src.k[j]);
        ++pos;
      }
    return;
  }
  if (out_mode == 2) {
#pragma unroll
    for (int j = 0; j < KPT; ++j)
      if (src.k[j] && src.k[j] >= T) out_keys[b * out_stride + pos++] = src.k[j];
    for (int i = Kq + threadIdx.x; i < out_stride; i += NT) out_keys[b * out_stride + i] = 0ull;
    return;
  }
  // RANK: selected keys to smem, then sort descending
#pragma unroll
  for (int j = 0; j < KPT; ++j)
    if (src.k[j] && src.k[j] >= T) s_sel[pos++] = src.k[j];
  __syncthreads();
  if (Kq >= 1 && Kq <= NT && Kq <= 256) {
    // rank = number of selected keys greater (keys unique). The Kq x Kq
    // compares are spread over the whole CTA: thread t takes key t % Kq and
    // the t / Kq-th segment of the list, partial ranks meet in shared memory
    // (a single thread per key walks the list at one dependent shared load
    // per step: 1.8 us for 64 keys, 4.1 us for 128).
    int* s_rank = reinterpret_cast<int*>(rs.ckeys);  // the select is done with its scratch
    const int S = NT / Kq, len = (Kq + S - 1) / S;
    for (int i = threadIdx.x; i < Kq; i += NT) s_rank[i] = 0;
    __syncthreads();
    if (threadIdx.x < Kq * S) {
      const int i = threadIdx.x % Kq, j0 = (threadIdx.x / Kq) * len, j1 = min(Kq, j0 + len);
      const uint64_t mine = s_sel[i];
      int r = 0;
#pragma unroll 4
      for (int j = j0; j < j1; ++j) r += s_sel[j] > mine;
      if (r) atomicAdd(&s_rank[i], r);
    }
    __syncthreads();
    const uint64_t mine = threadIdx.x < Kq ? s_sel[threadIdx.x] : 0ull;
    const int rank = threadIdx.x < Kq ? s_rank[threadIdx.x] : 0;
    __syncthreads();
    if (threadIdx.x < Kq) s_sel[rank] = mine;
    __syncthreads();
  } else {
    int P = 1;
    while (P < Kq) P <<= 1;
    for (int i = Kq + threadIdx.x; i < P; i += NT) s_sel[i] = 0ull;
    __syncthreads();
    for (int size = 2; size <= P; size <<= 1) {
      for (int st = size >> 1; st > 0; st >>= 1) {
        for (int i = threadIdx.x; i < P / 2; i += NT) {
          const int lo = 2 * i - (i & (st - 1));
          const int hi = lo + st;
          const bool desc = (lo & size) == 0;
          const uint64_t a = s_sel[lo], c2 = s_sel[hi];
          if ((a < c2) == desc) {
            s_sel[lo] = c2;
            s_sel[hi] = a;
          }
        }
        __syncthreads();
      }
    }
  }
  if (dbg) g_ktrace[78] = gtimer();
  for (int i = threadIdx.x; i < Kq; i += NT) {
    out_idx[b * out_stride + i] = key_index(s_sel[i]);
    out_val[b * out_stride + i] = key_value(s_sel[i]);
  }
  if (out_prob) {
    // hire.hpp:135-142: p_i = float(exp(double(v_i) - v_max)) / double sum
    const double vmax = static_cast<double>(key_value(s_sel[0]));
    // one exp per element when every thread holds at most one (the usual
    // case); the sum keeps its order: per-thread terms, butterfly, warps ascending
    const bool one = Kq <= NT;
    double mine_e = 0.0;
    double local = 0.0;
    if (one) {
      if (threadIdx.x < Kq) mine_e = exp(static_cast<double>(key_value(s_sel[threadIdx.x])) - vmax);
      local = mine_e;
    } else {
      for (int j = threadIdx.x; j < Kq; j += NT) local += exp(static_cast<double>(key_value(s_sel[j])) - vmax);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) local += __shfl_xor_sync(0xffffffffu, local, o);
    if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = local;
    __syncthreads();
    double sum = 0.0;
#pragma unroll
    for (int v = 0; v < NT / 32; ++v) sum += s_red[v];
    if (one) {
      if (threadIdx.x < Kq)
        out_prob[b * out_stride + threadIdx.x] =
            static_cast<float>(static_cast<double>(static_cast<float>(mine_e)) / sum);
    } else {
      for (int j = threadIdx.x; j < Kq; j += NT) {
        const float pj = static_cast<float>(exp(static_cast<double>(key_value(s_sel[j])) - vmax));
        out_prob[b * out_stride + j] = static_cast<float>(static_cast<double>(pj) / sum);
      }
    }
  }
  if (dbg) g_ktrace[79] = gtimer();
  if (g_ktrace && threadIdx.x == 0) atomicMin(&g_ktrace[83], gtimer());  // earliest CTA end
}

// ---------------------------------------------------------------------
// Final top-K, ranked, for K <= W = 32 * SL keys (hire.hpp:74-80, 135-142):
// every warp sorts its W pool keys in registers (bitonic network: element
// e = slot * 32 + lane, partners at distance >= 32 are register swaps, below
// that shuffles), then a merge tree over the warps: the upper warp of a pair
// parks its sorted list in shared memory, the lower one takes max(own[e],
// other[W-1-e]) — a bitonic sequence holding the pair's top W — and re-sorts
// it with one merge network. log2(warps) barriers in all, against ~20 for the
// range select + scan + rank sort of final2_kernel, whose CTA-wide barriers
// dominate at these sizes; the result is the same ordered set (keys are
// unique). Warp 0 writes indices, values and the softmax.
// ---------------------------------------------------------------------
template <int SL>
struct WarpKeys {
  static constexpr int W = 32 * SL;
  uint64_t k[SL];
  // one compare-exchange stage at distance j inside blocks of size ksz
  // (descending where (e & ksz) == 0)
  template <int J, int KSZ>
  __device__ __forceinline__ void stage(int lane) {
    if constexpr (J >= 32) {
      constexpr int DS = J / 32;
#pragma unroll
      for (int s = 0; s < SL; ++s) {
        if ((s & DS) == 0) {
          const int sp = s | DS;
          const bool desc = ((s * 32) & KSZ) == 0;
          const uint64_t a = k[s], c = k[sp];
          const uint64_t hi = a > c ? a : c, lo = a > c ? c : a;
          k[s] = desc ? hi : lo;
          k[sp] = desc ? lo : hi;
        }
      }
    } else {
#pragma unroll
      for (int s = 0; s < SL; ++s) {
        const uint64_t o = static_cast<uint64_t>(__shfl_xor_sync(0xffffffffu, static_cast<unsigned long long>(k[s]), J));
        const int e = s * 32 + lane;
        const bool keep_max = ((lane & J) == 0) == ((e & KSZ) == 0);
        k[s] = keep_max ? (k[s] > o ? k[s] : o) : (k[s] < o ? k[s] : o);
      }
    }
  }
  template <int J, int KSZ>
  __device__ __forceinline__ void merge_from(int lane) {
    stage<J, KSZ>(lane);
    if constexpr (J > 1) merge_from<J / 2, KSZ>(lane);
  }
  template <int KSZ>
  __device__ __forceinline__ void sort_from(int lane) {
    merge_from<KSZ / 2, KSZ>(lane);
    if constexpr (KSZ < W) sort_from<KSZ * 2>(lane);
  }
  __device__ __forceinline__ void sort_desc(int lane) { sort_from<2>(lane); }
  __device__ __forceinline__ void merge_desc(int lane) { merge_from<W / 2, W>(lane); }
};

template <int NT, int SL>
__global__ void __launch_bounds__(NT) final3_kernel(
    const float* __restrict__ vals, int64_t vs, const uint32_t* __restrict__ idx, int64_t is,
    const uint64_t* __restrict__ src_keys, int n_per, int64_t part_stride, int n, int K,
    uint32_t* __restrict__ out_idx, float* __restrict__ out_val, float* __restrict__ out_prob, int64_t out_stride) {
  constexpr int NW = NT / 32, W = 32 * SL;
  __shared__ uint64_t s_buf[NW * W];
  hire_dev::griddep_wait();
  hire_dev::griddep_launch();
  KTrace kt_(kKtFinal);
  const int b = blockIdx.x, lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  WarpKeys<SL> wk;
#pragma unroll
  for (int s = 0; s < SL; ++s) {
    const int i = wid * W + s * 32 + lane;
    uint64_t k = 0;
    if (i < n) {
      k = src_keys ? src_keys[static_cast<int64_t>(i / n_per) * part_stride + static_cast<int64_t>(b) * n_per + i % n_per]
                   : make_key(vals[b * vs + i], idx[b * is + i]);
    }
    wk.k[s] = k;
  }
  wk.sort_desc(lane);
#pragma unroll
  for (int lvl = 1; lvl < NW; lvl <<= 1) {
    const int m = wid & (2 * lvl - 1);
    if (m == lvl) {
#pragma unroll
      for (int s = 0; s < SL; ++s) s_buf[wid * W + s * 32 + lane] = wk.k[s];
    }
    __syncthreads();
    if (m == 0) {
      const uint64_t* o = s_buf + (wid + lvl) * W;
#pragma unroll
      for (int s = 0; s < SL; ++s) {
        const uint64_t v = o[W - 1 - (s * 32 + lane)];
        wk.k[s] = wk.k[s] > v ? wk.k[s] : v;
      }
      wk.merge_desc(lane);
    }
  }
  if (wid != 0) return;
  // zeros (padding) sort last: the valid keys among the first K
  int nz = 0;
#pragma unroll
  for (int s = 0; s < SL; ++s) nz += (s * 32 + lane < K && wk.k[s] != 0ull) ? 1 : 0;
  const int Kq = __reduce_add_sync(0xffffffffu, nz);
#pragma unroll
  for (int s = 0; s < SL; ++s) {
    const int e = s * 32 + lane;
    if (e < Kq) {
      out_idx[b * out_stride + e] = key_index(wk.k[s]);
      out_val[b * out_stride + e] = key_value(wk.k[s]);
    }
  }
  if (out_prob) {
    // hire.hpp:135-142: p_i = float(exp(double(v_i) - v_max)) / double sum
    const double vmax = static_cast<double>(
        key_value(static_cast<uint64_t>(__shfl_sync(0xffffffffu, static_cast<unsigned long long>(wk.k[0]), 0))));
    double ex[SL];
    double local = 0.0;
#pragma unroll
    for (int s = 0; s < SL; ++s) {
      ex[s] = (s * 32 + lane < Kq) ? exp(static_cast<double>(key_value(wk.k[s])) - vmax) : 0.0;
      local += ex[s];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) local += __shfl_xor_sync(0xffffffffu, local, o);
#pragma unroll
    for (int s = 0; s < SL; ++s)
      if (s * 32 + lane < Kq)
        out_prob[b * out_stride + s * 32 + lane] =
            static_cast<float>(static_cast<double>(static_cast<float>(ex[s])) / local);
  }
}

}  // namespace hire_dev

namespace hire_dev {

// ---------------------------------------------------------------------
// Cluster selection: one thread-block cluster (CS <= 16 CTAs) per query.
// CTA r of the cluster owns the contiguous chunk r of the score row (keys
// in registers, blocked per thread). Every pass of the 16-way range split
// counts locally, publishes the CTA's 16 bin totals in its shared memory and
// crosses ONE cluster barrier; then each CTA reads the cluster's totals
// through distributed shared memory (mapa + ld.shared::cluster) and takes
// the same decision. The <= 32 survivors are ranked by every CTA from the
// cluster's lists; the ordered emit takes its offset from the lower ranks'
// counts. Rows up to CS * NT * KPT keys in one launch, no global atomics.
#if HIRE_EXPERIMENTS
// ---------------------------------------------------------------------
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ unsigned cluster_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ unsigned cluster_size() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t dsmem_addr(const void* p, unsigned rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
  return r;
}
__device__ __forceinline__ unsigned dsmem_ld_u32(const void* p, unsigned rank) {
  unsigned v;
  asm volatile("ld.shared::cluster.u32 %0, [%1];" : "=r"(v) : "r"(dsmem_addr(p, rank)) : "memory");
  return v;
}
__device__ __forceinline__ uint64_t dsmem_ld_u64(const void* p, unsigned rank) {
  unsigned long long v;
  asm volatile("ld.shared::cluster.u64 %0, [%1];" : "=l"(v) : "r"(dsmem_addr(p, rank)) : "memory");
  return static_cast<uint64_t>(v);
}

struct ClusterScratch {
  unsigned tot[2][16];   // this CTA's bin totals, by pass parity
  unsigned mm[2][2];     // this CTA's min / max of the projected word, by minmax parity
  uint64_t small[32];    // this CTA's survivors at the finish
  int nsmall;
  unsigned emit;         // this CTA's selected count
  unsigned st_lo, st_hi;  // decision broadcast inside the CTA
  long long st_rr, st_cnt;
  uint64_t result;
};

template <int NT, int KPT>
__global__ void __launch_bounds__(NT) sel_cluster_kernel(const float* __restrict__ scores, int64_t stride,
                                                         uint32_t n, uint32_t K, uint32_t* __restrict__ cand,
                                                         int64_t cand_stride) {
  constexpr int NW = NT / 32;
  __shared__ RangeScratch rs;
  __shared__ ClusterScratch cs;
  hire_dev::griddep_wait();
  hire_dev::griddep_launch();
  KTrace kt_(kKtPivot);
  const int b = blockIdx.y;
  const unsigned rank = cluster_rank(), CS = cluster_size();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const uint64_t base_n = n / CS, extra = n % CS;
  const uint32_t first = static_cast<uint32_t>(rank * base_n + (rank < extra ? rank : extra));
  const uint32_t width = static_cast<uint32_t>(base_n + (rank < extra ? 1 : 0));
  const float* row = scores + b * stride;
  RegKeys<KPT> src;
  const uint32_t i0 = threadIdx.x * KPT;
#pragma unroll
  for (int j = 0; j < KPT; ++j) {
    const uint32_t i = i0 + j;
    src.k[j] = i < width ? make_key(row[first + i], first + i) : 0ull;
  }
  if (threadIdx.x == 0) cs.nsmall = 0;
  RangeState st;
  st.phase = 0;
  st.vstar = 0;
  st.rr = K;
  st.cnt = n;
  st.par = 0;
  st.above = 0;
  st.bracket = 0;
  st.stop = 0;
  int mpar = 0;
  // cluster min / max of the projected word
  auto cluster_minmax = [&]() {
    unsigned mn = 0xFFFFFFFFu, mx = 0u;
    src.each([&](uint64_t k, int) {
      unsigned x;
      const bool ok = rs_project(st, k, &x);
      mn = ok ? min(mn, x) : mn;
      mx = ok ? max(mx, x) : mx;
    });
    __syncwarp();
    mn = __reduce_min_sync(0xffffffffu, mn);
    mx = __reduce_max_sync(0xffffffffu, mx);
    if (lane == 0) {
      rs.red[0][wid] = mn;
      rs.red[1][wid] = mx;
    }
    __syncthreads();
    if (wid == 0) {
      unsigned a = lane < NW ? rs.red[0][lane] : 0xFFFFFFFFu, c = lane < NW ? rs.red[1][lane] : 0u;
      a = __reduce_min_sync(0xffffffffu, a);
      c = __reduce_max_sync(0xffffffffu, c);
      if (lane == 0) {
        cs.mm[mpar][0] = a;
        cs.mm[mpar][1] = c;
      }
    }
    cluster_sync_all();
    unsigned a = 0xFFFFFFFFu, c = 0u;
    if (lane < static_cast<int>(CS)) {
      a = dsmem_ld_u32(&cs.mm[mpar][0], lane);
      c = dsmem_ld_u32(&cs.mm[mpar][1], lane);
    }
    st.lo = __reduce_min_sync(0xffffffffu, a);
    st.hi = __reduce_max_sync(0xffffffffu, c);
    mpar ^= 1;
  };
  cluster_minmax();
  for (;;) {
    if (st.lo == st.hi) {
      if (st.phase == 1) break;  // index words are unique: T = (vstar, lo)
      if (st.cnt > 32) {
        st.phase = 1;
        st.vstar = st.lo;
        cluster_minmax();
        continue;
      }
    }
    if (st.cnt <= 32) break;
    const unsigned lo = st.lo, hi = st.hi, range = hi - lo;
    int sh = 32 - __clz(range) - 4;
    if (sh < 0) sh = 0;
    const int pp = st.par;
    unsigned w[8];
#pragma unroll
    for (int m = 0; m < 8; ++m) w[m] = 0;
    if (st.phase == 0 && lo != 0) {
      src.count_value_bins(lo, range, sh, w);
    } else {
      unsigned a = 0, c = 0;
      src.each([&](uint64_t k, int j) {
        unsigned x;
        const bool ok = rs_project(st, k, &x);
        const unsigned dlt = x - lo;
        const unsigned bin = dlt >> sh;
        const unsigned inc = (ok && dlt <= range) ? (1u << ((bin & 7u) << 2)) : 0u;
        a += (bin & 8u) ? 0u : inc;
        c += (bin & 8u) ? inc : 0u;
        if (j % 15 == 14) {
          widen_bins(a, c, w);
          a = 0;
          c = 0;
        }
      });
      widen_bins(a, c, w);
    }
    __syncwarp();
    unsigned a4[4], a2[2];
    {
      const bool h = lane & 4;
#pragma unroll
      for (int m = 0; m < 4; ++m)
        a4[m] = (h ? w[m + 4] : w[m]) + __shfl_xor_sync(0xffffffffu, h ? w[m] : w[m + 4], 4);
    }
    {
      const bool h = lane & 2;
#pragma unroll
      for (int m = 0; m < 2; ++m)
        a2[m] = (h ? a4[m + 2] : a4[m]) + __shfl_xor_sync(0xffffffffu, h ? a4[m] : a4[m + 2], 2);
    }
    const bool h1 = lane & 1;
    unsigned mine = (h1 ? a2[1] : a2[0]) + __shfl_xor_sync(0xffffffffu, h1 ? a2[0] : a2[1], 1);
    mine += __shfl_xor_sync(0xffffffffu, mine, 8);
    mine += __shfl_xor_sync(0xffffffffu, mine, 16);
    if (lane < 8) rs.cnt[pp][wid][lane] = mine;
    __syncthreads();
    if (wid == 0) {  // CTA totals of the 16 bins -> shared, for the cluster
      unsigned t = 0;
      if (lane < 16) {
#pragma unroll
        for (int v = 0; v < NW; ++v) t += rs.cnt[pp][v][lane >> 1];
        t = (lane & 1) ? (t >> 16) : (t & 0xFFFFu);
        cs.tot[pp][lane] = t;
      }
    }
    cluster_sync_all();
    // every warp: the cluster's totals, the same decision everywhere
    unsigned tot = 0;
    if (lane < 16)
      for (unsigned r2 = 0; r2 < CS; ++r2) tot += dsmem_ld_u32(&cs.tot[pp][lane], r2);
    st.par ^= 1;
    __syncwarp();
    unsigned cum = tot;
#pragma unroll
    for (int o = 1; o < 16; o <<= 1) {
      const unsigned t = __shfl_down_sync(0xffffffffu, cum, o);
      if (lane + o < 16) cum += t;
    }
    const unsigned bal = __ballot_sync(0xffffffffu, lane < 16 && static_cast<long long>(cum) >= st.rr);
    const int bs = 31 - __clz(bal & 0xFFFFu);
    const unsigned cum_next = __shfl_sync(0xffffffffu, cum, bs + 1);
    const unsigned tb = __shfl_sync(0xffffffffu, tot, bs);
    const unsigned nlo = lo + (static_cast<unsigned>(bs) << sh);
    const unsigned span = (1u << sh) - 1u;
    st.hi = (hi - nlo > span) ? nlo + span : hi;
    st.lo = nlo;
    st.rr -= static_cast<long long>(cum_next);
    st.cnt = tb;
  }
  uint64_t T;
  if (st.phase == 1 && st.lo == st.hi) {
    T = (static_cast<uint64_t>(st.vstar) << 32) | st.lo;
  } else {
    // <= 32 survivors over the cluster: each CTA lists its own, every CTA
    // ranks the union
    const unsigned lo = st.lo, hi = st.hi;
    src.each([&](uint64_t k, int) {
      unsigned x;
      if (rs_project(st, k, &x) && x - lo <= hi - lo) {
        const int p = atomicAdd(&cs.nsmall, 1);
        if (p < 32) cs.small[p] = k;
      }
    });
    cluster_sync_all();
    if (wid == 0) {
      // lane l gathers the l-th survivor of the union
      int cnt_r = lane < static_cast<int>(CS) ? static_cast<int>(dsmem_ld_u32(&cs.nsmall, lane)) : 0;
      cnt_r = min(cnt_r, 32);
      int incl = cnt_r;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
      }
      const int total = min(__shfl_sync(0xffffffffu, incl, 31), 32);
      if (lane < 16) rs.scan[lane] = incl;  // inclusive prefix by rank
      __syncwarp();
      uint64_t mine = 0;
      if (lane < total) {
        int r2 = 0;
        while (rs.scan[r2] <= lane) ++r2;
        const int before = r2 > 0 ? rs.scan[r2 - 1] : 0;
        mine = dsmem_ld_u64(&cs.small[lane - before], static_cast<unsigned>(r2));
      }
      int g = 0;
      for (int j = 0; j < total; ++j)
        g += static_cast<uint64_t>(__shfl_sync(0xffffffffu, static_cast<unsigned long long>(mine), j)) > mine ? 1 : 0;
      if (lane < total && g == st.rr - 1) cs.result = mine;
    }
    __syncthreads();
    T = cs.result;
  }
  // ordered emit: offset of this CTA = selected keys of the lower ranks
  int c = 0;
#pragma unroll
  for (int j = 0; j < KPT; ++j) c += (src.k[j] && src.k[j] >= T) ? 1 : 0;
  int total;
  int pos = block_scan_excl<NT>(c, rs.scan, &total);
  if (threadIdx.x == 0) cs.emit = static_cast<unsigned>(total);
  cluster_sync_all();
  unsigned off = 0;
  if (lane < static_cast<int>(rank)) off = dsmem_ld_u32(&cs.emit, lane);
  off = __reduce_add_sync(0xffffffffu, off);
  uint32_t* out = cand + b * cand_stride;
  pos += static_cast<int>(off);
#pragma unroll
  for (int j = 0; j < KPT; ++j)
    if (src.k[j] && src.k[j] >= T) out[pos++] = first + i0 + j;
  cluster_sync_all();  // no CTA leaves while its shared memory may still be read
}

#endif  // HIRE_EXPERIMENTS

}  // namespace hire_dev
