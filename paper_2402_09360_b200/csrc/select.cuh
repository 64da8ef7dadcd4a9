// select.cuh — exact top-k' / top-k selection on 64-bit rank keys.
//
// Reference semantics: topk_select (linalg.hpp:157-176) under ranks_before
// (linalg.hpp:129-133): value descending, index ascending. With the key
// encoding of common.cuh this is "the K largest keys", found by an 8-bit
// MSD radix select in shared memory (one CTA per query), then compacted in
// pool order (ascending index) or bitonic-sorted by rank.
//
// Bucketed candidate selection (BASELINE.json cfg3): the score vector is
// cut into contiguous buckets (the shard width rule, distributed.hpp:53-57);
// bucket_topt_kernel keeps each bucket's top-t survivors. Then
//   SEL_EXACT    : select top-k' of the survivors; any bucket whose weakest
//                  survivor made the cut may have lost members, so those
//                  buckets are re-read in full and the selection repeated.
//                  The result provably equals topk_select on all scores.
//   SEL_BUCKETED : the literal rule — top-k' of the survivors, no repair
//                  (oracle: orc_bucketed_select).
#pragma once
#include "common.cuh"

namespace hire_dev {

#ifdef HIRE_SEL_DEBUG
__device__ long long g_sel_dbg[32];
#define SEL_STAMP(i) do { if (threadIdx.x == 0) g_sel_dbg[i] = clock64(); } while (0)
#else
#define SEL_STAMP(i) do { } while (0)
#endif

// Block-wide exclusive scan of one int per thread. Returns the exclusive
// prefix; *total gets the block sum. s_tmp needs NT/32 + 1 ints.
template <int NT>
__device__ __forceinline__ int block_exclusive_scan(int v, int* s_tmp, int* total) {
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
    if (lane < NT / 32) s_tmp[lane] = t;  // inclusive warp-total prefix
    if (lane == NT / 32 - 1) s_tmp[NT / 32] = t;
  }
  __syncthreads();
  const int before = w > 0 ? s_tmp[w - 1] : 0;
  *total = s_tmp[NT / 32];
  __syncthreads();
  return before + inc - v;
}

constexpr int kSmallKeys = 1024;  // survivor buffer once the threshold bin is small
constexpr int kWinKeys = 2048;    // sampled-bracket window
constexpr int kWin2Keys = 1024;   // second-level window

struct SelectScratch {
  unsigned int wcnt[32][16];  // per-warp digit counts
  int scan[64];
  int sel[4];
  uint64_t red[2][32];
  uint64_t small[kSmallKeys];
  int small_n;
  uint64_t samp[256];
  uint64_t win[kWinKeys];
  uint64_t win2[kWin2Keys];
  int win_n;
  uint64_t piv[4];
};

// Packed digit counters: 16 bins of 16 bits in 4 u64 registers.
struct Cnt16 {
  uint64_t c[4];
  __device__ __forceinline__ void zero() { c[0] = c[1] = c[2] = c[3] = 0; }
  __device__ __forceinline__ void add(int d) {
    const uint64_t inc = 1ull << ((d & 3) * 16);
    const int r = d >> 2;
    c[0] += r == 0 ? inc : 0ull;
    c[1] += r == 1 ? inc : 0ull;
    c[2] += r == 2 ? inc : 0ull;
    c[3] += r == 3 ? inc : 0ull;
  }
  __device__ __forceinline__ void warp_reduce() {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
#pragma unroll
      for (int q = 0; q < 4; ++q) c[q] += __shfl_xor_sync(0xffffffffu, c[q], o);
  }
  __device__ __forceinline__ unsigned get(int d) const {
    const int r = d >> 2;
    const uint64_t v = r == 0 ? c[0] : (r == 1 ? c[1] : (r == 2 ? c[2] : c[3]));
    return static_cast<unsigned>((v >> ((d & 3) * 16)) & 0xFFFF);
  }
};

// Finds (prefix, mask) such that exactly K of the n keys satisfy
// (key & mask) >= prefix — i.e. the K largest. Keys must be unique among
// non-padding entries (indices are unique); 1 <= K <= n.
//   * bits shared by every key (AND == OR) are skipped up front;
//   * 4-bit digits, counted in packed 16-bit register counters and reduced
//     with warp shuffles — no shared-memory atomics (2 cycles/lane on
//     Blackwell, 32 per warp instruction when lanes collide);
//   * once the bin holding the K-th key has <= kSmallKeys members they are
//     compacted into a small buffer and the remaining digits are resolved
//     there;
//   * stops as soon as that bin is taken whole.
template <int NT, class KeyAt>
__device__ void block_radix_select(KeyAt key_at, int n, int K, SelectScratch* sc,
                                   uint64_t* out_prefix, uint64_t* out_mask) {
  static_assert(NT >= 32 && NT <= 1024, "block size");
  constexpr int NW = NT / 32;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint64_t band = ~0ull, bor = 0ull;
  for (int i = threadIdx.x; i < n; i += NT) {
    const uint64_t k = key_at(i);
    band &= k;
    bor |= k;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    band &= __shfl_xor_sync(0xffffffffu, band, o);
    bor |= __shfl_xor_sync(0xffffffffu, bor, o);
  }
  if (lane == 0) {
    sc->red[0][wid] = band;
    sc->red[1][wid] = bor;
  }
  if (threadIdx.x == 0) sc->small_n = 0;
  __syncthreads();
  if (threadIdx.x < 32) {
    uint64_t a = threadIdx.x < NW ? sc->red[0][threadIdx.x] : ~0ull;
    uint64_t o2 = threadIdx.x < NW ? sc->red[1][threadIdx.x] : 0ull;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      a &= __shfl_xor_sync(0xffffffffu, a, o);
      o2 |= __shfl_xor_sync(0xffffffffu, o2, o);
    }
    if (threadIdx.x == 0) {
      sc->red[0][0] = a;
      sc->red[1][0] = o2;
    }
  }
  __syncthreads();
  const uint64_t all_and = sc->red[0][0], all_or = sc->red[1][0];
  const uint64_t diff = all_and ^ all_or;
  __syncthreads();
  if (diff == 0) {  // one distinct key
    *out_prefix = all_and;
    *out_mask = ~0ull;
    return;
  }
  int hi = 63 - __clzll(static_cast<long long>(diff));
  uint64_t mask = hi == 63 ? 0ull : (~0ull << (hi + 1));
  uint64_t prefix = all_and & mask;
  int krem = K;
  bool small = false;
  int ns = 0;
  while (hi >= 0) {
    const int w = hi + 1 < 4 ? hi + 1 : 4;
    const int shift = hi - w + 1;
    const uint64_t dmask = ((1ull << w) - 1ull) << shift;
    Cnt16 cnt;
    cnt.zero();
    if (small) {
      for (int i = threadIdx.x; i < ns; i += NT) {
        const uint64_t k = sc->small[i];
        if ((k & mask) == prefix) cnt.add(static_cast<int>((k >> shift) & 0xF));
      }
    } else {
      for (int i = threadIdx.x; i < n; i += NT) {
        const uint64_t k = key_at(i);
        if ((k & mask) == prefix) cnt.add(static_cast<int>((k >> shift) & 0xF));
      }
    }
    cnt.warp_reduce();
    if (lane < 16) sc->wcnt[wid][lane] = cnt.get(lane);
    __syncthreads();
    if (threadIdx.x < 32) {
      // lane l owns digit 15 - l (descending), summed over warps
      unsigned v = 0;
      if (lane < 16)
        for (int q = 0; q < NW; ++q) v += sc->wcnt[q][15 - lane];
      unsigned inc = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned nn = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += nn;
      }
      if (lane < 16 && static_cast<int>(inc) >= krem && static_cast<int>(inc - v) < krem) {
        sc->sel[0] = 15 - lane;
        sc->sel[1] = krem - static_cast<int>(inc - v);
        sc->sel[2] = static_cast<int>(v);
      }
    }
    __syncthreads();
    const int dg = sc->sel[0];
    krem = sc->sel[1];
    const int cntb = sc->sel[2];
    prefix |= static_cast<uint64_t>(dg) << shift;
    mask |= dmask;
    if (cntb == krem) break;  // the whole bin is in the top K
    hi = shift - 1;
    if (!small && cntb <= kSmallKeys && hi >= 0) {
      // compact the bin's members (order is irrelevant for the threshold)
      __syncthreads();
      for (int i0 = 0; i0 < n; i0 += NT) {
        const int i = i0 + threadIdx.x;
        uint64_t k = 0;
        bool m = false;
        if (i < n) {
          k = key_at(i);
          m = (k & mask) == prefix;
        }
        const unsigned bal = __ballot_sync(0xffffffffu, m);
        int base = 0;
        if (lane == 0 && bal) base = atomicAdd(&sc->small_n, __popc(bal));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (m) sc->small[base + __popc(bal & ((1u << lane) - 1u))] = k;
      }
      __syncthreads();
      ns = sc->small_n;
      small = true;
    }
    __syncthreads();
  }
  __syncthreads();
  *out_prefix = prefix;
  *out_mask = mask;
}

__device__ __forceinline__ bool key_selected(uint64_t k, uint64_t prefix, uint64_t mask) {
  return (k & mask) >= prefix && k != 0;
}

// ---------------------------------------------------------------------
// K-th largest key by recursive sampled brackets (exact).
// Level: rank a 256-key sample by counting (S^2 compares, no sort), take the
// sample keys at ranks (K-1)S/n -/+ 3.5 sigma as pivots, make ONE pass that
// counts keys above the upper pivot and gathers the keys between the pivots
// into a buffer; recurse on the buffer with K' = K - above. At <= 256 keys
// the exact K-th key is found by rank-by-counting. Any miss (K-th outside the
// bracket, buffer overflow) falls back to the radix select — the threshold is
// exact either way. Returns prefix = K-th key, mask = all ones.
// ---------------------------------------------------------------------
// Rank of keys[t] among keys[0..n) (#greater), with NT/256 threads per key
// (adjacent lanes) each counting a slice and combining by shuffles.
// Calls f(t, rank) once per key t < n. All threads must call.
template <int NT, class F>
__device__ __forceinline__ void block_rank_256(const uint64_t* keys, int n, F f) {
  static_assert(NT % 256 == 0, "NT multiple of 256");
  constexpr int G = NT / 256;  // threads per key (1, 2 or 4)
  const int t = threadIdx.x / G, part = threadIdx.x % G;
  int r = 0;
  uint64_t mine = 0;
  if (t < n) {
    mine = keys[t];
    const int per = (n + G - 1) / G;
    const int j0 = part * per, j1 = min(n, j0 + per);
#pragma unroll 8
    for (int j = j0; j < j1; ++j) r += keys[j] > mine;
  }
#pragma unroll
  for (int o = 1; o < G; o <<= 1) r += __shfl_xor_sync(0xffffffffu, r, o);
  if (t < n && part == 0) f(t, r);
}

template <int NT>
__device__ uint64_t rank_select_small(const uint64_t* keys, int n, int K, SelectScratch* sc) {
  // n <= 256: the key whose rank (number of greater keys) is K-1
  if (threadIdx.x == 0) sc->piv[2] = 0ull;
  __syncthreads();
  block_rank_256<NT>(keys, n, [&](int t, int r) {
    if (r == K - 1) sc->piv[2] = keys[t];
  });
  __syncthreads();
  const uint64_t th = sc->piv[2];
  __syncthreads();
  return th;
}

// one bracketing level over key_at[0..n): returns false on a miss.
template <int NT, class KeyAt>
__device__ bool bracket_level(KeyAt key_at, int n, int K, SelectScratch* sc, uint64_t* dst, int cap,
                              int* out_n, int* out_need) {
  constexpr int S = 128;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  SEL_STAMP(0);
  for (int j = threadIdx.x; j < S; j += NT) sc->samp[j] = key_at(static_cast<int>((static_cast<int64_t>(j) * n) / S));
  if (threadIdx.x == 0) {
    sc->win_n = 0;
    sc->piv[0] = ~0ull;  // upper pivot (+inf)
    sc->piv[1] = 0ull;   // lower pivot (-inf: below every real key)
  }
  __syncthreads();
  SEL_STAMP(1);
  const float p = static_cast<float>(K) / static_cast<float>(n);
  const float mu = static_cast<float>(K - 1) * S / static_cast<float>(n);
  const float delta = fmaxf(3.5f * sqrtf(S * p * (1.0f - p)), 3.0f);
  const int r_hi = static_cast<int>(floorf(mu - delta));
  const int r_lo = static_cast<int>(ceilf(mu + delta));
  block_rank_256<NT>(sc->samp, S, [&](int j, int r) {
    if (r == r_hi) sc->piv[0] = sc->samp[j];
    if (r == r_lo) sc->piv[1] = sc->samp[j];
  });
  __syncthreads();
  SEL_STAMP(2);
  const uint64_t hi = sc->piv[0], lo = sc->piv[1];
  int above = 0;
  constexpr int UNR = 4;
  for (int i0 = 0; i0 < n; i0 += NT * UNR) {
    uint64_t k[UNR];
    bool in[UNR];
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      const int i = i0 + u * NT + threadIdx.x;
      k[u] = i < n ? key_at(i) : 0ull;
      in[u] = i < n && k[u] > lo && k[u] <= hi;
      above += (i < n) && k[u] > hi;
    }
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      const unsigned bal = __ballot_sync(0xffffffffu, in[u]);
      int base = 0;
      if (lane == 0 && bal) base = atomicAdd(&sc->win_n, __popc(bal));
      base = __shfl_sync(0xffffffffu, base, 0);
      const int pos = base + __popc(bal & ((1u << lane) - 1u));
      if (in[u] && pos < cap) dst[pos] = k[u];
    }
  }
  above = __reduce_add_sync(0xffffffffu, above);
  if (lane == 0) sc->scan[wid] = above;
  __syncthreads();
  int tot = 0;
  for (int w = 0; w < NT / 32; ++w) tot += sc->scan[w];
  const int nw = sc->win_n;
  __syncthreads();
  SEL_STAMP(3);
  *out_n = nw;
  *out_need = K - tot;
  return *out_need >= 1 && *out_need <= nw && nw <= cap;
}

template <int NT, class KeyAt>
__device__ void block_select_kth(KeyAt key_at, int n, int K, SelectScratch* sc,
                                 uint64_t* out_prefix, uint64_t* out_mask) {
  if (NT < 256) {
    block_radix_select<NT>(key_at, n, K, sc, out_prefix, out_mask);
    return;
  }
  *out_mask = ~0ull;
  if (n <= 256) {
    for (int i = threadIdx.x; i < n; i += NT) sc->win2[i] = key_at(i);
    __syncthreads();
    *out_prefix = rank_select_small<NT>(sc->win2, n, K, sc);
    return;
  }
  int n1 = n, k1 = K;
  bool ok = true;
  // level 1 over the source, level 2 over the window, then rank-count
  const uint64_t* cur = nullptr;
  if (n > 256) {
    ok = bracket_level<NT>(key_at, n, K, sc, sc->win, kWinKeys, &n1, &k1);
    cur = sc->win;
  }
  for (int lvl = 0; ok && n1 > 256 && lvl < 4; ++lvl) {
    uint64_t* dst = (cur == sc->win) ? sc->win2 : sc->win;
    const int cap = (dst == sc->win2) ? kWin2Keys : kWinKeys;
    int n2, k2;
    const uint64_t* src = cur;
    ok = bracket_level<NT>([&](int i) { return src[i]; }, n1, k1, sc, dst, cap, &n2, &k2);
    cur = dst;
    n1 = n2;
    k1 = k2;
  }
  SEL_STAMP(4);
  if (ok && n1 <= 256) {
    if (cur != sc->win2) {
      for (int i = threadIdx.x; i < n1; i += NT) sc->win2[i] = cur[i];
      __syncthreads();
    }
    *out_prefix = rank_select_small<NT>(sc->win2, n1, k1, sc);
    SEL_STAMP(5);
#ifdef HIRE_SEL_DEBUG
    if (threadIdx.x == 0) { g_sel_dbg[10] = n1; g_sel_dbg[11] = k1; }
#endif
    return;
  }
  SEL_STAMP(6);
  block_radix_select<NT>(key_at, n, K, sc, out_prefix, out_mask);
  SEL_STAMP(7);
}

// The exact K-th largest key (block_select_kth may return a (prefix, mask)
// bin rule from its radix fallback; this turns any result into one key).
template <int NT, class KeyAt>
__device__ uint64_t block_kth_key(KeyAt key_at, int n, int K, SelectScratch* sc) {
  uint64_t prefix, mask;
  block_select_kth<NT>(key_at, n, K, sc, &prefix, &mask);
  if (mask == ~0ull) return prefix;
  uint64_t t = ~0ull;
  for (int i = threadIdx.x; i < n; i += NT) {
    const uint64_t k = key_at(i);
    if (key_selected(k, prefix, mask) && k < t) t = k;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const uint64_t u = __shfl_xor_sync(0xffffffffu, t, o);
    t = u < t ? u : t;
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) sc->red[0][wid] = t;
  __syncthreads();
  uint64_t tt = ~0ull;
  for (int w = 0; w < NT / 32; ++w) tt = sc->red[0][w] < tt ? sc->red[0][w] : tt;
  __syncthreads();
  return tt;
}

// Order-preserving compaction of the selected keys. Warp w owns the
// contiguous range [w*seg, (w+1)*seg), walked 32 keys at a time
// (lane-contiguous, bank-conflict free). The count pass stores its ballots
// in the (now free) survivor buffer, so the emit pass only rebuilds the keys
// of selected lanes. emit(pos, i, key).
template <int NT, class KeyAt, class Emit>
__device__ void block_compact(KeyAt key_at, int n, uint64_t prefix, uint64_t mask,
                              SelectScratch* sc, Emit emit) {
  constexpr int NW = NT / 32;
  constexpr int CAP = kSmallKeys * 2;  // u32 ballots available
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int seg = ((n + NW - 1) / NW + 31) / 32 * 32;
  const int lo = min(n, wid * seg), hi = min(n, lo + seg);
  const int nchunks = (hi - lo + 31) / 32;
  const int cpw = (seg + 31) / 32;  // chunks per warp (stride in the ballot store)
  unsigned* bstore = reinterpret_cast<unsigned*>(sc->small);
  const bool keep = cpw * NW <= CAP;
  int cnt = 0;
#pragma unroll 4
  for (int c = 0; c < nchunks; ++c) {
    const int i = lo + 32 * c + lane;
    const bool s = i < hi && key_selected(key_at(i), prefix, mask);
    const unsigned b = __ballot_sync(0xffffffffu, s);
    if (keep && lane == 0) bstore[wid * cpw + c] = b;
    cnt += __popc(b);
  }
  if (lane == 0) sc->scan[wid] = cnt;
  __syncthreads();
  int base = 0;
  for (int w = 0; w < wid; ++w) base += sc->scan[w];
#pragma unroll 4
  for (int c = 0; c < nchunks; ++c) {
    const int i = lo + 32 * c + lane;
    unsigned b;
    uint64_t k = 0;
    if (keep) {
      b = bstore[wid * cpw + c];
      if ((b >> lane) & 1u) k = key_at(i);
    } else {
      const bool s = i < hi && key_selected(k = (i < hi ? key_at(i) : 0ull), prefix, mask);
      b = __ballot_sync(0xffffffffu, s);
    }
    if ((b >> lane) & 1u) emit(base + __popc(b & ((1u << lane) - 1u)), i, k);
    base += __popc(b);
  }
  __syncthreads();
}

// Contiguous partition (distributed.hpp:53-57).
__host__ __device__ __forceinline__ void part_range(int64_t n, int64_t parts, int64_t i,
                                                    int64_t* first, int64_t* width) {
  const int64_t base = n / parts, extra = n % parts;
  *first = i * base + (i < extra ? i : extra);
  *width = base + (i < extra ? 1 : 0);
}

// ---------------------------------------------------------------------
// Per-bucket top-t survivors, written in ascending index order, padded
// with key 0. grid = (n_buckets, B), 256 threads; bucket width <= 4096.
// ---------------------------------------------------------------------
constexpr int kBucketMaxWidth = 4096;

__global__ void __launch_bounds__(256) bucket_topt_kernel(
    const float* __restrict__ scores, int64_t score_stride, int64_t n, int n_buckets, int t,
    uint64_t* __restrict__ surv) {
  hire_dev::griddep_wait();
  hire_dev::griddep_launch();
  extern __shared__ __align__(16) unsigned char smem_bucket[];
  uint64_t* s_keys = reinterpret_cast<uint64_t*>(smem_bucket);  // [width <= kBucketMaxWidth]
  __shared__ SelectScratch sc;
  const int bk = blockIdx.x, b = blockIdx.y;
  int64_t first, width;
  part_range(n, n_buckets, bk, &first, &width);
  const float* s = scores + b * score_stride + first;
  uint64_t* out = surv + (static_cast<int64_t>(b) * n_buckets + bk) * t;
  const int w = static_cast<int>(width);
  block_copy_tf(s_keys, w, [&](int i) { return make_key(s[i], static_cast<uint32_t>(first + i)); });
  __syncthreads();
  if (w <= t) {
    for (int i = threadIdx.x; i < t; i += 256) out[i] = i < w ? s_keys[i] : 0ull;
    return;
  }
  uint64_t prefix, mask;
  auto key_at = [&](int i) { return s_keys[i]; };
  block_radix_select<256>(key_at, w, t, &sc, &prefix, &mask);
  block_compact<256>(key_at, w, prefix, mask, &sc, [&](int pos, int, uint64_t k) { out[pos] = k; });
}

// ---------------------------------------------------------------------
// Candidate selection: one CTA (1024 threads) per query.
//   mode 0 DIRECT : pool = the whole score vector (n <= kDirectMax) in smem
//   mode 1 BUCKET : pool = survivors; exact_fix repairs overflowed buckets
// Writes the K selected indices in ascending order to cand[b][0..K).
// ---------------------------------------------------------------------
constexpr int kSelectThreads = 512;
constexpr int kDirectMax = 32768;        // 128 KB of fp32 scores
constexpr int kPoolKeys = 22528;         // 176 KB of u64 keys (+ ~37 KB static scratch)

__global__ void __launch_bounds__(kSelectThreads) select_candidates_kernel(
    int mode, const float* __restrict__ scores, int64_t score_stride, int64_t n,
    const uint64_t* __restrict__ surv, int n_buckets, int t, int K, int exact_fix,
    uint32_t* __restrict__ cand, int64_t cand_stride, int* __restrict__ status) {
  hire_dev::griddep_wait();
  hire_dev::griddep_launch();
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ SelectScratch sc;
  __shared__ int s_flag[2];
  const int b = blockIdx.x;
  const float* sc_row = scores + b * score_stride;
  uint32_t* out = cand + b * cand_stride;
  constexpr int NT = kSelectThreads;
  uint64_t prefix, mask;

  if (mode == 0) {
    float* s_val = reinterpret_cast<float*>(smem);
    const int nn = static_cast<int>(n);
    block_copy(s_val, sc_row, nn);
    __syncthreads();
    auto key_at = [&](int i) { return make_key(s_val[i], static_cast<uint32_t>(i)); };
    block_select_kth<NT>(key_at, nn, K, &sc, &prefix, &mask);
    block_compact<NT>(key_at, nn, prefix, mask, &sc,
                      [&](int pos, int i, uint64_t) { out[pos] = static_cast<uint32_t>(i); });
    return;
  }

  uint64_t* pool = reinterpret_cast<uint64_t*>(smem);
  const int n1 = n_buckets * t;
  const uint64_t* sv = surv + static_cast<int64_t>(b) * n1;
  block_copy(pool, sv, n1);
  __syncthreads();
  auto key1 = [&](int i) { return pool[i]; };
  block_select_kth<NT>(key1, n1, K, &sc, &prefix, &mask);

  if (exact_fix) {
    // overflow test per bucket; sizes of the repaired pool
    if (threadIdx.x == 0) s_flag[0] = 0;
    __syncthreads();
    const int per = (n_buckets + NT - 1) / NT;
    const int blo = min(n_buckets, static_cast<int>(threadIdx.x) * per);
    const int bhi = min(n_buckets, blo + per);
    int my_size = 0, my_over = 0;
    for (int bk = blo; bk < bhi; ++bk) {
      int64_t f, w;
      part_range(n, n_buckets, bk, &f, &w);
      if (w > t) {
        uint64_t mn = ~0ull;
        for (int j = 0; j < t; ++j) mn = min(mn, pool[bk * t + j]);
        if (key_selected(mn, prefix, mask)) { my_over = 1; my_size += static_cast<int>(w); continue; }
      }
      my_size += static_cast<int>(w < t ? w : t);
    }
    if (my_over) atomicOr(&s_flag[0], 1);
    int total;
    int off = block_exclusive_scan<NT>(my_size, sc.scan, &total);
    if (s_flag[0]) {
      if (n1 + total <= kPoolKeys) {
        uint64_t* pool2 = pool + n1;
        for (int bk = blo; bk < bhi; ++bk) {
          int64_t f, w;
          part_range(n, n_buckets, bk, &f, &w);
          bool over = false;
          if (w > t) {
            uint64_t mn = ~0ull;
            for (int j = 0; j < t; ++j) mn = min(mn, pool[bk * t + j]);
            over = key_selected(mn, prefix, mask);
          }
          if (over) {
            for (int64_t j = 0; j < w; ++j) pool2[off++] = make_key(sc_row[f + j], static_cast<uint32_t>(f + j));
          } else {
            const int m = static_cast<int>(w < t ? w : t);
            for (int j = 0; j < m; ++j) pool2[off++] = pool[bk * t + j];
          }
        }
        __syncthreads();
        auto key2 = [&](int i) { return pool2[i]; };
        block_select_kth<NT>(key2, total, K, &sc, &prefix, &mask);
        block_compact<NT>(key2, total, prefix, mask, &sc,
                          [&](int pos, int, uint64_t k) { out[pos] = key_index(k); });
      } else {
        // too many overflowed buckets for shared memory: exact select
        // straight over the score vector in global memory (slow, rare).
        if (threadIdx.x == 0 && status) atomicAdd(status, 1);
        const int nn = static_cast<int>(n);
        auto keyg = [&](int i) { return make_key(sc_row[i], static_cast<uint32_t>(i)); };
        block_select_kth<NT>(keyg, nn, K, &sc, &prefix, &mask);
        block_compact<NT>(keyg, nn, prefix, mask, &sc,
                          [&](int pos, int i, uint64_t) { out[pos] = static_cast<uint32_t>(i); });
      }
      return;
    }
  }
  block_compact<NT>(key1, n1, prefix, mask, &sc,
                    [&](int pos, int, uint64_t k) { out[pos] = key_index(k); });
}

// ---------------------------------------------------------------------
// Final selection over explicit (value, index) pairs or pre-built keys.
// One CTA (1024 threads) per query. Pool entry i of query b:
//   src_keys == nullptr : key(vals[b*vs + i], idx[b*is + i])
//   src_keys != nullptr : src_keys[(i / n_per) * part_stride + b * n_per + i % n_per]
//                         (the [D][B][n_per] layout an all-gather produces)
// out_mode 0 RANK  : K keys sorted by rank -> out_idx/out_val (+ probs)
//          1 INDEX : K selected in ascending-index (pool) order
//          2 KEYS  : K selected keys, padded to out_stride with 0 (send buffer)
// ---------------------------------------------------------------------
constexpr int kFinalMax = 16384;  // keys sorted in dynamic smem (128 KB)

__global__ void __launch_bounds__(kSelectThreads) final_select_kernel(
    const float* __restrict__ vals, int64_t vs, const uint32_t* __restrict__ idx, int64_t is,
    const uint64_t* __restrict__ src_keys, int n_per, int64_t part_stride, int n, int K,
    int out_mode, uint32_t* __restrict__ out_idx, float* __restrict__ out_val,
    float* __restrict__ out_prob, uint64_t* __restrict__ out_keys, int64_t out_stride) {
  hire_dev::griddep_wait();
  hire_dev::griddep_launch();
  constexpr int NT = kSelectThreads;
  __shared__ SelectScratch sc;
  extern __shared__ __align__(16) unsigned char smem_final[];
  uint64_t* s_sel = reinterpret_cast<uint64_t*>(smem_final);
  __shared__ double s_red[NT / 32];
  const int b = blockIdx.x;
  auto key_at = [&](int i) -> uint64_t {
    if (src_keys) return src_keys[static_cast<int64_t>(i / n_per) * part_stride + static_cast<int64_t>(b) * n_per + i % n_per];
    return make_key(vals[b * vs + i], idx[b * is + i]);
  };
  uint64_t prefix, mask;
  block_select_kth<NT>(key_at, n, K, &sc, &prefix, &mask);
  if (out_mode == 1) {
    block_compact<NT>(key_at, n, prefix, mask, &sc, [&](int pos, int, uint64_t k) {
      out_idx[b * out_stride + pos] = key_index(k);
      out_val[b * out_stride + pos] = key_value(k);
    });
    return;
  }
  if (out_mode == 2) {
    block_compact<NT>(key_at, n, prefix, mask, &sc,
                      [&](int pos, int, uint64_t k) { out_keys[b * out_stride + pos] = k; });
    for (int i = K + threadIdx.x; i < out_stride; i += NT) out_keys[b * out_stride + i] = 0ull;
    return;
  }
  int P = 1;
  while (P < K) P <<= 1;
  for (int i = threadIdx.x; i < P; i += NT) s_sel[i] = 0ull;
  __syncthreads();
  block_compact<NT>(key_at, n, prefix, mask, &sc, [&](int pos, int, uint64_t k) { s_sel[pos] = k; });
  __syncthreads();
  // bitonic sort, descending (one warp with __syncwarp when P <= 64)
  if (P <= 64) {
    if (threadIdx.x < 32) {
      for (int size = 2; size <= P; size <<= 1)
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
          const int i = threadIdx.x;
          if (i < P / 2) {
            const int lo = 2 * i - (i & (stride - 1));
            const int hi = lo + stride;
            const bool desc = (lo & size) == 0;
            const uint64_t a = s_sel[lo], c = s_sel[hi];
            if ((a < c) == desc) { s_sel[lo] = c; s_sel[hi] = a; }
          }
          __syncwarp();
        }
    }
    __syncthreads();
  } else {
    for (int size = 2; size <= P; size <<= 1) {
      for (int stride = size >> 1; stride > 0; stride >>= 1) {
        for (int i = threadIdx.x; i < P / 2; i += NT) {
          const int lo = 2 * i - (i & (stride - 1));
          const int hi = lo + stride;
          const bool desc = (lo & size) == 0;
          const uint64_t a = s_sel[lo], c = s_sel[hi];
          if ((a < c) == desc) { s_sel[lo] = c; s_sel[hi] = a; }
        }
        __syncthreads();
      }
    }
  }
  for (int i = threadIdx.x; i < K; i += NT) {
    out_idx[b * out_stride + i] = key_index(s_sel[i]);
    out_val[b * out_stride + i] = key_value(s_sel[i]);
  }
  if (out_prob) {
    // hire.hpp:135-142: p_i = exp(double(v_i) - v_max) rounded to float,
    // renormalised by the double sum.
    const double vmax = static_cast<double>(key_value(s_sel[0]));
    double local = 0.0;
    float pf = 0.0f;
    const int i = threadIdx.x;
    if (i < K) {
      const double p = exp(static_cast<double>(key_value(s_sel[i])) - vmax);
      pf = static_cast<float>(p);
      local = p;
    }
    for (int j = i + NT; j < K; j += NT) local += exp(static_cast<double>(key_value(s_sel[j])) - vmax);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) local += __shfl_xor_sync(0xffffffffu, local, o);
    if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = local;
    __syncthreads();
    if (threadIdx.x == 0) {
      double s = 0.0;
      for (int w = 0; w < NT / 32; ++w) s += s_red[w];
      s_red[0] = s;
    }
    __syncthreads();
    const double sum = s_red[0];
    if (i < K) out_prob[b * out_stride + i] = static_cast<float>(static_cast<double>(pf) / sum);
    for (int j = i + NT; j < K; j += NT) {
      const float pj = static_cast<float>(exp(static_cast<double>(key_value(s_sel[j])) - vmax));
      out_prob[b * out_stride + j] = static_cast<float>(static_cast<double>(pj) / sum);
    }
  }
}

}  // namespace hire_dev
