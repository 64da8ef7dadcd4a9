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

struct SelectScratch {
  unsigned int hist[256];
  int scan[64];
  int sel[4];
};

// Finds (prefix, mask) such that exactly K of the n keys satisfy
// (key & mask) >= prefix — i.e. the K largest. Keys must be unique among
// non-padding entries (indices are unique); 1 <= K <= n.
template <int NT, class KeyAt>
__device__ void block_radix_select(KeyAt key_at, int n, int K, SelectScratch* sc,
                                   uint64_t* out_prefix, uint64_t* out_mask) {
  static_assert(NT >= 256, "digit scan uses 256 threads");
  uint64_t prefix = 0, mask = 0;
  int krem = K;
  const int lane = threadIdx.x & 31;
  const int n_round = (n + NT - 1) / NT * NT;
  for (int shift = 56; shift >= 0; shift -= 8) {
    if (threadIdx.x < 256) sc->hist[threadIdx.x] = 0;
    __syncthreads();
    for (int i = threadIdx.x; i < n_round; i += NT) {
      int dg = 0x1000;
      if (i < n) {
        const uint64_t k = key_at(i);
        if ((k & mask) == prefix) dg = static_cast<int>((k >> shift) & 0xFF);
      }
      const unsigned same = __match_any_sync(0xffffffffu, dg);
      if (dg != 0x1000 && lane == __ffs(same) - 1) atomicAdd(&sc->hist[dg], __popc(same));
    }
    __syncthreads();
    if (threadIdx.x < 256) {
      // descending digit order: thread t looks at digit 255 - t
      const int v = sc->hist[255 - threadIdx.x];
      int inc = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int nn = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += nn;
      }
      if (lane == 31) sc->scan[threadIdx.x >> 5] = inc;
      asm volatile("bar.sync 1, 256;");
      int before = 0;
      for (int w = 0; w < static_cast<int>(threadIdx.x >> 5); ++w) before += sc->scan[w];
      inc += before;
      if (inc >= krem && inc - v < krem) {
        sc->sel[0] = 255 - threadIdx.x;
        sc->sel[1] = krem - (inc - v);
        sc->sel[2] = v;
      }
    }
    __syncthreads();
    const int dg = sc->sel[0];
    krem = sc->sel[1];
    const int cnt = sc->sel[2];
    prefix |= static_cast<uint64_t>(dg) << shift;
    mask |= static_cast<uint64_t>(0xFF) << shift;
    __syncthreads();
    if (cnt == krem) break;  // every key of this digit is in the top K
  }
  *out_prefix = prefix;
  *out_mask = mask;
}

__device__ __forceinline__ bool key_selected(uint64_t k, uint64_t prefix, uint64_t mask) {
  return (k & mask) >= prefix && k != 0;
}

// Order-preserving compaction of the selected keys: thread t owns the
// contiguous segment [t*seg, (t+1)*seg). emit(pos, i, key).
template <int NT, class KeyAt, class Emit>
__device__ void block_compact(KeyAt key_at, int n, uint64_t prefix, uint64_t mask,
                              SelectScratch* sc, Emit emit) {
  const int seg = (n + NT - 1) / NT;
  const int lo = min(n, static_cast<int>(threadIdx.x) * seg), hi = min(n, lo + seg);
  int cnt = 0;
  for (int i = lo; i < hi; ++i) cnt += key_selected(key_at(i), prefix, mask);
  int total;
  int pos = block_exclusive_scan<NT>(cnt, sc->scan, &total);
  for (int i = lo; i < hi; ++i) {
    const uint64_t k = key_at(i);
    if (key_selected(k, prefix, mask)) emit(pos++, i, k);
  }
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
  __shared__ uint64_t s_keys[kBucketMaxWidth];
  __shared__ SelectScratch sc;
  const int bk = blockIdx.x, b = blockIdx.y;
  int64_t first, width;
  part_range(n, n_buckets, bk, &first, &width);
  const float* s = scores + b * score_stride + first;
  uint64_t* out = surv + (static_cast<int64_t>(b) * n_buckets + bk) * t;
  const int w = static_cast<int>(width);
  for (int i = threadIdx.x; i < w; i += 256) s_keys[i] = make_key(s[i], static_cast<uint32_t>(first + i));
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
constexpr int kSelectThreads = 1024;
constexpr int kDirectMax = 32768;        // 128 KB of fp32 scores
constexpr int kPoolKeys = 24576;         // 192 KB of u64 keys

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
    for (int i = threadIdx.x; i < nn; i += NT) s_val[i] = sc_row[i];
    __syncthreads();
    auto key_at = [&](int i) { return make_key(s_val[i], static_cast<uint32_t>(i)); };
    block_radix_select<NT>(key_at, nn, K, &sc, &prefix, &mask);
    block_compact<NT>(key_at, nn, prefix, mask, &sc,
                      [&](int pos, int i, uint64_t) { out[pos] = static_cast<uint32_t>(i); });
    return;
  }

  uint64_t* pool = reinterpret_cast<uint64_t*>(smem);
  const int n1 = n_buckets * t;
  const uint64_t* sv = surv + static_cast<int64_t>(b) * n1;
  for (int i = threadIdx.x; i < n1; i += NT) pool[i] = sv[i];
  __syncthreads();
  auto key1 = [&](int i) { return pool[i]; };
  block_radix_select<NT>(key1, n1, K, &sc, &prefix, &mask);

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
        block_radix_select<NT>(key2, total, K, &sc, &prefix, &mask);
        block_compact<NT>(key2, total, prefix, mask, &sc,
                          [&](int pos, int, uint64_t k) { out[pos] = key_index(k); });
      } else {
        // too many overflowed buckets for shared memory: exact select
        // straight over the score vector in global memory (slow, rare).
        if (threadIdx.x == 0 && status) atomicAdd(status, 1);
        const int nn = static_cast<int>(n);
        auto keyg = [&](int i) { return make_key(sc_row[i], static_cast<uint32_t>(i)); };
        block_radix_select<NT>(keyg, nn, K, &sc, &prefix, &mask);
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
  block_radix_select<NT>(key_at, n, K, &sc, &prefix, &mask);
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
  // bitonic sort, descending
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
