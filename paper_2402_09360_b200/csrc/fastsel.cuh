// fastsel.cuh — block-wide exact order statistic over 64-bit rank keys by
// shared-memory histograms (sm_100a).
//
// Returns the K-th largest non-zero key held by the CTA (keys in registers,
// KPT per thread; key 0 is padding). Rank keys are unique (common.cuh
// make_key), so "the K-th largest" is exact and the caller's emit of keys
// >= T reproduces topk_select (linalg.hpp:157-176) bit for bit.
//
// Each pass bins the projected word (phase 0: the value word key >> 32;
// phase 1: the index word, among keys sharing one value word) over the
// current range [lo, hi] into 2048 equal bins with shared-memory atomics,
// finds the bin holding rank r with one block scan, and narrows to it. Once
// the bin holds <= 1024 keys they are compacted to shared memory and the
// loop continues on those; <= 32 keys are ranked directly by one warp. For
// the score distributions of the HiRE path one pass usually leaves a handful
// of keys: ~10 barriers in total, against one barrier per 16-way split in
// block_range_select (select2.cuh).
#pragma once
#include "common.cuh"

namespace hire_dev {

constexpr int kFsBins = 2048;
constexpr int kFsCand = 1024;

struct FastSelScratch {
  unsigned hist[kFsBins];
  uint64_t cand[2][kFsCand];
  unsigned mn[32], mx[32], cn[32];
  int scan[40];
  unsigned bstar, m, ncand;
  long long above;
  uint64_t result;
};

template <int NT>
__device__ __forceinline__ int fs_scan_excl(int v, int* s_tmp, int* total) {
  constexpr int NW = NT / 32;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int n = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += n;
  }
  if (lane == 31) s_tmp[w] = inc;
  __syncthreads();
  int before = 0, tot = 0;
#pragma unroll
  for (int i = 0; i < NW; ++i) {
    const int x = s_tmp[i];
    before += i < w ? x : 0;
    tot += x;
  }
  *total = tot;
  return before + inc - v;
}

// K-th largest (1 <= K <= number of non-zero keys) of the CTA's keys.
// Block-uniform result. Every thread of the CTA (NT of them) must call it.
// sf != nullptr: the keys are make_key(sf[i], i) for i < nf, read from
// shared memory (rows too long for registers); keys[] is then unused.
template <int NT, int KPT>
__device__ __forceinline__ uint64_t block_fast_select(const uint64_t (&keys)[KPT], long long K, FastSelScratch* s,
                                                      unsigned long long* tr = nullptr, const float* sf = nullptr,
                                                      unsigned nf = 0) {
  int trn = 0;  // debug timeline: tr[0..7] = %globaltimer after each phase (thread 0)
  auto stamp = [&]() {
    if (tr && threadIdx.x == 0 && trn < 8) tr[trn] = gtimer();
    ++trn;
  };
  static_assert(kFsBins % NT == 0 && NT >= 64 && NT <= 1024, "bins per thread");
  constexpr int BPT = kFsBins / NT;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  int phase = 0;
  unsigned vstar = 0;
  int src = -1;         // -1: registers; 0/1: s->cand[src][0..ncand)
  unsigned ncand = 0;
  long long r = K;

  auto project = [&](uint64_t k, unsigned* x) -> bool {
    const unsigned hi32 = static_cast<unsigned>(k >> 32);
    *x = phase == 0 ? hi32 : static_cast<unsigned>(k);
    return k != 0 && (phase == 0 || hi32 == vstar);
  };
  if (sf) src = -2;
  auto each = [&](auto f) {
    if (src == -2) {  // shared-memory scores, uniform trip count
      for (unsigned i0 = 0; i0 < nf; i0 += NT) {
        const unsigned i = i0 + tid;
        f(i < nf ? make_key(sf[i], i) : 0ull);
      }
    } else if (src < 0) {
#pragma unroll
      for (int j = 0; j < KPT; ++j) f(keys[j]);
    } else {  // uniform trip count: f may use warp collectives
      for (unsigned i0 = 0; i0 < ncand; i0 += NT) {
        const unsigned i = i0 + tid;
        f(i < ncand ? s->cand[src][i] : 0ull);
      }
    }
  };
  auto minmax = [&](unsigned* lo, unsigned* hi, long long* cnt) {
    unsigned a = 0xFFFFFFFFu, b = 0u, n = 0u;
    each([&](uint64_t k) {
      unsigned x;
      if (project(k, &x)) {
        a = min(a, x);
        b = max(b, x);
        ++n;
      }
    });
    a = __reduce_min_sync(0xffffffffu, a);
    b = __reduce_max_sync(0xffffffffu, b);
    n = __reduce_add_sync(0xffffffffu, n);
    if (lane == 0) {
      s->mn[wid] = a;
      s->mx[wid] = b;
      s->cn[wid] = n;
    }
    __syncthreads();
    a = lane < NT / 32 ? s->mn[lane] : 0xFFFFFFFFu;
    b = lane < NT / 32 ? s->mx[lane] : 0u;
    n = lane < NT / 32 ? s->cn[lane] : 0u;
    *lo = __reduce_min_sync(0xffffffffu, a);
    *hi = __reduce_max_sync(0xffffffffu, b);
    *cnt = __reduce_add_sync(0xffffffffu, n);
  };

  unsigned lo, hi;
  long long total;  // keys in play within [lo, hi]
  minmax(&lo, &hi, &total);
  stamp();
  // First pass on a value-linear scale: the value word is logarithmic in
  // |v| (exponent bits), so equal ord-space bins over a wide range put most
  // keys of a bell-shaped score row into a few bins (shared-atomic
  // contention). (v - vmin) * scale is monotone in v, so each bin is still a
  // contiguous key range and the pass narrows [lo, hi] exactly.
  {
    const float fmin = value_of_ord(lo), fmax = value_of_ord(hi);
    if (lo != hi && isfinite(fmin) && isfinite(fmax) && fmax > fmin && total > 32) {
      const float scale = static_cast<float>(kFsBins - 1) / (fmax - fmin);
      auto vbin = [&](uint64_t k) -> unsigned {
        const float b = (key_value(k) - fmin) * scale;
        return b >= static_cast<float>(kFsBins - 1) ? kFsBins - 1u : (b > 0.0f ? static_cast<unsigned>(b) : 0u);
      };
      for (int i = tid; i < kFsBins; i += NT) s->hist[i] = 0u;
      __syncthreads();
      each([&](uint64_t k) {
        if (k != 0) {
          const unsigned bin = vbin(k);
          if (bin) atomicAdd(&s->hist[bin], 1u);
        }
      });
      __syncthreads();
      unsigned c[BPT];
      int local = 0;
#pragma unroll
      for (int j = 0; j < BPT; ++j) {
        c[j] = s->hist[kFsBins - 1 - (tid * BPT + j)];
        local += static_cast<int>(c[j]);
      }
      int tot;
      const long long ex = fs_scan_excl<NT>(local, s->scan, &tot);
      if (tid == NT - 1) {
        c[BPT - 1] = static_cast<unsigned>(total - tot);
        local += static_cast<int>(c[BPT - 1]);
      }
      if (ex < r && ex + local >= r) {
        long long cum = ex;
#pragma unroll
        for (int j = 0; j < BPT; ++j) {
          if (cum < r && cum + c[j] >= r) {
            s->bstar = static_cast<unsigned>(kFsBins - 1 - (tid * BPT + j));
            s->above = cum;
            s->m = c[j];
            s->ncand = 0u;
          }
          cum += c[j];
        }
      }
      __syncthreads();
      const unsigned bstar = s->bstar;
      r -= s->above;
      if (s->m <= 32u) {
        // the usual case for the HiRE score rows: the bin holds a handful of
        // keys — gather them by bin number and rank them directly (no range
        // pass, no separate compaction: two barriers and a pass fewer)
        each([&](uint64_t k) {
          const bool in = k != 0 && vbin(k) == bstar;
          const unsigned bal = __ballot_sync(0xffffffffu, in);
          if (bal) {
            const int leader = __ffs(bal) - 1;
            unsigned base = 0;
            if (lane == leader) base = atomicAdd(&s->ncand, static_cast<unsigned>(__popc(bal)));
            base = __shfl_sync(0xffffffffu, base, leader);
            if (in) s->cand[0][base + __popc(bal & ((1u << lane) - 1u))] = k;
          }
        });
        __syncthreads();
        stamp();
        const unsigned m = s->ncand;
        if (wid == 0) {
          const uint64_t mine = lane < static_cast<int>(m) ? s->cand[0][lane] : 0ull;
          int gt = 0;
          for (unsigned j = 0; j < m; ++j) gt += s->cand[0][j] > mine ? 1 : 0;
          if (lane < static_cast<int>(m) && gt == r - 1) s->result = mine;
        }
        __syncthreads();
        return s->result;
      }
      // the chosen bin's keys are one contiguous ord range: find it
      unsigned a = 0xFFFFFFFFu, b = 0u, nn = 0u;
      each([&](uint64_t k) {
        if (k != 0 && vbin(k) == bstar) {
          const unsigned x = static_cast<unsigned>(k >> 32);
          a = min(a, x);
          b = max(b, x);
          ++nn;
        }
      });
      a = __reduce_min_sync(0xffffffffu, a);
      b = __reduce_max_sync(0xffffffffu, b);
      nn = __reduce_add_sync(0xffffffffu, nn);
      if (lane == 0) {
        s->mn[wid] = a;
        s->mx[wid] = b;
        s->cn[wid] = nn;
      }
      __syncthreads();
      a = lane < NT / 32 ? s->mn[lane] : 0xFFFFFFFFu;
      b = lane < NT / 32 ? s->mx[lane] : 0u;
      nn = lane < NT / 32 ? s->cn[lane] : 0u;
      lo = __reduce_min_sync(0xffffffffu, a);
      hi = __reduce_max_sync(0xffffffffu, b);
      total = __reduce_add_sync(0xffffffffu, nn);
      __syncthreads();  // mn/mx/hist reuse
      stamp();
    }
  }
  // compaction of the in-play keys within [lo, hi] into the other buffer
  auto compact = [&]() {
    const int dst = src == 0 ? 1 : 0;
    if (tid == 0) s->ncand = 0u;
    __syncthreads();
    each([&](uint64_t k) {
      unsigned x;
      const bool in = project(k, &x) && x - lo <= hi - lo;
      const unsigned bal = __ballot_sync(0xffffffffu, in);
      if (bal) {
        const int leader = __ffs(bal) - 1;
        unsigned base = 0;
        if (lane == leader) base = atomicAdd(&s->ncand, static_cast<unsigned>(__popc(bal)));
        base = __shfl_sync(0xffffffffu, base, leader);
        if (in) s->cand[dst][base + __popc(bal & ((1u << lane) - 1u))] = k;
      }
    });
    __syncthreads();
    ncand = s->ncand;
    src = dst;
  };
  for (;;) {
    if (total <= 32) {  // rank the survivors directly (keys are unique)
      compact();
      stamp();
      const unsigned m = ncand;
      if (wid == 0) {
        const uint64_t mine = lane < static_cast<int>(m) ? s->cand[src][lane] : 0ull;
        int gt = 0;
        for (unsigned j = 0; j < m; ++j) gt += s->cand[src][j] > mine ? 1 : 0;
        if (lane < static_cast<int>(m) && gt == r - 1) s->result = mine;
      }
      __syncthreads();
      return s->result;
    }
    if (lo == hi && phase == 0) {
      // > 32 keys share one value word: rank on the index word among them
      phase = 1;
      vstar = lo;
      __syncthreads();  // mn/mx reuse
      minmax(&lo, &hi, &total);
      continue;
    }
    const unsigned range = hi - lo;
    const int sh = range < static_cast<unsigned>(kFsBins) ? 0 : (32 - __clz(range)) - 11;
    for (int i = tid; i < kFsBins; i += NT) s->hist[i] = 0u;
    __syncthreads();
    // bin 0 (the range minimum: ReLU zeros, the padding side of a tie
    // class) is not counted with atomics — its count is the in-range total
    // minus the other bins, so heavy ties at the bottom cost no contention
    each([&](uint64_t k) {
      unsigned x;
      if (project(k, &x) && x - lo <= range) {
        const unsigned bin = (x - lo) >> sh;
        if (bin) atomicAdd(&s->hist[bin], 1u);
      }
    });
    __syncthreads();
    // thread t owns bins top-down: kFsBins-1 - (t*BPT + j)
    unsigned c[BPT];
    int local = 0;
#pragma unroll
    for (int j = 0; j < BPT; ++j) {
      c[j] = s->hist[kFsBins - 1 - (tid * BPT + j)];
      local += static_cast<int>(c[j]);
    }
    int tot;
    const long long ex = fs_scan_excl<NT>(local, s->scan, &tot);
    if (tid == NT - 1) {  // owns bin 0
      c[BPT - 1] = static_cast<unsigned>(total - tot);
      local += static_cast<int>(c[BPT - 1]);
    }
    if (ex < r && ex + local >= r) {
      long long cum = ex;
#pragma unroll
      for (int j = 0; j < BPT; ++j) {
        if (cum < r && cum + c[j] >= r) {
          s->bstar = static_cast<unsigned>(kFsBins - 1 - (tid * BPT + j));
          s->above = cum;
          s->m = c[j];
        }
        cum += c[j];
      }
    }
    __syncthreads();
    const unsigned bstar = s->bstar, m = s->m;
    r -= s->above;
    total = m;
    const unsigned nlo = lo + (bstar << sh);
    const unsigned span = (1u << sh) - 1u;  // sh <= 21
    lo = nlo;
    hi = (hi - nlo > span) ? nlo + span : hi;
    __syncthreads();  // hist / bstar reuse
    if (total > 32 && total <= kFsCand && (src < 0 || total < ncand)) compact();
    stamp();
  }
}

}  // namespace hire_dev
