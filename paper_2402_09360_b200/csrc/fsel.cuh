// fsel.cuh — candidate selection fused into the proxy GEMV (sm_100a).
//
// Same contract as topk_select(k') (linalg.hpp:157-176) followed by the
// ascending sort of hire.hpp:65-67: the k' largest rank keys, returned as
// indices in ascending order. The grid-wide selector of select2.cuh needs
// four launches after the proxy kernel (pivot, window, window-select, emit),
// each re-reading the score row. Here the proxy kernel filters its scores
// while they are still in registers, and one small kernel finishes:
//
//   proxy kernel (q4_score_mma_sel): the unfused kernel's strided schedule
//   (round rd, CTA c, warp w scores row-block rd*U + c*RPC + w, U = G*RPC)
//   with no barrier in the streaming loop. Each row-block's keys >= lo form
//   its own list (list id = row-block id, so lists in id order are in index
//   order; 16 slots: a list can never overflow).
//     A. every samp_step-th CTA publishes the keys of its round-0 row-blocks
//        (scored anyway: no extra bytes; stratified over the index range)
//        straight into the sample slots (key 0 = not yet written).
//     B. nbrk extra bracket CTAs (no rows of their own) poll the sample,
//        take the sample value word of rank r_lo (~ k'/n * S + 4 sigma) as
//        the query's lower bound lo and publish it (lo[b] != 0 = ready).
//     C. each warp issues a load of lo[] at the start of every round and
//        looks at it after the row-block (the L2 round trip overlaps the
//        MMA stream); once all bounds are known it filters each row-block
//        from registers; row-blocks finished before that (the backlog) are
//        filtered from L2 once, when the bounds arrive.
//   sel_fin_kernel, one CTA per query: prefix sums of the list counts,
//     listed keys staged in shared memory in list order, T = the k'-th
//     largest (block_fast_select), emit keys >= T in list order; clears the
//     sample slots and lo[] (zero at rest, so a CUDA graph replays the pair
//     without re-initialisation).
//
// Exactness: every key >= lo is listed, so when at least k' keys are listed
// T is the true k'-th key and the emitted set is exactly topk_select's. A
// bracket miss (fewer than k' listed), too many listed keys, or a bound that
// never arrived (spin timeout) is detected in sel_fin_kernel, which then
// selects over the whole score row (correct, slow, counted in `status`).
//
// Co-residency: streaming CTAs wait (only at the end, with a timeout) on the
// bracket CTAs, which wait on sampling CTAs that never wait; the host sizes
// the grid to one wave (every CTA resident at once).
#pragma once
#include "common.cuh"
#include "select2.cuh"
#include "fastsel.cuh"
#include "exact.cuh"

namespace hire_dev {

constexpr int kFselSampleMax = 4096;           // sampled keys per query
constexpr int kFinThreads = 1024;
constexpr int kFinKpt = 8;
constexpr int kFinCap = kFinThreads * kFinKpt; // listed keys handled on chip
constexpr int kFinMaxRows = 1 << 19;           // emit bitmap: rows per query
constexpr int kFselCtr = 16;                   // claim counters (128 B apart)
constexpr int kFselDynLog = 16;                // claimed row-blocks remembered per warp before the bounds
constexpr int kFselMaxB = 64;
constexpr unsigned long long kFselTimeoutNs = 20000000ull;  // 20 ms

struct FuseSel {
  uint32_t n;        // rows per query
  uint32_t K;        // k'
  int g_stream;      // streaming CTAs; CTAs beyond are bracket CTAs
  int nbrk;          // bracket CTAs (query b handled by bracket CTA b % nbrk)
  int samp_step;     // every samp_step-th streaming CTA samples its round-0 row-blocks
  int n_samp;        // sampled keys per query (<= kFselSampleMax)
  int r_lo;          // sample rank of the lower bound
  uint64_t* samp;    // [B][kFselSampleMax], zero at rest
  unsigned long long* lo;  // [B], zero at rest; 0 = not yet known
  unsigned* cnt;     // [B] listed keys (bit 31: a bound never arrived), zero at rest
  unsigned* ctr;     // [kFselCtr * 32] row-block claim counters (dynamic tail), zero at rest
  int n_static;      // rounds scheduled statically (>= 1; the rest is claimed, KS == 1)
  const float* xf;   // non-null: quantise x here (prep_x_int8_kernel folded in; small B)
  uint64_t* lists;   // [B][kFinCap] listed keys (unordered)
  // stream path (sel_stream_kernel): lo[b] = the query's bound tau (the
  // finisher accepts T only if T >= tau), cnt[b] as above
  int stream;
};

// Sample keys rebuilt from value words staged in shared memory: slot j of
// value word v becomes (v << 32) | ~j (unique, value order preserved).
struct SmemWordKeys {
  static constexpr int kFixed = 0;
  const unsigned* w;
  uint32_t n;
  template <class F>
  __device__ __forceinline__ void each(F f) const {
    int j = 0;
    for (uint32_t i = threadIdx.x; i < n; i += 256) f((static_cast<uint64_t>(w[i]) << 32) | (0xFFFFFFFFu - i), j++);
  }
};

__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// ---------------------------------------------------------------------
// K1 (int4 x int8 on the tensor cores, see q4_score_mma) with the fused
// pre-selection.
// ---------------------------------------------------------------------
#ifndef HIRE_FSEL_MINB
#define HIRE_FSEL_MINB 3
#endif
template <int NT, int KS>
__global__ void __launch_bounds__(256, HIRE_FSEL_MINB) q4_score_mma_sel(
    const uint4* __restrict__ wmma, int64_t rows, int d, const float* __restrict__ scales,
    const int8_t* __restrict__ xq, const float* __restrict__ sx, const int* __restrict__ sumxq,
    int B, int phi, float* __restrict__ scores, int64_t score_stride, FuseSel fs) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ RangeScratch rs;
  __shared__ unsigned s_vw[kFselSampleMax];
  constexpr int RPC = 8 / KS;  // row-blocks per CTA per round
  const int xs = d + 16;
  int8_t* s_x = reinterpret_cast<int8_t*>(smem);
  int* s_acc = reinterpret_cast<int*>(smem + static_cast<size_t>(NT) * 8 * xs);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int nkb = d / 64;
  const int64_t n_rb = (rows + 15) / 16;
  const int rb_local = wid / KS, ks = wid % KS;
  const int kb0 = ks * nkb / KS, kb1 = (ks + 1) * nkb / KS;
  // the bracket CTAs take the lowest block ids (scheduled first even when a
  // predecessor kernel still holds a few slots); streaming CTA c = id - nbrk
  const int G = fs.g_stream, c = static_cast<int>(blockIdx.x) - fs.nbrk;
  const int64_t U = static_cast<int64_t>(G) * RPC;
  const int rounds = static_cast<int>((n_rb + U - 1) / U);

  constexpr int UL = 4;
  uint4 a[UL];
  // prologue independent of the producer kernel: first weight loads
  if (c >= 0) {
    const int64_t rb = static_cast<int64_t>(c) * RPC + rb_local;
    if (rb < n_rb) {
#pragma unroll
      for (int u = 0; u < UL; ++u)
        if (kb0 + u < kb1) a[u] = ldg_stream(wmma + ((rb * nkb + kb0 + u) * 32 + lane));
    }
  }
  griddep_wait();
  griddep_launch();
  KTrace kt_(kKtProxy);

  // ---- B: bracket CTAs ----
  if (c < 0) {
    constexpr int KPT = kFselSampleMax / 256;
    const int S = fs.n_samp;
    for (int b = static_cast<int>(blockIdx.x); b < B; b += fs.nbrk) {
      const unsigned long long* sp = reinterpret_cast<const unsigned long long*>(fs.samp) +
                                     static_cast<int64_t>(b) * kFselSampleMax;
      const unsigned long long t0 = gtimer();
      bool ok = true;
      for (;;) {  // poll the sample slots (0 = not yet written); stage value words
        int missing = 0;
#pragma unroll
        for (int j = 0; j < KPT; ++j) {
          const int i = threadIdx.x + j * 256;
          const unsigned long long k = ld_relaxed_u64(sp + i);
          missing |= (i < S && k == 0ull) ? 1 : 0;
          s_vw[i] = (i < S && k > 1ull) ? static_cast<unsigned>(k >> 32) : 0u;  // 1 = padding row
        }
        if (!__syncthreads_or(missing)) break;
        if (gtimer() - t0 > kFselTimeoutNs) {
          ok = false;
          break;
        }
        __nanosleep(256);
      }
      if (g_ktrace && threadIdx.x == 0) atomicMax(&g_ktrace[52], gtimer());
      uint64_t lo = 1ull;  // failure: list everything -> overflow -> exact fallback
      if (ok) {
        // rank r_lo value word of the sample (zero words = padding, skipped)
        SmemWordKeys src{s_vw, static_cast<uint32_t>(S)};
        const uint64_t kr = block_range_select<256>(src, S, fs.r_lo, &rs);
        lo = (kr >> 32) << 32;  // every key with that value word or above
      }
      if (threadIdx.x == 0) {
        atomicExch(fs.lo + b, static_cast<unsigned long long>(lo ? lo : 1ull));
        if (g_ktrace) atomicMax(&g_ktrace[53], gtimer());
      }
      __syncthreads();  // s_vw / rs reuse
    }
    return;
  }

  __shared__ float s_sx[8];
  __shared__ int s_sumq[8];
  __shared__ float s_red[8];
  __shared__ int s_redi[8];
  if (fs.xf) {
    // prep_x_int8_kernel folded in (B <= 2): every CTA quantises x itself,
    // with the same arithmetic (bit-identical sx, codes and code sums)
    for (int n = 0; n < NT * 8; ++n) {
      if (n >= B) {
        for (int i = threadIdx.x; i < d / 16; i += blockDim.x) *reinterpret_cast<int4*>(s_x + n * xs + i * 16) = make_int4(0, 0, 0, 0);
        continue;
      }
      const float* xb = fs.xf + static_cast<int64_t>(n) * d;
      float m = 0.0f;
      for (int i = threadIdx.x; i < d; i += blockDim.x) m = fmaxf(m, fabsf(__ldg(xb + i)));
      m = warp_max_f32(m);
      if (lane == 0) s_red[wid] = m;
      __syncthreads();
      float mx = 0.0f;
#pragma unroll
      for (int w = 0; w < 8; ++w) mx = fmaxf(mx, s_red[w]);
      const float sxv = mx > 0.0f ? __fdiv_rn(mx, 127.0f) : 1.0f;
      int sum = 0;
      for (int i = threadIdx.x; i < d; i += blockDim.x) {
        const int qv = rhaz_clamp(__fdiv_rn(__ldg(xb + i), sxv), 127);
        sum += qv;
        s_x[n * xs + i] = static_cast<int8_t>(qv);
      }
      sum = warp_sum_i32(sum);
      if (lane == 0) s_redi[wid] = sum;
      __syncthreads();
      if (threadIdx.x == 0) {
        int t2 = 0;
        for (int w = 0; w < 8; ++w) t2 += s_redi[w];
        s_sumq[n] = t2;
        s_sx[n] = sxv;
      }
      __syncthreads();
    }
  } else {
    for (int i = threadIdx.x; i < NT * 8 * (d / 16); i += blockDim.x) {
      const int n = i / (d / 16), cc = i % (d / 16);
      int4 v = make_int4(0, 0, 0, 0);
      if (n < B) v = *reinterpret_cast<const int4*>(xq + static_cast<int64_t>(n) * d + cc * 16);
      *reinterpret_cast<int4*>(s_x + n * xs + cc * 16) = v;
    }
    if (threadIdx.x < B && threadIdx.x < 8) {
      s_sx[threadIdx.x] = sx[threadIdx.x];
      s_sumq[threadIdx.x] = sumxq[threadIdx.x];
    }
  }
  __syncthreads();

  // one row-block's integer dot products (k range [kb0, kb1) of this warp),
  // exact int32; w[] holds the first UL loads on entry
  auto rowblock = [&](int64_t rb, uint4 (&w)[UL], int (&acc)[NT][4]) {
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) acc[nt][0] = acc[nt][1] = acc[nt][2] = acc[nt][3] = 0;
    for (int kb = kb0; kb < kb1; kb += UL) {
      uint4 nxt[UL];
#pragma unroll
      for (int u = 0; u < UL; ++u)
        if (kb + UL + u < kb1) nxt[u] = ldg_stream(wmma + ((rb * nkb + kb + UL + u) * 32 + lane));
#pragma unroll
      for (int u = 0; u < UL; ++u) {
        if (kb + u >= kb1) break;
        const uint32_t w4[4] = {w[u].x, w[u].y, w[u].z, w[u].w};
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const uint32_t u0 = w4[2 * j] ^ 0x88888888u, u1 = w4[2 * j + 1] ^ 0x88888888u;
          const uint32_t a0 = u0 & 0x0F0F0F0Fu, a1 = (u0 >> 4) & 0x0F0F0F0Fu;
          const uint32_t a2 = u1 & 0x0F0F0F0Fu, a3 = (u1 >> 4) & 0x0F0F0F0Fu;
          const int k0 = (kb + u) * 64 + 32 * j;
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) {
            const int8_t* xr = s_x + (nt * 8 + g) * xs + k0 + 4 * t;
            const uint32_t b0 = *reinterpret_cast<const uint32_t*>(xr);
            const uint32_t b1 = *reinterpret_cast<const uint32_t*>(xr + 16);
            mma_u8s8(acc[nt], a0, a1, a2, a3, b0, b1);
          }
        }
      }
#pragma unroll
      for (int u = 0; u < UL; ++u) w[u] = nxt[u];
    }
  };

  // append keys to query n's list (unordered; one atomic per warp and group)
  auto append = [&](int n, bool in, uint64_t key, unsigned bal, unsigned rank) {
    if (!bal) return;
    unsigned base = 0;
    if (lane == 0) base = atomicAdd(fs.cnt + n, static_cast<unsigned>(__popc(bal)));
    base = __shfl_sync(0xffffffffu, base, 0);
    if (in && base + rank < static_cast<unsigned>(kFinCap)) fs.lists[static_cast<int64_t>(n) * kFinCap + base + rank] = key;
  };
  // backlog: row-blocks this warp scored before the bounds were known,
  // re-read from L2 (its own scores); nrb of them, rb_of(i) gives the i-th.
  // Loads of all of them in flight at once (an L2 round trip costs
  // microseconds while HBM is saturated); lanes 0-15 / 16-31 take two
  // row-blocks per load, lane order = row order.
  auto filter_from_l2 = [&](int nrb, auto rb_of, unsigned long long la, unsigned long long lb) {
    if (ks != 0) return;
    constexpr int RB = 8;
    for (int n = 0; n < B; ++n) {
      const uint64_t lo = __shfl_sync(0xffffffffu, n < 32 ? la : lb, n & 31);
      const float* srow = scores + static_cast<int64_t>(n) * score_stride;
      for (int i0 = 0; i0 < nrb; i0 += RB) {
        float v[RB / 2];
        int64_t rbs[RB / 2];
#pragma unroll
        for (int j = 0; j < RB / 2; ++j) {
          const int i = i0 + 2 * j + (lane >> 4);
          rbs[j] = i < nrb ? rb_of(i) : n_rb;
          const int64_t row = rbs[j] * 16 + (lane & 15);
          v[j] = (rbs[j] < n_rb && row < rows) ? __ldcg(srow + row) : 0.0f;
        }
#pragma unroll
        for (int j = 0; j < RB / 2; ++j) {
          const int64_t row = rbs[j] * 16 + (lane & 15);
          const uint64_t key = make_key(v[j], static_cast<uint32_t>(row));
          const bool in = rbs[j] < n_rb && row < rows && key >= lo;
          const unsigned bal = __ballot_sync(0xffffffffu, in);
          append(n, in, key, bal, __popc(bal & ((1u << lane) - 1u)));
        }
      }
    }
  };

  const bool sampler = c % fs.samp_step == 0;
  bool ready = false;
  unsigned long long lo_a = 0, lo_b = 0;  // lane l: lo[l], lo[l + 32]
  // schedule: rounds [0, n_static) static (round-robin row-blocks as in the
  // unfused kernel); KS == 1: the remaining row-blocks are claimed one at a
  // time from kFselCtr interleaved counters (claim issued one row-block
  // ahead), so warps on slower SMs take fewer and all finish together
  const int n_static = KS == 1 ? min(fs.n_static, rounds) : rounds;
  const int64_t s_rb = static_cast<int64_t>(n_static) * U;
  const int q = (c * 8 + wid) & (kFselCtr - 1);
  __shared__ int64_t s_dyn[8][kFselDynLog];
  int n_dyn = 0;        // claimed row-blocks scored before the bounds (logged)
  bool dyn_over = false;
  unsigned claim = 0;
  int64_t rb = static_cast<int64_t>(c) * RPC + rb_local;
  for (int rd = 0;; ++rd) {
    if (KS == 1 ? rb >= n_rb : rd >= rounds) break;
    const bool next_static = rd + 1 < n_static;
    if (KS == 1 && !next_static && lane == 0) claim = atomicAdd(fs.ctr + q * 32, 1u);
    // issue the bound poll now, look at it after the row-block
    unsigned long long pa = 0, pb = 0;
    if (!ready) {
      if (lane < B) pa = ld_relaxed_u64(fs.lo + lane);
      if (lane + 32 < B) pb = ld_relaxed_u64(fs.lo + lane + 32);
    }
    int acc[NT][4];
    if (rb < n_rb) {
      rowblock(rb, a, acc);
    } else {
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) acc[nt][0] = acc[nt][1] = acc[nt][2] = acc[nt][3] = 0;
    }
    const int64_t rbn = (KS > 1 || next_static)
                            ? rb + U
                            : s_rb + q + static_cast<int64_t>(kFselCtr) * __shfl_sync(0xffffffffu, claim, 0);
    if (rbn < n_rb) {
#pragma unroll
      for (int u = 0; u < UL; ++u)
        if (kb0 + u < kb1) a[u] = ldg_stream(wmma + ((rbn * nkb + kb0 + u) * 32 + lane));
    }
    if constexpr (KS > 1) {
      int* mine = s_acc + (wid * NT * 4) * 32;
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int e = 0; e < 4; ++e) mine[(nt * 4 + e) * 32 + lane] = acc[nt][e];
      __syncthreads();
      if (ks == 0) {
        for (int o = 1; o < KS; ++o) {
          const int* other = s_acc + ((wid + o) * NT * 4) * 32;
#pragma unroll
          for (int nt = 0; nt < NT; ++nt)
#pragma unroll
            for (int e = 0; e < 4; ++e) acc[nt][e] += other[(nt * 4 + e) * 32 + lane];
        }
      }
      __syncthreads();
    }
    // keys of this warp's row-block (ks == 0 warps), scores to L2/HBM
    const bool own = ks == 0 && rb < n_rb;
    uint64_t key[NT][4];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int64_t row = rb * 16 + g + ((e & 2) ? 8 : 0);
        const int n = nt * 8 + 2 * t + (e & 1);
        key[nt][e] = 0ull;
        if (own && row < rows && n < B) {
          const int aint = acc[nt][e] - 8 * s_sumq[n];
          const float cs = __fmul_rn(scales[row], s_sx[n]);
          const float sc = apply_phi(phi, __fmul_rn(static_cast<float>(aint), cs));
          scores[static_cast<int64_t>(n) * score_stride + row] = sc;
          key[nt][e] = make_key(sc, static_cast<uint32_t>(row));
        }
      }
    if (rd == 0 && sampler && ks == 0) {
      const int slot0 = (c / fs.samp_step) * RPC * 16 + rb_local * 16;
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int rr = g + ((e & 2) ? 8 : 0);
          const int n = nt * 8 + 2 * t + (e & 1);
          if (n < B && slot0 + rr < fs.n_samp)
            fs.samp[static_cast<int64_t>(n) * kFselSampleMax + slot0 + rr] = key[nt][e] ? key[nt][e] : 1ull;
        }
    }
    if (!ready) {
      const bool have = (lane >= B || pa != 0ull) && (lane + 32 >= B || pb != 0ull);
      if (__all_sync(0xffffffffu, have)) {
        ready = true;
        lo_a = pa;
        lo_b = pb;
        if (g_ktrace && threadIdx.x == 0) atomicMax(&g_ktrace[63], gtimer());
        // backlog: static rounds before this one, then the logged claims
        const int ns = min(rd, n_static);
        filter_from_l2(ns, [&](int i) { return static_cast<int64_t>(i) * U + static_cast<int64_t>(c) * RPC + rb_local; },
                       lo_a, lo_b);
        filter_from_l2(n_dyn, [&](int i) { return s_dyn[wid][i]; }, lo_a, lo_b);
        if (dyn_over && ks == 0 && lane < B) {
          atomicOr(fs.cnt + lane, 0x80000000u);  // claims not logged: exact fallback
          if (lane + 32 < B) atomicOr(fs.cnt + lane + 32, 0x80000000u);
        }
      } else if (rd >= n_static && rb < n_rb) {  // log this claimed row-block
        if (n_dyn < kFselDynLog) {
          if (lane == 0) s_dyn[wid][n_dyn] = rb;
          __syncwarp();
          ++n_dyn;
        } else {
          dyn_over = true;
        }
      }
    }
    if (ready && own) {
      // from registers: query n's 16 keys sit in the 8 lanes with
      // t == (n & 7) >> 1 — rows g (e = n & 1), then rows g + 8 (e = 2 + (n & 1))
      const unsigned below = (1u << lane) - 1u;
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const int n = nt * 8 + q;
          if (n >= B) break;
          const uint64_t lo = __shfl_sync(0xffffffffu, n < 32 ? lo_a : lo_b, n & 31);
          const bool mine = t == (q >> 1);
          const uint64_t k0 = (q & 1) ? key[nt][1] : key[nt][0];
          const uint64_t k1 = (q & 1) ? key[nt][3] : key[nt][2];
          const bool in0 = mine && k0 != 0 && k0 >= lo, in1 = mine && k1 != 0 && k1 >= lo;
          const unsigned bb0 = __ballot_sync(0xffffffffu, in0), bb1 = __ballot_sync(0xffffffffu, in1);
          const unsigned bal = bb0 | bb1;  // disjoint lanes hold k0 / k1 of different rows
          if (!bal) continue;
          const unsigned c0 = __popc(bb0);
          unsigned base = 0;
          if (lane == 0) base = atomicAdd(fs.cnt + n, c0 + __popc(bb1));
          base = __shfl_sync(0xffffffffu, base, 0);
          uint64_t* Lk = fs.lists + static_cast<int64_t>(n) * kFinCap + base;
          const unsigned lim = static_cast<unsigned>(kFinCap) - min(base, static_cast<unsigned>(kFinCap));
          if (in0 && __popc(bb0 & below) < lim) Lk[__popc(bb0 & below)] = k0;
          if (in1 && c0 + __popc(bb1 & below) < lim) Lk[c0 + __popc(bb1 & below)] = k1;
        }
    }
    rb = rbn;
  }
  if (g_ktrace && lane == 0) {
    atomicMin(&g_ktrace[54], gtimer());
    atomicMax(&g_ktrace[55], gtimer());
  }
  if (!ready) {
    // short problems: the bounds arrive after the last round
    unsigned long long pa = 0, pb = 0;
    const unsigned long long t0 = gtimer();
    for (;;) {
      if (lane < B) pa = ld_relaxed_u64(fs.lo + lane);
      if (lane + 32 < B) pb = ld_relaxed_u64(fs.lo + lane + 32);
      const bool have = (lane >= B || pa != 0ull) && (lane + 32 >= B || pb != 0ull);
      if (__all_sync(0xffffffffu, have)) {
        ready = true;
        break;
      }
      if (gtimer() - t0 > kFselTimeoutNs) break;
      __nanosleep(128);
    }
    if (ready) {
      filter_from_l2(n_static, [&](int i) { return static_cast<int64_t>(i) * U + static_cast<int64_t>(c) * RPC + rb_local; },
                     pa, pb);
      filter_from_l2(n_dyn, [&](int i) { return s_dyn[wid][i]; }, pa, pb);
      if (dyn_over && ks == 0 && lane < B) {
        atomicOr(fs.cnt + lane, 0x80000000u);
        if (lane + 32 < B) atomicOr(fs.cnt + lane + 32, 0x80000000u);
      }
    } else if (ks == 0 && lane < B) {
      atomicOr(fs.cnt + lane, 0x80000000u);  // no bound: sel_fin_kernel falls back
      if (lane + 32 < B) atomicOr(fs.cnt + lane + 32, 0x80000000u);
    }
  }
  if (g_ktrace && lane == 0) atomicMax(&g_ktrace[56], gtimer());
}

// ---------------------------------------------------------------------
// Finish: one 1024-thread CTA per query. T = the K-th largest listed key
// (keys striped over the threads: order is irrelevant to the order
// statistic); the emit in ascending index order goes through a row bitmap
// in shared memory (set bits, popcount prefix, ordered write) — no sort.
// Dynamic shared memory: ceil(n / 32) words.
// ---------------------------------------------------------------------
union FinShared {
  RangeScratch rs;
  FastSelScratch fss;
};

// The finisher for query b (one 1024-thread CTA); s_bm: ceil(n/32) words of
// shared memory for the ordered emit.
__device__ __noinline__ void fin_select_emit(const float* __restrict__ scores, int64_t stride, const FuseSel& fs,
                                             uint32_t* __restrict__ cand, int64_t cand_stride, int ordered,
                                             int* __restrict__ status, int b, FinShared& u, unsigned* s_bm) {
  constexpr int NT = kFinThreads, KPT = kFinKpt;
  RangeScratch& rs = u.rs;
  const uint32_t n = fs.n, K = fs.K;
  const unsigned total_raw = __ldcg(fs.cnt + b);
  const unsigned long long tau_max = fs.stream ? __ldcg(fs.lo + b) : 0ull;
  const bool dbg = g_ktrace && threadIdx.x == 0 && b == 0;
  if (dbg) g_ktrace[57] = gtimer();
  __syncthreads();  // everyone has read the count before it is cleared
  {  // zero at rest for the next call / replay: sample slots, bound, count
    unsigned long long* sp = reinterpret_cast<unsigned long long*>(fs.samp) + static_cast<int64_t>(b) * kFselSampleMax;
    for (int i = threadIdx.x; i < fs.n_samp; i += NT) sp[i] = 0ull;
    if (threadIdx.x == 0) {
      fs.lo[b] = 0ull;
      fs.cnt[b] = 0u;
    }
    if (b == 0 && threadIdx.x < kFselCtr) fs.ctr[threadIdx.x * 32] = 0u;
  }
  uint32_t* out = cand + static_cast<int64_t>(b) * cand_stride;
  const int total = static_cast<int>(total_raw & 0x7FFFFFFFu);
  const bool stream = fs.stream != 0;
  if (!(total_raw & 0x80000000u) && total >= static_cast<int>(K) && total <= kFinCap) {
    const unsigned long long* L = reinterpret_cast<const unsigned long long*>(fs.lists) + static_cast<int64_t>(b) * kFinCap;
    uint64_t k[KPT];
#pragma unroll
    for (int j = 0; j < KPT; ++j) {
      const int e = threadIdx.x + j * NT;
      k[j] = e < total ? __ldcg(L + e) : 0ull;
    }
    const int nw = static_cast<int>((n + 31) / 32);
    for (int i = threadIdx.x; i < nw; i += NT) s_bm[i] = 0u;
    if (dbg) g_ktrace[58] = gtimer();
    const uint64_t T = block_fast_select<NT, KPT>(k, K, &u.fss, (g_ktrace && b == 0) ? g_ktrace + 24 : nullptr);
    if (dbg) { g_ktrace[59] = gtimer(); g_ktrace[61] = total; }
    // stream path: T is exact only if no chunk's bound lies above it
    if (stream && tau_max > T) {
      if (g_ktrace && threadIdx.x == 0) { g_ktrace[84] = total_raw; g_ktrace[85] = tau_max; g_ktrace[86] = T; g_ktrace[87] = 4; g_ktrace[88] = b; }
      goto fallback;
    }
    if (!ordered) {
      // the caller does not return the candidate list: any order will do
      // (the exact recompute and the final top-k are order-independent)
      int c = 0;
#pragma unroll
      for (int j = 0; j < KPT; ++j) c += (k[j] != 0 && k[j] >= T) ? 1 : 0;
      int tot2;
      int pos = block_scan_excl<NT>(c, u.fss.scan, &tot2);
#pragma unroll
      for (int j = 0; j < KPT; ++j)
        if (k[j] != 0 && k[j] >= T) out[pos++] = key_index(k[j]);
      if (dbg) g_ktrace[60] = gtimer();
      return;
    }
#pragma unroll
    for (int j = 0; j < KPT; ++j)
      if (k[j] != 0 && k[j] >= T) {
        const uint32_t idx = key_index(k[j]);
        atomicOr(s_bm + (idx >> 5), 1u << (idx & 31));
      }
    __syncthreads();
    // thread t owns words [t*W, t*W + W): popcounts -> prefix -> ordered write
    const int W = (nw + NT - 1) / NT;
    const int w0 = threadIdx.x * W;
    int mine = 0;
    for (int i = 0; i < W; ++i)
      if (w0 + i < nw) mine += __popc(s_bm[w0 + i]);
    int tot2;
    int pos = block_scan_excl<NT>(mine, u.fss.scan, &tot2);
    for (int i = 0; i < W; ++i) {
      if (w0 + i >= nw) break;
      unsigned word = s_bm[w0 + i];
      while (word) {
        const int bit = __ffs(word) - 1;
        out[pos++] = static_cast<uint32_t>((w0 + i) * 32 + bit);
        word &= word - 1u;
      }
    }
    if (dbg) g_ktrace[60] = gtimer();
    return;
  }
  if (g_ktrace && threadIdx.x == 0) { g_ktrace[84] = total_raw; g_ktrace[85] = tau_max; g_ktrace[87] = 1; g_ktrace[88] = b; }
fallback:
  // fallback: exact select over the whole row, then an ordered emit
  __syncthreads();  // the scratch union changes hands
  if (threadIdx.x == 0 && status) atomicAdd(status, 1);
  if (dbg) g_ktrace[62] = 1;
  (void)rs;
  RowKeys rk{scores + static_cast<int64_t>(b) * stride, n};
  const uint64_t T = block_range_select<NT>(rk, n, K, &rs);
  const float* row = scores + static_cast<int64_t>(b) * stride;
  int base = 0;
  for (uint32_t i0 = 0; i0 < n; i0 += NT * KPT) {
    uint64_t k[KPT];
    int cnt = 0;
#pragma unroll
    for (int j = 0; j < KPT; ++j) {
      const uint32_t i = i0 + threadIdx.x * KPT + j;
      k[j] = i < n ? make_key(__ldcg(row + i), i) : 0ull;
      cnt += (i < n && k[j] >= T) ? 1 : 0;
    }
    int tot2;
    int pos = base + block_scan_excl<NT>(cnt, rs.scan, &tot2);
#pragma unroll
    for (int j = 0; j < KPT; ++j)
      if (k[j] != 0 && k[j] >= T) out[pos++] = key_index(k[j]);
    base += tot2;
  }
}


// ---------------------------------------------------------------------
// Small rows (n <= kFinCap = 8192), one 1024-thread CTA per query: the whole
// row in registers (thread t owns indices [8t, 8t + 8)), T = the K-th largest
// key by the shared-memory histogram select (block_fast_select: ~10 barriers
// whatever the rank, against one 16-way split per barrier in
// block_range_select — 9.1 -> 7.3 us for K = 820 of 8192, the FFN layers'
// top-10 %; cfg2 B=8 step 39.1 -> 37.6 us), ordered emit from the blocked layout.
// ---------------------------------------------------------------------
__global__ void __launch_bounds__(kFinThreads) sel_exact_fast_kernel(
    const float* __restrict__ scores, int64_t stride, uint32_t n, uint32_t K, uint32_t* __restrict__ cand,
    int64_t cand_stride) {
  constexpr int NT = kFinThreads, KPT = kFinKpt;
  __shared__ FastSelScratch fss;
  griddep_wait();
  griddep_launch();
  KTrace kt_(kKtPivot);
  const int b = blockIdx.x;
  const float* row = scores + static_cast<int64_t>(b) * stride;
  uint64_t k[KPT];
  const uint32_t i0 = threadIdx.x * KPT;
  if ((reinterpret_cast<uintptr_t>(row) & 15) == 0 && i0 + KPT <= n) {
#pragma unroll
    for (int j = 0; j < KPT; j += 4) {
      const float4 v = *reinterpret_cast<const float4*>(row + i0 + j);
      k[j] = make_key(v.x, i0 + j);
      k[j + 1] = make_key(v.y, i0 + j + 1);
      k[j + 2] = make_key(v.z, i0 + j + 2);
      k[j + 3] = make_key(v.w, i0 + j + 3);
    }
  } else {
#pragma unroll
    for (int j = 0; j < KPT; ++j) k[j] = i0 + j < n ? make_key(row[i0 + j], i0 + j) : 0ull;
  }
  const uint64_t T = block_fast_select<NT, KPT>(k, K, &fss);
  int c = 0;
#pragma unroll
  for (int j = 0; j < KPT; ++j) c += (k[j] != 0ull && k[j] >= T) ? 1 : 0;
  int total;
  int pos = block_scan_excl<NT>(c, fss.scan, &total);
  uint32_t* out = cand + static_cast<int64_t>(b) * cand_stride;
#pragma unroll
  for (int j = 0; j < KPT; ++j)
    if (k[j] != 0ull && k[j] >= T) out[pos++] = i0 + j;
}

__global__ void __launch_bounds__(kFinThreads) sel_fin_kernel(
    const float* __restrict__ scores, int64_t stride, FuseSel fs, uint32_t* __restrict__ cand,
    int64_t cand_stride, int ordered, int* __restrict__ status) {
  __shared__ FinShared u;
  extern __shared__ __align__(16) unsigned char fin_smem[];
  griddep_wait();
  griddep_launch();
  KTrace kt_(kKtEmit);
  fin_select_emit(scores, stride, fs, cand, cand_stride, ordered, status, blockIdx.x, u,
                  reinterpret_cast<unsigned*>(fin_smem));
}

#if HIRE_EXPERIMENTS
// ---------------------------------------------------------------------
// One launch for everything after the fused proxy kernel (hire_topk):
//   CTAs [0, B)   : the finisher of query b (fin_select_emit), then flag[b]
//   CTAs [B, B+R) : recompute workers — for each query in turn, wait for its
//                   flag, gather + score its candidate rows (the arithmetic
//                   of recompute_fast: lane chunks in order, fmaf, fixed
//                   butterfly -> bit-identical values), then take a ticket;
//                   the last worker of query b runs the final top-k +
//                   softmax (hire.hpp:74-80, 135-142) and clears flag/ticket.
// Two kernel boundaries and two cold starts fewer than fin -> K4 -> K5.
// post: [2B] zero-at-rest words (flags, tickets). All CTAs co-resident (one
// per SM, B + R <= SMs).
// ---------------------------------------------------------------------
constexpr int kPostMaxK = 256;

template <typename T, int CPL>
__device__ __forceinline__ float post_row_dot(const T* __restrict__ w, int64_t pitch_vec, int64_t row,
                                              const float* s_x, int lane) {
  constexpr int E = Vec16<T>::kElems;
  const uint4* rp = reinterpret_cast<const uint4*>(w) + row * pitch_vec;
  float acc = 0.0f;
#pragma unroll
  for (int c0 = 0; c0 < CPL; c0 += 4) {
    uint4 v[4];
#pragma unroll
    for (int c = 0; c < 4; ++c)
      if (c0 + c < CPL) v[c] = ldg_stream(rp + lane + 32 * (c0 + c));
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      if (c0 + c >= CPL) break;
      float f[E], xv[E];
      Vec16<T>::expand(v[c], f);
      load_x_vec<E>(s_x + (lane + 32 * (c0 + c)) * E, xv);
#pragma unroll
      for (int e = 0; e < E; ++e) acc = fmaf(f[e], xv[e], acc);
    }
  }
  return warp_sum_f32(acc);
}

template <typename T, int CPL>
__global__ void __launch_bounds__(kFinThreads, 1) fsel_post_kernel(
    const float* __restrict__ scores, int64_t stride, FuseSel fs, uint32_t* __restrict__ cand, int64_t cand_stride,
    int ordered, int* __restrict__ status, const T* __restrict__ w, int d, const float* __restrict__ x, int phi,
    float* __restrict__ vals, int kp, int K, uint32_t* __restrict__ out_idx, float* __restrict__ out_val,
    float* __restrict__ out_prob, int64_t out_stride, unsigned* __restrict__ post, int R) {
  constexpr int NT = kFinThreads;
  __shared__ FinShared u;
  __shared__ uint64_t s_sel[kPostMaxK];
  __shared__ double s_red[NT / 32];
  __shared__ unsigned s_last;
  extern __shared__ __align__(16) unsigned char post_smem[];
  griddep_wait();
  griddep_launch();
  const int B = static_cast<int>(gridDim.x) - R;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  if (static_cast<int>(blockIdx.x) < B) {
    KTrace kt_(kKtEmit);
    const int b = blockIdx.x;
    fin_select_emit(scores, stride, fs, cand, cand_stride, ordered, status, b, u,
                    reinterpret_cast<unsigned*>(post_smem));
    __syncthreads();
    if (tid == 0) {
      __threadfence();
      atomicExch(post + b, 1u);
    }
    return;
  }
  KTrace kt_(kKtRecompute);
  const int j = blockIdx.x - B;
  float* s_x = reinterpret_cast<float*>(post_smem);
  constexpr int E = Vec16<T>::kElems;
  const int64_t pitch_vec = static_cast<int64_t>(d) / E;
  for (int b = 0; b < B; ++b) {
    if (tid == 0) {
      const unsigned long long t0 = gtimer();
      while (ld_relaxed_gpu(post + b) == 0u && gtimer() - t0 < kFselTimeoutNs) __nanosleep(64);
      fence_acq_rel_gpu();
    }
    block_copy(s_x, x + static_cast<int64_t>(b) * d, d);
    __syncthreads();
    for (int i = j * 32 + wid; i < kp; i += R * 32) {
      const int64_t row = __ldcg(cand + static_cast<int64_t>(b) * cand_stride + i);
      const float acc = post_row_dot<T, CPL>(w, pitch_vec, row, s_x, lane);
      if (lane == 0) vals[static_cast<int64_t>(b) * kp + i] = apply_phi(phi, acc);
    }
    __syncthreads();
    if (tid == 0) {
      __threadfence();
      s_last = atomicAdd(post + B + b, 1u) == static_cast<unsigned>(R - 1) ? 1u : 0u;
      if (s_last) fence_acq_rel_gpu();
    }
    __syncthreads();
    if (s_last) {
      // final top-K of the kp exact values (ties by index), rank order
      constexpr int KPT = kFinKpt;
      RegKeys<KPT> src;
#pragma unroll
      for (int q = 0; q < KPT; ++q) {
        const int i = tid * KPT + q;
        src.k[q] = i < kp ? make_key(__ldcg(vals + static_cast<int64_t>(b) * kp + i),
                                     __ldcg(cand + static_cast<int64_t>(b) * cand_stride + i))
                          : 0ull;
      }
      const int Kq = min(K, kp);
      const uint64_t T2 = Kq >= kp ? 1ull : block_range_select<NT>(src, kp, Kq, &u.rs);
      int c = 0;
#pragma unroll
      for (int q = 0; q < KPT; ++q) c += (src.k[q] && src.k[q] >= T2) ? 1 : 0;
      int total;
      int pos = block_scan_excl<NT>(c, u.rs.scan, &total);
#pragma unroll
      for (int q = 0; q < KPT; ++q)
        if (src.k[q] && src.k[q] >= T2) s_sel[pos++] = src.k[q];
      __syncthreads();
      const uint64_t mine = tid < Kq ? s_sel[tid] : 0ull;
      int rank = 0;
      for (int q = 0; q < Kq; ++q) rank += s_sel[q] > mine ? 1 : 0;
      __syncthreads();
      if (tid < Kq) s_sel[rank] = mine;
      __syncthreads();
      if (tid < Kq) {
        out_idx[b * out_stride + tid] = key_index(s_sel[tid]);
        out_val[b * out_stride + tid] = key_value(s_sel[tid]);
      }
      if (out_prob) {
        // hire.hpp:135-142: p_i = float(exp(double(v_i) - v_max)) / double sum
        const double vmax = static_cast<double>(key_value(s_sel[0]));
        double local = 0.0;
        for (int q = tid; q < Kq; q += NT) local += exp(static_cast<double>(key_value(s_sel[q])) - vmax);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) local += __shfl_xor_sync(0xffffffffu, local, o);
        if (lane == 0) s_red[wid] = local;
        __syncthreads();
        double sum = 0.0;
#pragma unroll
        for (int v = 0; v < NT / 32; ++v) sum += s_red[v];
        for (int q = tid; q < Kq; q += NT) {
          const float pj = static_cast<float>(exp(static_cast<double>(key_value(s_sel[q])) - vmax));
          out_prob[b * out_stride + q] = static_cast<float>(static_cast<double>(pj) / sum);
        }
      }
      if (tid == 0) {
        post[b] = 0u;
        post[B + b] = 0u;
      }
    }
    __syncthreads();  // s_x / s_sel reuse
  }
}

#endif  // HIRE_EXPERIMENTS

}  // namespace hire_dev
