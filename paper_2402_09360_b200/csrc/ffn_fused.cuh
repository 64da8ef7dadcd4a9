// ffn_fused.cuh — the whole HiRE-FFN layer (ffn_group_sparse with g = 1,
// ffn.hpp:211-219) as ONE persistent cooperative kernel for decode batches
// (B <= 16), so the latency-bound chain of 7 launches collapses into phases
// separated by flag hand-offs instead of kernel boundaries:
//
//   P0 every CTA  : quantise x to int8 in shared memory (redundantly — no
//                   hand-off needed), stage x fp32 for the recompute
//   P1 every CTA  : int4 x int8 proxy scores on the tensor cores (the K1
//                   mma.sync m16n8k32 u8*s8 loop), phi = ReLU, -> scores[B][m]
//   P2 CTA b < B  : exact top-k' of scores[b] (radix select in smem), written
//                   in ascending unit order -> cand[b]          (ffn.hpp:181)
//   P3 every CTA  : exact phi(<U_j, x_b>) for the B*k' candidates (warp per
//                   row, fixed tree — same arithmetic as recompute_fast)
//   P4 CTA b < B  : top-k by exact activation, ascending unit order + values
//                   -> sel[b], selact[b]                   (ffn.hpp:188-199)
//   P5 every CTA  : down-projection partial sums over chunks of 8 selected
//                   units (same chunking/order as ffn_down_partial)
//   P6 every CTA  : fixed-order reduction of the partials -> out[B][d]
//
// Hand-offs: counters in global memory, written after a gpu-scope fence and
// read with acquire loads; consumers re-read produced data through L2
// (__ldcg). The last CTA to leave resets the counters for the next launch.
// Co-residency of all CTAs is guaranteed by the cooperative launch (one CTA
// per SM). Results are bit-identical to the unfused fast path.
#pragma once
#include "common.cuh"
#include "exact.cuh"
#include "score.cuh"
#include "select.cuh"
#include "select2.cuh"

namespace hire_dev {

struct FusedFfnArgs {
  const uint4* u_mma;      // int4 proxy of U, MMA-tiled
  const float* scales;     // [m]
  const void* u;           // U [m][d] (T)
  const void* v;           // V [m][d] (T)
  const float* x;          // [B][d]
  int B, m, d, kp, k, phi;
  float* scores;           // [B][m]
  uint64_t* piv;           // [B][2] bracket pivots (hi, lo)
  uint64_t* thr;           // [B] exact k'-th proxy key
  int* qcnt;               // unused (kept for layout)
  int* acnt;               // [B][G] keys above the bracket, per CTA slice
  int* pcnt;               // [B][G] candidates per CTA slice
  unsigned* gh;            // [B][kWinGroups][kWinBins] window histogram (zeroed in P2a)
  uint64_t* lists;         // [B][kWinGroups][kWinBins][kBinCap] window keys by bin
  int wmax;                // max rows per CTA slice
  uint64_t* pairs;         // [B][G][wmax] (exact activation, unit) keys per CTA slice
  uint32_t* sel;           // [B][k]   (out, ascending)
  float* selact;           // [B][k]
  float* partial;          // [B][nch][d]
  float* out;              // [B][d]
  int* counters;           // hand-off counters, one 128-B line each
  long long* trace;        // optional %globaltimer stamps (CTA 0, thread 0)
};

__device__ __forceinline__ long long globaltimer() {
  long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// Hand-off counters. Arrivals of many CTAs on one address serialise at the
// L2 atomic unit (~27 cycles each: 148 arrivals ~ 2 us), so every barrier
// spreads its arrivals over kSpread counters on separate 128-B lines; the
// waiter sums them.
constexpr int kSpread = 16;
constexpr int kBarInts = kSpread * 32;  // one barrier's counter block
enum { kCntGemv = 0, kCntPiv = 1 * kBarInts, kCntWin = 2 * kBarInts, kCntThr = 3 * kBarInts,
       kCntPairs = 4 * kBarInts, kCntSel = 5 * kBarInts, kCntDown = 6 * kBarInts, kCntExit = 7 * kBarInts,
       kCntInts = 8 * kBarInts };

// One warp polls the spread counters with relaxed loads (an acquire probe
// invalidates the SM's L1 every time). Once the target is reached the warp
// re-reads all counters with one acquire load (synchronising with every
// arriving CTA's release) — cheaper than a gpu-scope fence.
__device__ __forceinline__ int ld_acquire_gpu_i32(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void cta_wait_geq(const int* p, int target) {
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    for (;;) {
      const int v = lane < kSpread ? static_cast<int>(ld_relaxed_gpu(reinterpret_cast<const unsigned*>(p + lane * 32))) : 0;
      if (__reduce_add_sync(0xffffffffu, v) >= target) break;
    }
    if (lane < kSpread) (void)ld_acquire_gpu_i32(p + lane * 32);
  }
  __syncthreads();
}

// The CTA barrier orders every thread's writes before thread 0's
// gpu-scope release (cumulative), which then arrives: one fence per CTA
// instead of a MEMBAR in every thread.
__device__ __forceinline__ void cta_arrive(int* p, int inc) {
  __syncthreads();
  if (threadIdx.x == 0) {
    int old;  // returning atomic: performed at L2 before the CTA moves on
    asm volatile("atom.release.gpu.global.add.s32 %0, [%1], %2;"
                 : "=r"(old)
                 : "l"(p + (blockIdx.x % kSpread) * 32), "r"(inc)
                 : "memory");
  }
}

constexpr int kFusedThreads = 512;
constexpr int kFusedWarps = kFusedThreads / 32;
constexpr int kFusedCh = 8;  // units per down-projection chunk (= ffn_down_partial's)

#define FUSED_STAMP(i)                                                  \
  do {                                                                  \
    if (a.trace && blockIdx.x == 0 && threadIdx.x == 0) a.trace[i] = globaltimer(); \
  } while (0)

template <typename T, int NT, int KS>
__global__ void __launch_bounds__(kFusedThreads, 1) ffn_fused_kernel(FusedFfnArgs a) {
  griddep_wait();
  FUSED_STAMP(0);
  if (a.trace && blockIdx.x == 0 && threadIdx.x == 0) a.trace[20] = clock64();
  extern __shared__ __align__(16) unsigned char smem[];
  constexpr int E = Vec16<T>::kElems;
  const int B = a.B, m = a.m, d = a.d;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int G = gridDim.x;
  const int xs = d + 16;
  // shared memory: [x fp32 B*d] [xq NT*8*xs] [acc 16 warps*NT*4*32 ints] ; the
  // selector pool (m floats / kp keys) aliases the xq+acc region after P1.
  float* s_xf = reinterpret_cast<float*>(smem);
  int8_t* s_xq = reinterpret_cast<int8_t*>(smem + static_cast<size_t>(B) * d * 4);
  int* s_acc = reinterpret_cast<int*>(s_xq + static_cast<size_t>(NT) * 8 * xs);
  unsigned char* s_pool = reinterpret_cast<unsigned char*>(s_xq);
  __shared__ float s_sx[16];
  __shared__ int s_sum[16];
  __shared__ float s_red[kFusedWarps];
  __shared__ int s_redi[kFusedWarps];
  struct FusedScratch {
    uint64_t samp[128];
    uint64_t piv[4];
    int scan[64];
  };
  __shared__ FusedScratch sc;

  const int nkb = d / 64;
  const int n_rb = (m + 15) / 16;
  constexpr int RB_PER_CTA = kFusedWarps / KS;
  const int rb_local = wid / KS, ks = wid % KS;
  const int kb0 = ks * nkb / KS, kb1 = (ks + 1) * nkb / KS;
  const int g = lane >> 2, t = lane & 3;

  // ---- prologue: first proxy loads (independent of x) -------------------
  constexpr int U = 4;
  uint4 av[U];
  {
    const int rb = blockIdx.x * RB_PER_CTA + rb_local;
    if (rb < n_rb)
#pragma unroll
      for (int uu = 0; uu < U; ++uu)
        if (kb0 + uu < kb1) av[uu] = ldg_stream(a.u_mma + ((static_cast<int64_t>(rb) * nkb + kb0 + uu) * 32 + lane));
  }

  // ---- P0: x -> smem (fp32) and int8 quantisation (prep_x_int8 rule) ----
  // all queries at once: warps are split evenly over the B queries (wpq
  // warps each); two barriers in total, independent of B.
  // x fp32 in shared memory; for 8-element row chunks (bf16 rows) each
  // query's vector is stored as [d/2 low halves | d/2 high halves] of the
  // chunks so the P3 128-bit reads are conflict-free (lane stride 16 B)
  auto xf_idx = [&](int b, int i) -> int {
    if constexpr (E == 8) return b * d + ((i >> 2) & 1) * (d >> 1) + (i >> 3) * 4 + (i & 3);
    else return b * d + i;
  };
  for (int v = tid; v < B * d / 4; v += kFusedThreads) {
    const int i = 4 * v, b = i / d, ii = i % d;
    *reinterpret_cast<float4*>(s_xf + xf_idx(b, ii)) = __ldg(reinterpret_cast<const float4*>(a.x) + v);
  }
  __syncthreads();
  FUSED_STAMP(13);
  {
    const int wpq = kFusedWarps / B > 0 ? kFusedWarps / B : 1;  // warps per query
    const int qb = wid / wpq, qw = wid % wpq;                     // my query, my rank in it
    const bool active = qb < B;
    float mx = 0.0f;
    if (active)
      for (int i = qw * 32 + lane; i < d; i += wpq * 32) mx = fmaxf(mx, fabsf(s_xf[xf_idx(qb, i)]));
    mx = warp_max_f32(mx);
    if (lane == 0) s_red[wid] = mx;
    __syncthreads();
    float sx = 1.0f;
    if (active) {
      float v = 0.0f;
      for (int w = 0; w < wpq; ++w) v = fmaxf(v, s_red[qb * wpq + w]);
      sx = v > 0.0f ? __fdiv_rn(v, 127.0f) : 1.0f;
    }
    int local = 0;
    if (active)
      for (int i = qw * 32 + lane; i < d; i += wpq * 32) {
        const int q = rhaz_clamp(__fdiv_rn(s_xf[xf_idx(qb, i)], sx), 127);
        local += q;
        s_xq[qb * xs + i] = static_cast<int8_t>(q);
      }
    local = warp_sum_i32(local);
    if (lane == 0) s_redi[wid] = local;
    if (active && qw == 0 && lane == 0) s_sx[qb] = sx;
    // zero the padded queries of the MMA B operand (16-byte stores)
    for (int i = tid; i < (NT * 8 - B) * (d / 16); i += kFusedThreads) {
      const int n = B + i / (d / 16), c = i % (d / 16);
      *reinterpret_cast<int4*>(s_xq + n * xs + c * 16) = make_int4(0, 0, 0, 0);
    }
    __syncthreads();
    if (tid < B) {
      int sum = 0;
      for (int w = 0; w < wpq; ++w) sum += s_redi[tid * wpq + w];
      s_sum[tid] = sum;
    }
    __syncthreads();
  }
  FUSED_STAMP(1);

  // ---- P1: proxy scores on the tensor cores -------------------------------
  int done_rb = 0;
  for (int rb_base = blockIdx.x * RB_PER_CTA; rb_base < n_rb; rb_base += G * RB_PER_CTA) {
    const int rb = rb_base + rb_local;
    int acc[NT][4];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) acc[nt][0] = acc[nt][1] = acc[nt][2] = acc[nt][3] = 0;
    if (rb < n_rb) {
      for (int kb = kb0; kb < kb1; kb += U) {
        uint4 nxt[U];
#pragma unroll
        for (int uu = 0; uu < U; ++uu)
          if (kb + U + uu < kb1) nxt[uu] = ldg_stream(a.u_mma + ((static_cast<int64_t>(rb) * nkb + kb + U + uu) * 32 + lane));
#pragma unroll
        for (int uu = 0; uu < U; ++uu) {
          if (kb + uu >= kb1) break;
          const uint32_t w4[4] = {av[uu].x, av[uu].y, av[uu].z, av[uu].w};
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            const uint32_t u0 = w4[2 * j] ^ 0x88888888u, u1 = w4[2 * j + 1] ^ 0x88888888u;
            const uint32_t a0 = u0 & 0x0F0F0F0Fu, a1 = (u0 >> 4) & 0x0F0F0F0Fu;
            const uint32_t a2 = u1 & 0x0F0F0F0Fu, a3 = (u1 >> 4) & 0x0F0F0F0Fu;
            const int k0 = (kb + uu) * 64 + 32 * j;
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) {
              const int8_t* xr = s_xq + (nt * 8 + g) * xs + k0 + 4 * t;
              mma_u8s8(acc[nt], a0, a1, a2, a3, *reinterpret_cast<const uint32_t*>(xr),
                       *reinterpret_cast<const uint32_t*>(xr + 16));
            }
          }
        }
#pragma unroll
        for (int uu = 0; uu < U; ++uu) av[uu] = nxt[uu];
      }
    }
    const int rbn = rb + G * RB_PER_CTA;
    if (rbn < n_rb)
#pragma unroll
      for (int uu = 0; uu < U; ++uu)
        if (kb0 + uu < kb1) av[uu] = ldg_stream(a.u_mma + ((static_cast<int64_t>(rbn) * nkb + kb0 + uu) * 32 + lane));
    if constexpr (KS > 1) {
      int* mine = s_acc + (wid * NT * 4) * 32;
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int e = 0; e < 4; ++e) mine[(nt * 4 + e) * 32 + lane] = acc[nt][e];
      __syncthreads();
      if (ks == 0)
        for (int o = 1; o < KS; ++o) {
          const int* other = s_acc + ((wid + o) * NT * 4) * 32;
#pragma unroll
          for (int nt = 0; nt < NT; ++nt)
#pragma unroll
            for (int e = 0; e < 4; ++e) acc[nt][e] += other[(nt * 4 + e) * 32 + lane];
        }
      __syncthreads();
    }
    if (ks == 0 && rb < n_rb) {
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int row = rb * 16 + g + ((e & 2) ? 8 : 0);
          const int n = nt * 8 + 2 * t + (e & 1);
          if (row < m && n < B) {
            const float cs = __fmul_rn(a.scales[row], s_sx[n]);
            a.scores[static_cast<int64_t>(n) * m + row] =
                apply_phi(a.phi, __fmul_rn(static_cast<float>(acc[nt][e] - 8 * s_sum[n]), cs));
          }
        }
    }
    ++done_rb;
  }
  FUSED_STAMP(2);
  if (a.trace && tid == 0) atomicMax(reinterpret_cast<unsigned long long*>(a.trace + 33), static_cast<unsigned long long>(globaltimer()));
  cta_arrive(a.counters + kCntGemv, 1);
  if (a.trace && tid == 0) atomicMax(reinterpret_cast<unsigned long long*>(a.trace + 35), static_cast<unsigned long long>(globaltimer()));

  // ---- P2a: bracket pivots for the k'-th proxy key (CTA b per query) ------
  // A 128-key sample of scores[b] ranked by counting; the sample keys at
  // ranks (k'-1)S/m -/+ 3.5 sigma bracket the k'-th key (select.cuh). The
  // bracket is split into kWinBins value-word bins for P2b/P2c.
  int f_row, w_row;  // this CTA's row slice (width rule)
  {
    const int base = m / G, extra = m % G;
    f_row = blockIdx.x * base + (blockIdx.x < extra ? blockIdx.x : extra);
    w_row = base + (blockIdx.x < extra ? 1 : 0);
  }
  __shared__ RangeScratch rs2;
  if (blockIdx.x < B) {
    const int b = blockIdx.x;
    for (int i = tid; i < kWinGroups * kWinBins; i += kFusedThreads) a.gh[b * kWinGroups * kWinBins + i] = 0u;
    cta_wait_geq(a.counters + kCntGemv, G);
    FUSED_STAMP(3);
    constexpr int S = 128;
    __shared__ unsigned s_top;
    if (tid < S) {
      const int i = static_cast<int>((static_cast<int64_t>(tid) * m) / S);
      sc.samp[tid] = make_key(__ldcg(a.scores + static_cast<int64_t>(b) * m + i), static_cast<uint32_t>(i));
    }
    if (tid == 0) {
      sc.piv[0] = ~0ull;
      sc.piv[1] = 0ull;
      s_top = 0u;
    }
    __syncthreads();
    if (tid < S) atomicMax(&s_top, static_cast<unsigned>(sc.samp[tid] >> 32));
    const float p = static_cast<float>(a.kp) / static_cast<float>(m);
    const float mu = static_cast<float>(a.kp - 1) * S / static_cast<float>(m);
    const float delta = fmaxf(3.5f * sqrtf(S * p * (1.0f - p)), 3.0f);
    const int r_hi = static_cast<int>(floorf(mu - delta));
    const int r_lo = static_cast<int>(ceilf(mu + delta));
    block_rank_256<kFusedThreads>(sc.samp, S, [&](int jj, int r) {
      if (r == r_hi) sc.piv[0] = sc.samp[jj];
      if (r == r_lo) sc.piv[1] = sc.samp[jj];
    });
    __syncthreads();
    if (tid == 0) {
      const uint64_t hi = sc.piv[0], lo = sc.piv[1];
      const unsigned vlo = static_cast<unsigned>(lo >> 32);
      const unsigned vtop = max(vlo, hi != ~0ull ? static_cast<unsigned>(hi >> 32) : s_top);
      const int bits = 32 - __clz(vtop - vlo);
      const int sh = bits > 8 ? bits - 8 : 0;
      a.piv[4 * b] = hi;
      a.piv[4 * b + 1] = lo;
      a.piv[4 * b + 2] = static_cast<uint64_t>(vlo) | (static_cast<uint64_t>(sh) << 32);
    }
    cta_arrive(a.counters + kCntPiv, 1);
  }

  // ---- P2b: every CTA counts its slice above the bracket and files the ---
  // bracket keys by bin (per chunk-group lists); counts per CTA slot, no
  // same-address atomics across CTAs.
  cta_wait_geq(a.counters + kCntPiv, B);
  FUSED_STAMP(4);
  {
    __shared__ int s_above[16];
    __shared__ unsigned s_pf[64];  // rows of the slice above some query's lower pivot (bitmap)
    if (tid < B) s_above[tid] = 0;
    if (tid < 64) s_pf[tid] = 0u;
    __syncthreads();
    const int wpq = kFusedWarps / B > 0 ? kFusedWarps / B : 1;
    const int qb = wid / wpq, qw = wid % wpq;
    if (qb < B) {
      const uint64_t hi = __ldcg(a.piv + 4 * qb), lo = __ldcg(a.piv + 4 * qb + 1), bp = __ldcg(a.piv + 4 * qb + 2);
      const unsigned vlo = static_cast<unsigned>(bp);
      const int bsh = static_cast<int>(bp >> 32);
      unsigned* ghg = a.gh + (static_cast<int64_t>(qb) * kWinGroups + blockIdx.x % kWinGroups) * kWinBins;
      uint64_t* lsg = a.lists + (static_cast<int64_t>(qb) * kWinGroups + blockIdx.x % kWinGroups) * kWinBins * kBinCap;
      int above = 0;
      for (int r0 = qw * 32; r0 < w_row; r0 += wpq * 32) {
        const int r = r0 + lane;
        if (r < w_row) {
          const uint64_t key = make_key(__ldcg(a.scores + static_cast<int64_t>(qb) * m + f_row + r), static_cast<uint32_t>(f_row + r));
          above += key > hi ? 1 : 0;
          if (key > lo) atomicOr(&s_pf[r >> 5], 1u << (r & 31));
          if (key > lo && key <= hi) {
            const unsigned bin = win_bin(key, vlo, bsh);
            const unsigned lp = atomicAdd(&ghg[bin], 1u);
            if (lp < kBinCap) lsg[bin * kBinCap + lp] = key;
          }
        }
      }
      above = warp_sum_i32(above);
      if (lane == 0 && above) atomicAdd(&s_above[qb], above);
    }
    __syncthreads();
    if (tid < B) a.acnt[tid * G + blockIdx.x] = s_above[tid];
    // likely k'-candidates: start streaming their U rows into L2 so the P3
    // gather after the threshold hand-off reads L2, not HBM
    if (tid < w_row && ((s_pf[tid >> 5] >> (tid & 31)) & 1u))
      bulk_prefetch_l2(static_cast<const unsigned char*>(a.u) + static_cast<int64_t>(f_row + tid) * d * sizeof(T),
                       static_cast<unsigned>(d * sizeof(T)));
    if (a.trace && tid == 0) atomicMax(reinterpret_cast<unsigned long long*>(a.trace + 28), static_cast<unsigned long long>(globaltimer()));
  }
  cta_arrive(a.counters + kCntWin, 1);

  // ---- P2c: exact k'-th key per query (CTA b): the bin holding rank ------
  // k' - above, then the rank among that bin's keys.
  if (blockIdx.x < B) {
    const int b = blockIdx.x;
    cta_wait_geq(a.counters + kCntWin, G);
    FUSED_STAMP(5);
    __shared__ long long s_red2[kFusedWarps];
    __shared__ int s_bstar, s_m, s_bad;
    __shared__ long long s_r2;
    __shared__ uint64_t s_T;
    long long ab = 0;
    for (int c = tid; c < G; c += kFusedThreads) ab += __ldcg(a.acnt + b * G + c);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ab += __shfl_xor_sync(0xffffffffu, ab, o);
    if (lane == 0) s_red2[wid] = ab;
    if (tid == 0) {
      s_bad = 1;
      rs2.small_n = 0;
    }
    __syncthreads();
    long long above_t = 0;
#pragma unroll
    for (int w = 0; w < kFusedWarps; ++w) above_t += s_red2[w];
    const long long r = static_cast<long long>(a.kp) - above_t;
    // bins, top first: thread t < kWinBins holds bin kWinBins-1-t
    unsigned hb = 0, hmax = 0;
    if (tid < kWinBins) {
#pragma unroll
      for (int g2 = 0; g2 < kWinGroups; ++g2) {
        const unsigned v = __ldcg(a.gh + (static_cast<int64_t>(b) * kWinGroups + g2) * kWinBins + (kWinBins - 1 - tid));
        hb += v;
        hmax = max(hmax, v);
      }
    }
    int tot;
    const int ex = block_exclusive_scan<kFusedThreads>(static_cast<int>(hb), sc.scan, &tot);
    if (tid < kWinBins && r >= 1 && ex < r && ex + static_cast<long long>(hb) >= r) {
      s_bstar = kWinBins - 1 - tid;
      s_r2 = r - ex;
      s_m = static_cast<int>(hb);
      s_bad = hmax > kBinCap ? 2 : 0;
    }
    __syncthreads();
    FUSED_STAMP(29);
    uint64_t T;
    if (!s_bad) {
      const unsigned bstar = static_cast<unsigned>(s_bstar);
      if (tid < kWinGroups * kBinCap) {
        const int g2 = tid / kBinCap, j = tid % kBinCap;
        const unsigned cg = __ldcg(a.gh + (static_cast<int64_t>(b) * kWinGroups + g2) * kWinBins + bstar);
        if (static_cast<unsigned>(j) < cg) {
          const uint64_t kk = __ldcg(reinterpret_cast<const unsigned long long*>(a.lists) +
                                     ((static_cast<int64_t>(b) * kWinGroups + g2) * kWinBins + bstar) * kBinCap + j);
          const int pidx = atomicAdd(&rs2.small_n, 1);
          rs2.ckeys[pidx] = kk;
        }
      }
      __syncthreads();
      const int mb = s_m;
      RegKeys<1> src;
      src.k[0] = tid < mb ? rs2.ckeys[tid] : 0ull;
      __syncthreads();
      T = block_range_select<kFusedThreads>(src, mb, s_r2, &rs2);
    } else {  // bracket missed or a bin list overflowed: exact select over all m scores
      RowKeys src{a.scores + static_cast<int64_t>(b) * m, static_cast<uint32_t>(m)};
      T = block_range_select<kFusedThreads>(src, m, a.kp, &rs2);
    }
    FUSED_STAMP(30);
    if (tid == 0) a.thr[b] = T;
    cta_arrive(a.counters + kCntThr, 1);
  }

  // ---- P3: every CTA recomputes the candidates in its own rows ------------
  cta_wait_geq(a.counters + kCntThr, B);
  FUSED_STAMP(6);
  if (a.trace && tid == 0) atomicMax(reinterpret_cast<unsigned long long*>(a.trace + 23), static_cast<unsigned long long>(globaltimer()));
  {
    // candidate mask per row of this slice (bit b: row is a k'-candidate of
    // query b); rows with any bit are recomputed once for all their queries
    unsigned* s_mask = reinterpret_cast<unsigned*>(s_pool);          // [w_row]
    int* s_rows = reinterpret_cast<int*>(s_mask + w_row);             // [w_row] compacted
    uint64_t* s_key = reinterpret_cast<uint64_t*>(s_rows + w_row);  // [B][w_row] (8 w_row bytes in: aligned)
    __shared__ int s_nrow;
    __shared__ int s_nb[16];
    for (int r = tid; r < w_row; r += kFusedThreads) s_mask[r] = 0u;
    if (tid < B) s_nb[tid] = 0;
    __syncthreads();
    for (int t2 = tid; t2 < B * w_row; t2 += kFusedThreads) {
      const int qb = t2 / w_row, r = t2 % w_row;
      const uint64_t T = __ldcg(a.thr + qb);
      if (make_key(__ldcg(a.scores + static_cast<int64_t>(qb) * m + f_row + r), static_cast<uint32_t>(f_row + r)) >= T)
        atomicOr(&s_mask[r], 1u << qb);
    }
    __syncthreads();
    if (a.trace && tid == 0) atomicMax(reinterpret_cast<unsigned long long*>(a.trace + 36), static_cast<unsigned long long>(globaltimer()));
    if (wid == 0) {
      int n = 0;
      for (int r0 = 0; r0 < w_row; r0 += 32) {
        const int r = r0 + lane;
        const bool c = r < w_row && s_mask[r] != 0u;
        const unsigned bc = __ballot_sync(0xffffffffu, c);
        if (c) s_rows[n + __popc(bc & ((1u << lane) - 1u))] = r;
        n += __popc(bc);
      }
      if (lane == 0) s_nrow = n;
    }
    __syncthreads();
    if (a.trace && tid == 0) atomicMax(reinterpret_cast<unsigned long long*>(a.trace + 37), static_cast<unsigned long long>(globaltimer()));
    const int nrow = s_nrow;
    const long long p3_t0 = a.trace ? globaltimer() : 0;
    const T* U_ = static_cast<const T*>(a.u);
    const int64_t pitch_vec = d / E;
    // warp-strided rows, the next row's 16-byte chunks loaded while the
    // current one is consumed; each row's dot with every query in its mask,
    // arithmetic identical to recompute_fast (lane chunks lane + 32c, fmaf in
    // element order, fixed butterfly). Rows fit one pass: d * sizeof(T) <= 4096.
    constexpr int CH = 8;
    auto load_row = [&](int idx, uint4 (&v)[CH]) {
      const uint4* rp = reinterpret_cast<const uint4*>(U_) + static_cast<int64_t>(f_row + s_rows[idx]) * pitch_vec;
#pragma unroll
      for (int c = 0; c < CH; ++c) {
        const int vi = lane + 32 * c;
        v[c] = vi < pitch_vec ? ldg_stream(rp + vi) : make_uint4(0, 0, 0, 0);
      }
    };
    uint4 cur[CH];
    if (wid < nrow) load_row(wid, cur);
    for (int idx = wid; idx < nrow; idx += kFusedWarps) {
      uint4 nxt[CH];
      if (idx + kFusedWarps < nrow) load_row(idx + kFusedWarps, nxt);
      const int rr = s_rows[idx];
      unsigned bits = s_mask[rr];
      while (bits) {
        const int qb = __ffs(bits) - 1;
        bits &= bits - 1;
        float acc = 0.0f;
#pragma unroll
        for (int c = 0; c < CH; ++c) {
          const int vi = lane + 32 * c;
          if (vi < pitch_vec) {
            float f[E], xv[E];
            Vec16<T>::expand(cur[c], f);
            if constexpr (E == 8) {
              const float4 xa = *reinterpret_cast<const float4*>(s_xf + qb * d + vi * 4);
              const float4 xb = *reinterpret_cast<const float4*>(s_xf + qb * d + (d >> 1) + vi * 4);
              xv[0] = xa.x; xv[1] = xa.y; xv[2] = xa.z; xv[3] = xa.w;
              xv[4 % E] = xb.x; xv[5 % E] = xb.y; xv[6 % E] = xb.z; xv[7 % E] = xb.w;
            } else {
              load_x_vec<E>(s_xf + qb * d + vi * E, xv);
            }
#pragma unroll
            for (int e = 0; e < E; ++e) acc = fmaf(f[e], xv[e], acc);
          }
        }
        acc = warp_sum_f32(acc);
        if (lane == 0) {
          const int j2 = atomicAdd(&s_nb[qb], 1);
          s_key[qb * w_row + j2] = make_key(apply_phi(a.phi, acc), static_cast<uint32_t>(f_row + rr));
        }
      }
#pragma unroll
      for (int c = 0; c < CH; ++c) cur[c] = nxt[c];
    }
    __syncthreads();
    if (a.trace && tid == 0) {
      const unsigned long long now = static_cast<unsigned long long>(globaltimer());
      atomicMax(reinterpret_cast<unsigned long long*>(a.trace + 38), now);
      // per-CTA dot-phase duration (ns) and row count, packed: max over CTAs
      atomicMax(reinterpret_cast<unsigned long long*>(a.trace + 40), ((now - static_cast<unsigned long long>(p3_t0)) << 16) | nrow);
      atomicAdd(reinterpret_cast<unsigned long long*>(a.trace + 41), now - static_cast<unsigned long long>(p3_t0));
    }
    for (int t2 = tid; t2 < B * w_row; t2 += kFusedThreads) {
      const int qb = t2 / w_row, j2 = t2 % w_row;
      if (j2 < s_nb[qb]) a.pairs[(static_cast<int64_t>(qb) * G + blockIdx.x) * a.wmax + j2] = s_key[t2];
    }
    if (tid < B) a.pcnt[tid * G + blockIdx.x] = s_nb[tid];
    const int ntask = nrow;
    if (a.trace && tid == 0) {
      atomicMax(reinterpret_cast<unsigned long long*>(a.trace + 22), static_cast<unsigned long long>(globaltimer()));
      atomicMax(reinterpret_cast<unsigned long long*>(a.trace + 24), static_cast<unsigned long long>(ntask));
    }
  }
  cta_arrive(a.counters + kCntPairs, 1);

  // ---- P4: top-k by exact activation, emitted in ascending unit order ----
  if (blockIdx.x < B) {
    const int b = blockIdx.x;
    cta_wait_geq(a.counters + kCntPairs, G);
    FUSED_STAMP(7);
    unsigned* s_bits = reinterpret_cast<unsigned*>(s_pool);
    const int nwords = (m + 31) / 32;
    float* s_au = reinterpret_cast<float*>(s_bits + nwords);
    unsigned* s_pre = reinterpret_cast<unsigned*>(s_au + m);  // [G] slot prefix
    unsigned char* s_seg = reinterpret_cast<unsigned char*>(s_pre + G);  // [k'] slot of pair i
    for (int w = tid; w < nwords; w += kFusedThreads) s_bits[w] = 0u;
    int tot2 = 0;
    {
      const int c = tid;
      const int v = c < G ? __ldcg(a.pcnt + b * G + c) : 0;
      const int ex2 = block_exclusive_scan<kFusedThreads>(v, sc.scan, &tot2);
      if (c < G) {
        s_pre[c] = static_cast<unsigned>(ex2);
        for (int j = 0; j < v; ++j) s_seg[ex2 + j] = static_cast<unsigned char>(c);
      }
    }
    __syncthreads();
    // the order statistic runs on 4 warps (per-pass overhead scales with the
    // warp count): 128 threads x KP pairs (k' <= 1024 here)
    constexpr int KP = 8, NTS = 128;
    RegKeys<KP> src;
#pragma unroll
    for (int j = 0; j < KP; ++j) {
      const int i = tid + j * NTS;
      uint64_t kk = 0;
      if (tid < NTS && i < tot2) {
        const int sg = s_seg[i];
        kk = __ldcg(reinterpret_cast<const unsigned long long*>(a.pairs) +
                    (static_cast<int64_t>(b) * G + sg) * a.wmax + (i - s_pre[sg]));
      }
      src.k[j] = kk;
    }
    FUSED_STAMP(25);
    __shared__ uint64_t s_T2;
    if (tid < NTS) {
      const uint64_t t2 = block_range_select<NTS>(src, tot2, min(a.k, tot2), &rs2);
      if (tid == 0) s_T2 = t2;
    }
    __syncthreads();
    const uint64_t T2 = s_T2;
    FUSED_STAMP(26);
#pragma unroll
    for (int j = 0; j < KP; ++j) {
      const uint64_t key = src.k[j];
      if (key && key >= T2) {
        const uint32_t u = key_index(key);
        atomicOr(&s_bits[u >> 5], 1u << (u & 31));
        s_au[u] = key_value(key);
      }
    }
    __syncthreads();
    // ordered emit: thread t owns words [t*per, (t+1)*per)
    const int per = (nwords + kFusedThreads - 1) / kFusedThreads;
    const int w0 = min(nwords, tid * per), w1 = min(nwords, w0 + per);
    int cnt = 0;
    for (int w = w0; w < w1; ++w) cnt += __popc(s_bits[w]);
    int total;
    int pos = block_exclusive_scan<kFusedThreads>(cnt, sc.scan, &total);
    for (int w = w0; w < w1; ++w) {
      unsigned bits = s_bits[w];
      while (bits) {
        const int bit = __ffs(bits) - 1;
        bits &= bits - 1;
        const int u = w * 32 + bit;
        a.sel[static_cast<int64_t>(b) * a.k + pos] = static_cast<uint32_t>(u);
        a.selact[static_cast<int64_t>(b) * a.k + pos] = s_au[u];
        ++pos;
      }
    }
    FUSED_STAMP(27);
    cta_arrive(a.counters + kCntSel, 1);
  }

  // ---- P5: down-projection partial sums -----------------------------------
  FUSED_STAMP(8);
  cta_wait_geq(a.counters + kCntSel, B);
  FUSED_STAMP(9);
  const int nch = (a.k + kFusedCh - 1) / kFusedCh;
  {
    const T* V_ = static_cast<const T*>(a.v);
    const int64_t pitch_vec = d / E;
    const int half = tid >> 8, htid = tid & 255;  // two 256-thread workers per CTA
    const int tasks = B * nch;
    for (int task = half * G + blockIdx.x; task < tasks; task += G * 2) {
      const int b = task / nch, c = task % nch;
      const int lo = c * kFusedCh, hi = min(a.k, lo + kFusedCh);
      float* pout = a.partial + (static_cast<int64_t>(b) * nch + c) * d;
      for (int col0 = htid; col0 < pitch_vec; col0 += 256) {
        float accv[E];
#pragma unroll
        for (int e = 0; e < E; ++e) accv[e] = 0.0f;
        uint4 uq[kFusedCh];
        float aq[kFusedCh];
#pragma unroll
        for (int q = 0; q < kFusedCh; ++q) {
          if (lo + q < hi) {
            const int64_t row = __ldcg(a.sel + static_cast<int64_t>(b) * a.k + lo + q);
            aq[q] = __ldcg(a.selact + static_cast<int64_t>(b) * a.k + lo + q);
            uq[q] = ldg_stream(reinterpret_cast<const uint4*>(V_) + row * pitch_vec + col0);
          }
        }
        // same association as ffn_down_partial: groups of 4 units, then tail
#pragma unroll
        for (int q = 0; q < kFusedCh; ++q) {
          if (lo + q < hi) {
            float f[E];
            Vec16<T>::expand(uq[q], f);
#pragma unroll
            for (int e = 0; e < E; ++e) accv[e] = fmaf(aq[q], f[e], accv[e]);
          }
        }
#pragma unroll
        for (int e = 0; e < E; ++e) pout[col0 * E + e] = accv[e];
      }
    }
  }
  if (a.trace && tid == 0) atomicMax(reinterpret_cast<unsigned long long*>(a.trace + 31), static_cast<unsigned long long>(globaltimer()));
  cta_arrive(a.counters + kCntDown, 1);

  // ---- P6: fixed-order reduction over chunks ------------------------------
  FUSED_STAMP(10);
  cta_wait_geq(a.counters + kCntDown, G);
  FUSED_STAMP(11);
  for (int id = blockIdx.x * kFusedThreads + tid; id < B * d; id += G * kFusedThreads) {
    const int b = id / d, col = id % d;
    const float* p = a.partial + static_cast<int64_t>(b) * nch * d + col;
    float s = 0.0f;
    for (int c = 0; c < nch; ++c) s = __fadd_rn(s, __ldcg(p + static_cast<int64_t>(c) * d));
    a.out[id] = s;
  }

  // ---- exit: last CTA resets the hand-off counters -------------------------
  FUSED_STAMP(12);
  if (a.trace && blockIdx.x == 0 && threadIdx.x == 0) a.trace[21] = clock64();
  __syncthreads();
  if (tid == 0) {
    // two-level exit count: the CTA completing its group arrives at the top
    // counter; the one completing the top resets every counter
    __threadfence();
    const int grp = blockIdx.x % kSpread;
    const int members = (G - grp + kSpread - 1) / kSpread;
    const int prev = atomicAdd(a.counters + kCntExit + grp * 32, 1);
    if (prev == members - 1) {
      const int ngrp = G < kSpread ? G : kSpread;
      if (atomicAdd(a.counters + kCntExit + kSpread * 32 - 8, 1) == ngrp - 1) {
        for (int i = 0; i < kCntInts; i += 32) a.counters[i] = 0;
        a.counters[kCntExit + kSpread * 32 - 8] = 0;
        __threadfence();
      }
    }
  }
}

}  // namespace hire_dev
