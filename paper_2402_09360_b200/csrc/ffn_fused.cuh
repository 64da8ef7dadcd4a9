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
  int* qcnt;               // [B][4] above / window / pairs counts (zeroed per launch)
  uint64_t* win;           // [B][wcap] bracket windows
  int wcap;
  uint64_t* pairs;         // [B][kp] (exact activation, unit) keys of the candidates
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

enum { kCntGemv = 0, kCntPiv = 32, kCntWin = 64, kCntThr = 96, kCntPairs = 128, kCntSel = 160, kCntDown = 192,
       kCntExit = 224 };  // one 128-B line each

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// One poller per CTA: relaxed probes (an acquire probe invalidates the
// SM's L1 every time), one acquire fence once the target is reached.
__device__ __forceinline__ void cta_wait_geq(const int* p, int target) {
  if (threadIdx.x == 0) {
    while (static_cast<int>(ld_relaxed_gpu(reinterpret_cast<const unsigned*>(p))) < target) {
    }
    fence_acq_rel_gpu();
  }
  __syncthreads();
}

// every thread fences its own writes, then one arrival per CTA
__device__ __forceinline__ void cta_arrive(int* p, int inc) {
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) atomicAdd(p, inc);
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
  __shared__ SelectScratch sc;

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
  block_copy(s_xf, a.x, B * d);
  __syncthreads();
  FUSED_STAMP(13);
  {
    const int wpq = kFusedWarps / B > 0 ? kFusedWarps / B : 1;  // warps per query
    const int qb = wid / wpq, qw = wid % wpq;                     // my query, my rank in it
    const bool active = qb < B;
    float mx = 0.0f;
    if (active)
      for (int i = qw * 32 + lane; i < d; i += wpq * 32) mx = fmaxf(mx, fabsf(s_xf[qb * d + i]));
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
        const int q = rhaz_clamp(__fdiv_rn(s_xf[qb * d + i], sx), 127);
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
  cta_arrive(a.counters + kCntGemv, 1);

  // ---- P2a: bracket pivots for the k'-th proxy key (CTA b per query) ------
  // A 128-key sample of scores[b] ranked by counting; the sample keys at
  // ranks (k'-1)S/m -/+ 3.5 sigma bracket the k'-th key (select.cuh).
  int f_row, w_row;  // this CTA's row slice (width rule)
  {
    const int base = m / G, extra = m % G;
    f_row = blockIdx.x * base + (blockIdx.x < extra ? blockIdx.x : extra);
    w_row = base + (blockIdx.x < extra ? 1 : 0);
  }
  if (blockIdx.x < B) {
    const int b = blockIdx.x;
    cta_wait_geq(a.counters + kCntGemv, G);
    FUSED_STAMP(3);
    constexpr int S = 128;
    if (tid < S) {
      const int i = static_cast<int>((static_cast<int64_t>(tid) * m) / S);
      sc.samp[tid] = make_key(__ldcg(a.scores + static_cast<int64_t>(b) * m + i), static_cast<uint32_t>(i));
    }
    if (tid == 0) {
      sc.piv[0] = ~0ull;
      sc.piv[1] = 0ull;
    }
    __syncthreads();
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
      a.piv[2 * b] = sc.piv[0];
      a.piv[2 * b + 1] = sc.piv[1];
    }
    cta_arrive(a.counters + kCntPiv, 1);
  }

  // ---- P2b: every CTA counts / gathers the bracket over its own rows ------
  // query-aligned warp groups (wpq warps per query) walk the slice; ballot
  // counts go to per-query shared counters; one global atomic per query.
  cta_wait_geq(a.counters + kCntPiv, B);
  FUSED_STAMP(4);
  {
    __shared__ int s_above[16], s_win[16], s_wbase[16];
    uint64_t* s_stage = reinterpret_cast<uint64_t*>(s_pool);  // [B][w_row]
    if (tid < B) s_above[tid] = s_win[tid] = 0;
    __syncthreads();
    const int wpq = kFusedWarps / B > 0 ? kFusedWarps / B : 1;
    const int qb = wid / wpq, qw = wid % wpq;
    if (qb < B) {
      const uint64_t hi = __ldcg(a.piv + 2 * qb), lo = __ldcg(a.piv + 2 * qb + 1);
      for (int r0 = qw * 32; r0 < w_row; r0 += wpq * 32) {
        const int r = r0 + lane;
        uint64_t key = 0;
        bool above = false, in = false;
        if (r < w_row) {
          key = make_key(__ldcg(a.scores + static_cast<int64_t>(qb) * m + f_row + r), static_cast<uint32_t>(f_row + r));
          above = key > hi;
          in = key > lo && key <= hi;
        }
        const unsigned ba = __ballot_sync(0xffffffffu, above), bi = __ballot_sync(0xffffffffu, in);
        int base = 0;
        if (lane == 0) {
          if (ba) atomicAdd(&s_above[qb], __popc(ba));
          if (bi) base = atomicAdd(&s_win[qb], __popc(bi));
        }
        base = __shfl_sync(0xffffffffu, base, 0);
        if (in) s_stage[qb * w_row + base + __popc(bi & ((1u << lane) - 1u))] = key;
      }
    }
    __syncthreads();
    if (tid < B) {
      if (s_above[tid]) atomicAdd(a.qcnt + 4 * tid, s_above[tid]);
      s_wbase[tid] = s_win[tid] ? atomicAdd(a.qcnt + 4 * tid + 1, s_win[tid]) : 0;
    }
    __syncthreads();
    for (int t2 = tid; t2 < B * w_row; t2 += kFusedThreads) {
      const int b = t2 / w_row, j2 = t2 % w_row;
      if (j2 < s_win[b] && s_wbase[b] + j2 < a.wcap)
        a.win[static_cast<int64_t>(b) * a.wcap + s_wbase[b] + j2] = s_stage[t2];
    }
  }
  cta_arrive(a.counters + kCntWin, 1);

  // ---- P2c: exact k'-th key per query from its window (CTA b) -------------
  if (blockIdx.x < B) {
    const int b = blockIdx.x;
    cta_wait_geq(a.counters + kCntWin, G);
    FUSED_STAMP(5);
    const int above = __ldcg(a.qcnt + 4 * b), nw = __ldcg(a.qcnt + 4 * b + 1);
    const int need = a.kp - above;
    uint64_t T;
    if (need >= 1 && need <= nw && nw <= a.wcap) {
      uint64_t* s_w = reinterpret_cast<uint64_t*>(s_pool);
      block_copy_cg(s_w, a.win + static_cast<int64_t>(b) * a.wcap, nw);
      __syncthreads();
      T = block_kth_key<kFusedThreads>([&](int i) { return s_w[i]; }, nw, need, &sc);
    } else {  // bracket missed: exact select over all m scores
      float* s_val = reinterpret_cast<float*>(s_pool);
      block_copy_cg(s_val, a.scores + static_cast<int64_t>(b) * m, m);
      __syncthreads();
      T = block_kth_key<kFusedThreads>([&](int i) { return make_key(s_val[i], static_cast<uint32_t>(i)); },
                                       m, a.kp, &sc);
    }
    if (tid == 0) a.thr[b] = T;
    cta_arrive(a.counters + kCntThr, 1);
  }

  // ---- P3: every CTA recomputes the candidates in its own rows ------------
  cta_wait_geq(a.counters + kCntThr, B);
  FUSED_STAMP(6);
  {
    // stage (b, row) candidates of this slice, query-major
    int* s_cand = reinterpret_cast<int*>(s_pool);                    // [B*w_row] rows
    float* s_act = reinterpret_cast<float*>(s_pool) + B * w_row;      // [B*w_row]
    __shared__ int s_off[17];
    __shared__ int s_nb[16];
    __shared__ int s_pbase[16];
    if (tid < B) s_nb[tid] = 0;
    __syncthreads();
    {
      const int wpq = kFusedWarps / B > 0 ? kFusedWarps / B : 1;
      const int qb = wid / wpq, qw = wid % wpq;
      if (qb < B) {
        const uint64_t T = __ldcg(a.thr + qb);
        for (int r0 = qw * 32; r0 < w_row; r0 += wpq * 32) {
          const int r = r0 + lane;
          bool c = false;
          if (r < w_row)
            c = make_key(__ldcg(a.scores + static_cast<int64_t>(qb) * m + f_row + r), static_cast<uint32_t>(f_row + r)) >= T;
          const unsigned bc = __ballot_sync(0xffffffffu, c);
          int base = 0;
          if (lane == 0 && bc) base = atomicAdd(&s_nb[qb], __popc(bc));
          base = __shfl_sync(0xffffffffu, base, 0);
          if (c) s_cand[qb * w_row + base + __popc(bc & ((1u << lane) - 1u))] = f_row + r;
        }
      }
    }
    __syncthreads();
    if (tid == 0) {
      s_off[0] = 0;
      for (int b = 0; b < B; ++b) s_off[b + 1] = s_off[b] + s_nb[b];
    }
    __syncthreads();
    const int ntask = s_off[B];
    const T* U_ = static_cast<const T*>(a.u);
    const int64_t pitch_vec = d / E;
    // two rows in flight per warp; per-row arithmetic identical to recompute_fast
    for (int t0 = wid; t0 < ntask; t0 += 2 * kFusedWarps) {
      int bt[2], rw[2], slot[2];
      bool ok[2];
      const uint4* rp[2];
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        const int task = t0 + r * kFusedWarps;
        ok[r] = task < ntask;
        int b = 0;
        if (ok[r])
          while (task >= s_off[b + 1]) ++b;
        bt[r] = b;
        slot[r] = ok[r] ? b * w_row + (task - s_off[b]) : 0;
        rw[r] = ok[r] ? s_cand[slot[r]] : 0;
        rp[r] = reinterpret_cast<const uint4*>(U_) + static_cast<int64_t>(rw[r]) * pitch_vec;
      }
      float accf[2] = {0.0f, 0.0f};
      for (int c0 = 0; c0 < pitch_vec; c0 += 256) {  // 8 vectors per lane per pass
        uint4 vv[2][8];
#pragma unroll
        for (int r = 0; r < 2; ++r)
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            const int vi = c0 + lane + 32 * c;
            vv[r][c] = (ok[r] && vi < pitch_vec) ? ldg_stream(rp[r] + vi) : make_uint4(0, 0, 0, 0);
          }
#pragma unroll
        for (int r = 0; r < 2; ++r)
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            const int vi = c0 + lane + 32 * c;
            if (vi < pitch_vec) {
              float f[E], xv[E];
              Vec16<T>::expand(vv[r][c], f);
              load_x_vec<E>(s_xf + bt[r] * d + vi * E, xv);
#pragma unroll
              for (int e = 0; e < E; ++e) accf[r] = fmaf(f[e], xv[e], accf[r]);
            }
          }
      }
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        const float s2 = warp_sum_f32(accf[r]);
        if (lane == 0 && ok[r]) s_act[slot[r]] = apply_phi(a.phi, s2);
      }
    }
    __syncthreads();
    if (tid < B) s_pbase[tid] = s_nb[tid] ? atomicAdd(a.qcnt + 4 * tid + 2, s_nb[tid]) : 0;
    __syncthreads();
    for (int task = tid; task < ntask; task += kFusedThreads) {
      int b = 0;
      while (task >= s_off[b + 1]) ++b;
      const int j2 = task - s_off[b];
      const int sl = b * w_row + j2;
      a.pairs[static_cast<int64_t>(b) * a.kp + s_pbase[b] + j2] = make_key(s_act[sl], static_cast<uint32_t>(s_cand[sl]));
    }
  }
  cta_arrive(a.counters + kCntPairs, 1);

  // ---- P4: top-k by exact activation, emitted in ascending unit order ----
  if (blockIdx.x < B) {
    const int b = blockIdx.x;
    cta_wait_geq(a.counters + kCntPairs, G);
    FUSED_STAMP(7);
    uint64_t* s_keys = reinterpret_cast<uint64_t*>(s_pool);
    unsigned* s_bits = reinterpret_cast<unsigned*>(s_keys + a.kp);
    const int nwords = (m + 31) / 32;
    float* s_au = reinterpret_cast<float*>(s_bits + nwords);
    block_copy_cg(s_keys, a.pairs + static_cast<int64_t>(b) * a.kp, a.kp);
    for (int w = tid; w < nwords; w += kFusedThreads) s_bits[w] = 0u;
    __syncthreads();
    const uint64_t T2 = block_kth_key<kFusedThreads>([&](int i) { return s_keys[i]; }, a.kp, a.k, &sc);
    for (int i = tid; i < a.kp; i += kFusedThreads) {
      const uint64_t key = s_keys[i];
      if (key >= T2) {
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
    __threadfence();
    const int prev = atomicAdd(a.counters + kCntExit, 1);
    if (prev == G - 1) {
      for (int i = 0; i <= kCntExit; i += 32) a.counters[i] = 0;
      for (int i = 0; i < 4 * B; ++i) a.qcnt[i] = 0;
      __threadfence();
    }
  }
}

}  // namespace hire_dev
