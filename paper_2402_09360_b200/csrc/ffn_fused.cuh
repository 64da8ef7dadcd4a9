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
  uint32_t* cand;          // [B][kp]
  float* act;              // [B][kp]
  uint32_t* sel;           // [B][k]   (out, ascending)
  float* selact;           // [B][k]
  float* partial;          // [B][nch][d]
  float* out;              // [B][d]
  int* counters;           // [8] zeroed between launches
  long long* trace;        // optional [16] %globaltimer stamps (CTA 0, thread 0)
};

__device__ __forceinline__ long long globaltimer() {
  long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

enum { kCntGemv = 0, kCntCand = 32, kCntAct = 64, kCntSel = 96, kCntDown = 128, kCntExit = 160 };  // one 128-B line each

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// One poller per CTA with exponential backoff: 148 SMs spinning on one line
// at ~64 ns would saturate its L2 slice and stall every other access that
// maps there (measured: a 4 KB row gather taking 8.5 us).
__device__ __forceinline__ void cta_wait_geq(const int* p, int target) {
  if (threadIdx.x == 0) {
    unsigned ns = 32;
    while (ld_acquire(p) < target) {
      __nanosleep(ns);
      ns = ns < 1024 ? ns * 2 : 1024;
    }
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
  // all warps work on every query: max|x| (block reduce), sx = max/127,
  // xq = RHAZ(x/sx), sum(xq) (block reduce)
  block_copy(s_xf, a.x, B * d);
  __syncthreads();
  for (int b = 0; b < B; ++b) {
    float mx = 0.0f;
    for (int i = tid; i < d; i += kFusedThreads) mx = fmaxf(mx, fabsf(s_xf[b * d + i]));
    mx = warp_max_f32(mx);
    if (lane == 0) s_red[wid] = mx;
    __syncthreads();
    float v = 0.0f;
#pragma unroll
    for (int w = 0; w < kFusedWarps; ++w) v = fmaxf(v, s_red[w]);
    const float sx = v > 0.0f ? __fdiv_rn(v, 127.0f) : 1.0f;
    int local = 0;
    for (int i = tid; i < d; i += kFusedThreads) {
      const int q = rhaz_clamp(__fdiv_rn(s_xf[b * d + i], sx), 127);
      local += q;
      s_xq[b * xs + i] = static_cast<int8_t>(q);
    }
    local = warp_sum_i32(local);
    __syncthreads();  // s_red reuse
    if (lane == 0) s_redi[wid] = local;
    if (tid == 0) s_sx[b] = sx;
    __syncthreads();
    if (tid == 0) {
      int sum = 0;
      for (int w = 0; w < kFusedWarps; ++w) sum += s_redi[w];
      s_sum[b] = sum;
    }
  }
  for (int i = tid; i < (NT * 8 - B) * d; i += kFusedThreads) s_xq[(B + i / d) * xs + i % d] = 0;
  __syncthreads();
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

  // ---- P2: candidate selection, one CTA per query ------------------------
  if (blockIdx.x < B) {
    const int b = blockIdx.x;
    cta_wait_geq(a.counters + kCntGemv, G);
    FUSED_STAMP(3);
    float* s_val = reinterpret_cast<float*>(s_pool);
    block_copy_cg(s_val, a.scores + static_cast<int64_t>(b) * m, m);
    __syncthreads();
    FUSED_STAMP(13);
    uint64_t prefix, mask;
    auto key_at = [&](int i) { return make_key(s_val[i], static_cast<uint32_t>(i)); };
    block_select_kth<kFusedThreads>(key_at, m, a.kp, &sc, &prefix, &mask);
    FUSED_STAMP(14);
    uint32_t* cb = a.cand + static_cast<int64_t>(b) * a.kp;
    block_compact<kFusedThreads>(key_at, m, prefix, mask, &sc,
                                 [&](int pos, int i, uint64_t) { cb[pos] = static_cast<uint32_t>(i); });
    FUSED_STAMP(15);
    cta_arrive(a.counters + kCntCand, 1);
  }

  // ---- P3: exact activations of the B*k' candidates ---------------------
  FUSED_STAMP(4);
  cta_wait_geq(a.counters + kCntCand, B);
  FUSED_STAMP(5);
  {
    const T* U_ = static_cast<const T*>(a.u);
    const int64_t pitch_vec = d / E;
    const int tasks = B * a.kp;
    const int stride = G * kFusedWarps;
    // two rows in flight per warp; per-row arithmetic identical to recompute_fast
    // CTA-minor task order: consecutive tasks land on different SMs, so a
    // small B*k' spreads over all SMs (x is re-read from smem per row)
    const int tbase = wid * G + blockIdx.x;
    for (int t0 = tbase; t0 < tasks; t0 += 2 * stride) {
      int bt[2], it[2];
      bool ok[2];
      const uint4* rp[2];
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        const int task = t0 + r * stride;
        ok[r] = task < tasks;
        bt[r] = ok[r] ? task / a.kp : 0;
        it[r] = ok[r] ? task % a.kp : 0;
        const int64_t row = ok[r] ? __ldcg(a.cand + static_cast<int64_t>(bt[r]) * a.kp + it[r]) : 0;
        rp[r] = reinterpret_cast<const uint4*>(U_) + row * pitch_vec;
      }
      if (t0 == tbase) FUSED_STAMP(16);
      long long c_a = clock64();
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
        if (a.trace && blockIdx.x == 0 && threadIdx.x == 0 && c0 == 0) {
          a.trace[22] = clock64() - c_a;
          a.trace[23] = static_cast<long long>(vv[0][0].x ^ vv[0][7].w);  // forces the loads
          a.trace[24] = clock64() - c_a;
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
      if (t0 == tbase) FUSED_STAMP(17);
      if (a.trace && blockIdx.x == 0 && threadIdx.x == 0 && t0 == tbase) a.trace[25] = clock64() - c_a;
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        const float s2 = warp_sum_f32(accf[r]);
        if (lane == 0 && ok[r]) a.act[static_cast<int64_t>(bt[r]) * a.kp + it[r]] = apply_phi(a.phi, s2);
      }
    }
  }
  FUSED_STAMP(18);
  cta_arrive(a.counters + kCntAct, 1);
  FUSED_STAMP(19);

  // ---- P4: final top-k per query, ascending unit order --------------------
  if (blockIdx.x < B) {
    const int b = blockIdx.x;
    FUSED_STAMP(6);
    cta_wait_geq(a.counters + kCntAct, G);
    FUSED_STAMP(7);
    uint64_t* s_keys = reinterpret_cast<uint64_t*>(s_pool);
    block_copy_tf(s_keys, a.kp, [&](int i) {
      return make_key(__ldcg(a.act + static_cast<int64_t>(b) * a.kp + i),
                      __ldcg(a.cand + static_cast<int64_t>(b) * a.kp + i));
    });
    __syncthreads();
    uint64_t prefix, mask;
    auto key_at = [&](int i) { return s_keys[i]; };
    block_select_kth<kFusedThreads>(key_at, a.kp, a.k, &sc, &prefix, &mask);
    block_compact<kFusedThreads>(key_at, a.kp, prefix, mask, &sc, [&](int pos, int, uint64_t key) {
      a.sel[static_cast<int64_t>(b) * a.k + pos] = key_index(key);
      a.selact[static_cast<int64_t>(b) * a.k + pos] = key_value(key);
    });
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
      __threadfence();
    }
  }
}

}  // namespace hire_dev
