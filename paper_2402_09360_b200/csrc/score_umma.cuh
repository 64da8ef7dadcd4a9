// score_umma.cuh — K1 for batches of 9..64 queries on the 5th-generation
// tensor cores: the int4 proxy GEMV becomes a skinny GEMM
//   S[row][q] = sum_k code[row][k] * xq[q][k]          (exact int32)
// with the vocab rows as the MMA's M (128 per tcgen05.mma), the queries as
// N (16/32/48/64) and K = d. Reference op: the int4 scorer,
// approx.hpp:395-403, in BASELINE's int8-x integer mode (DESIGN.md
// "Semantics"): score = phi(float(S - 8 * sum(xq)) * (scale * sx)).
//
// Data path per CTA (persistent, one CTA per SM, rows in 128-row blocks):
//   HBM --TMA (cp.async.bulk.tensor.2d, 16 KB stages, mbarrier ring)--> smem
//   smem --4 converter warps: LDS.128, int4 digits -> u8 in registers,
//          tcgen05.st--> TMEM (the A operand: lane = row, 4 codes per column)
//   TMEM A x smem x (B operand, int8, resident) --tcgen05.mma kind::i8,
//          one elected thread--> TMEM accumulators (s32, 2 buffers)
//   TMEM --tcgen05.ld, epilogue (scale, phi)--> scores [B][rows]
// The int4 codes are stored in a tensor-core layout built once per scorer
// (q4_to_umma_layout): [row block][k chunk of 32][row 128][16 B], byte
// 4j+b = (code[8j+b] + 8) | (code[8j+4+b] + 8) << 4, so the two nibble masks
// of one 32-bit word give 8 consecutive k in natural order (unsigned digits
// c + 8; the 8 * sum(xq) correction makes the sum exact).
#pragma once
#include <cuda.h>
#include <cstdint>

#include "common.cuh"
#include "umma.cuh"

namespace hire_dev {

constexpr int kUmmaRows = 128;         // rows per MMA / per row block
constexpr int kUmmaStageChunks = 8;    // k chunks (32 codes each) per pipeline stage
constexpr int kUmmaStageBytes = kUmmaStageChunks * kUmmaRows * 16;  // 16 KB
constexpr int kUmmaStages = 4;         // smem ring depth
constexpr int kUmmaABufs = 4;          // TMEM A-operand stage buffers (64 columns each)
#ifndef HIRE_UMMA_CONV_GROUPS
#define HIRE_UMMA_CONV_GROUPS 3
#endif
#ifndef HIRE_UMMA_EPI_GROUPS
#define HIRE_UMMA_EPI_GROUPS 2
#endif
// converter warpgroups; group g converts chunks [g*8/G, (g+1)*8/G) of every stage
constexpr int kUmmaConvGroups = HIRE_UMMA_CONV_GROUPS;
constexpr int kUmmaConvWarps = 4 * kUmmaConvGroups;
constexpr int kUmmaEpiGroups = HIRE_UMMA_EPI_GROUPS;    // epilogue warpgroups, alternate row blocks
constexpr int kUmmaEpiWarp = kUmmaConvWarps;            // warps +0..+4E-1: epilogue
constexpr int kUmmaTmaWarp = kUmmaEpiWarp + 4 * kUmmaEpiGroups;  // TMA producer
constexpr int kUmmaMmaWarp = kUmmaTmaWarp + 1;          // MMA issuers (+0..+3; +0 allocates TMEM)
constexpr int kUmmaMaxIssuers = 4;
constexpr int kUmmaThreads = 32 * (kUmmaMmaWarp + kUmmaMaxIssuers);
static_assert(kUmmaEpiGroups == 1 || kUmmaEpiGroups == 2, "one accumulator pair per epilogue group");
// One thread issues a tcgen05.mma about every 78 cycles whatever N is
// (tools/probes/probe_umma_rate.cu), far from the tensor floor at N <= 32
// (16 cycles): n_iss issuer warps each own whole stages (st % n_iss) and an
// accumulator of their own; the epilogue adds the n_iss partial sums (exact
// int32). n_iss divides the stages per row block, and 4 A buffers + n_iss x 2
// accumulators of nq columns fit the 512 TMEM columns.
__host__ __device__ inline int umma_issuers(int nq, int d) {
  const int n_st = d / 32 / kUmmaStageChunks;
  for (int n = kUmmaMaxIssuers; n > 1; n >>= 1)
    if (n_st % n == 0 && 64 * kUmmaABufs + n * 2 * nq <= 512) return n;
  return 1;
}

// canonical [rows][pitch] (low nibble = even column) -> UMMA layout words
__global__ void q4_to_umma_layout(const uint8_t* __restrict__ wq, int64_t pitch, int64_t rows, int d,
                                  uint32_t* __restrict__ out, int64_t n_words) {
  hire_dev::griddep_wait();  // no early trigger: consumers prefetch this layout before their wait
  const int64_t id = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (id >= n_words) return;
  const int nkc = d / 32;
  const int j = static_cast<int>(id & 3);
  const int r = static_cast<int>((id >> 2) & 127);
  const int64_t blk = id >> 9;  // (row block, k chunk)
  const int64_t rb = blk / nkc, kc = blk % nkc;
  const int64_t row = rb * kUmmaRows + r;
  uint32_t word = 0x88888888u;  // padding rows: code 0
  if (row < rows) {
    word = 0;
#pragma unroll
    for (int b = 0; b < 4; ++b)
#pragma unroll
      for (int hi = 0; hi < 2; ++hi) {
        const int64_t col = kc * 32 + 8 * j + 4 * hi + b;
        const uint8_t byte = wq[row * pitch + col / 2];
        const uint32_t nib = ((col & 1) ? (byte >> 4) : (byte & 0xF)) ^ 0x8u;  // code + 8
        word |= nib << (8 * b + 4 * hi);
      }
  }
  out[id] = word;
}

constexpr int kUmmaMaxStages = 12;

// shared memory: ring of int4 stages, the x operand, barriers
struct UmmaSmem {
  static __host__ __device__ size_t x_off(int stages) { return static_cast<size_t>(stages) * kUmmaStageBytes; }
  static __host__ __device__ size_t bar_off(int stages, int nq, int d) {
    return x_off(stages) + static_cast<size_t>(nq) * d;
  }
  static __host__ __device__ size_t bytes(int stages, int nq, int d) {
    return qc_off(stages, nq, d) + 64 * 8;
  }
  // per-query epilogue constants: float sx[64], int 8 * sum(xq)[64]
  static __host__ __device__ size_t qc_off(int stages, int nq, int d) {
    return (bar_off(stages, nq, d) + (2 * kUmmaMaxStages + 2 * kUmmaABufs + 5) * 8 + 16 + 15) & ~static_cast<size_t>(15);
  }
  // deepest ring that fits next to an x operand of nq queries
  static __host__ int stages_for(int nq, int d, size_t smem_max) {
    int st = kUmmaMaxStages;
    while (st > 2 && bytes(st, nq, d) > smem_max) --st;
    return st;
  }
};

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::
          "r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
// L2 policies (HIRE_UMMA_L2 != 0): the weight stream is read once per call
// (evict first), the score rows are read again right away by the selector
// (evict last) — 263 MB of weights would otherwise push the 1 MB-per-query
// scores out of the 126 MB L2 before the selector reads them.
#ifndef HIRE_UMMA_L2
#define HIRE_UMMA_L2 1
#endif
__device__ __forceinline__ uint64_t l2_policy_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ uint64_t l2_policy_evict_normal() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ uint64_t l2_policy_evict_last() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void tma_load_2d_hint(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar,
                                                 uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, %3}], "
      "[%4], %5;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void st_hint_f32(float* p, float v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.f32 [%0], %1, %2;" ::"l"(p), "f"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ void tma_prefetch_desc(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

// x operand in global memory, written by prep_x_int8_kernel (mode 1) in the
// MMA's B layout so one bulk copy stages it: queries in groups of 8, each
// group a [d/16][8 queries][16 B] block (8-row x 16-byte core matrices),
// offset(n, k) = (n/8)*8d + (k/16)*128 + (n%8)*16 + k%16; padding queries 0.
__host__ __device__ __forceinline__ int64_t xg_offset(int64_t n, int64_t k, int64_t d) {
  return (n >> 3) * 8 * d + (k >> 4) * 128 + (n & 7) * 16 + (k & 15);
}

// nq: MMA N = queries rounded up to 16 (<= 64); nb <= nq real queries.
// Tensor map: 2-D u64 view [n_rb * nkc][256] of the UMMA layout (one k chunk
// of a row block = 256 x 8 B = 2 KB), box {256, kUmmaStageChunks}.
__global__ void __launch_bounds__(kUmmaThreads, 1) q4_score_umma(
    const __grid_constant__ CUtensorMap wmap, int64_t rows, int d, const float* __restrict__ scales,
    const int8_t* __restrict__ xg, const float* __restrict__ sx, const int* __restrict__ sumxq, int nb, int nq,
    int stages, int phi, float* __restrict__ scores, int64_t score_stride) {
  extern __shared__ __align__(1024) unsigned char smem[];
  KTrace kt_(kKtProxy);
  uint8_t* ring = smem;
  uint8_t* s_x = smem + UmmaSmem::x_off(stages);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + UmmaSmem::bar_off(stages, nq, d));
  uint64_t* full = bars;                          // [stages] TMA -> converters
  uint64_t* empty = bars + kUmmaMaxStages;        // [stages] converters -> TMA (128 arrivals)
  uint64_t* afull = bars + 2 * kUmmaMaxStages;    // [kUmmaABufs] converters -> MMA (128 arrivals)
  uint64_t* aempty = afull + kUmmaABufs;          // [kUmmaABufs] MMA commit -> converters
  uint64_t* dfull = aempty + kUmmaABufs;          // [2] MMA commit -> epilogue
  uint64_t* dempty = dfull + 2;                   // [2] epilogue -> MMA (128 arrivals)
  uint64_t* xbar = dempty + 2;                    // x operand bulk copy
  uint32_t* s_tmem = reinterpret_cast<uint32_t*>(xbar + 1);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nkc = d / 32, n_st = nkc / kUmmaStageChunks;
  const int64_t n_rb = (rows + kUmmaRows - 1) / kUmmaRows;
  constexpr uint32_t kTmemCols = 512;  // A: kUmmaABufs x 64 columns, D: n_iss x 2 x nq columns
  constexpr uint32_t kColA = 0, kColD = 64 * kUmmaABufs;
  const int n_iss = umma_issuers(nq, d);

  if (tid == 0) {
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 32 * kUmmaConvWarps);
    }
    for (int i = 0; i < kUmmaABufs; ++i) {
      mbar_init(&afull[i], 32 * kUmmaConvWarps);
      mbar_init(&aempty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&dfull[i], n_iss);
      mbar_init(&dempty[i], 128);
    }
    mbar_init(xbar, 1);
    fence_mbar_init();
  }
  if (warp == kUmmaTmaWarp && lane == 0) tma_prefetch_desc(&wmap);
  if (warp == kUmmaMmaWarp) {
    umma::tmem_alloc(s_tmem, kTmemCols);
    umma::tmem_relinquish();
  }
  umma::fence_before();
  __syncthreads();
  umma::fence_after();
  const uint32_t tmem = *s_tmem;

  if (warp == kUmmaTmaWarp) {
    // ===== TMA producer: weights are read-only, so it streams before the
    // programmatic-dependency wait (independent prologue)
    if (lane == 0) {
      const uint64_t pol_w = l2_policy_evict_first();
      (void)pol_w;
      int it = 0;
      for (int64_t rb = blockIdx.x; rb < n_rb; rb += gridDim.x)
        for (int st = 0; st < n_st; ++st, ++it) {
          const int slot = it % stages;
          if (it >= stages) mbar_wait(&empty[slot], ((it / stages) - 1) & 1);
          mbar_arrive_expect_tx(&full[slot], kUmmaStageBytes);
#if HIRE_UMMA_L2
          tma_load_2d_hint(ring + static_cast<size_t>(slot) * kUmmaStageBytes, &wmap, 0,
                           static_cast<int>(rb * nkc + st * kUmmaStageChunks), &full[slot], pol_w);
          continue;
#endif
          tma_load_2d(ring + static_cast<size_t>(slot) * kUmmaStageBytes, &wmap, 0,
                      static_cast<int>(rb * nkc + st * kUmmaStageChunks), &full[slot]);
        }
    }
  } else if (warp >= kUmmaMmaWarp) {
    // ===== MMA issuers: issuer j takes stages j, j + n_iss, ... of every
    // row block into its own accumulator pair (x operand: one bulk copy
    // after the programmatic-dependency wait, by issuer 0)
    const int j = warp - kUmmaMmaWarp;
    if (lane == 0 && j < n_iss) {
      griddep_wait();  // x quantisation (prep_x_int8_kernel) is complete
      if (j == 0) {
        const unsigned xbytes = static_cast<unsigned>(nq) * static_cast<unsigned>(d);
        mbar_arrive_expect_tx(xbar, xbytes);
        bulk_g2s(s_x, xg, xbytes, xbar);
      }
      const uint32_t idesc = umma::idesc_i8(kUmmaRows, nq, /*a_signed=*/false, /*b_signed=*/true);
      const uint32_t xbase = smem_u32(s_x);
      mbar_wait(xbar, 0);
      int rbi = 0;
      for (int64_t rb = blockIdx.x; rb < n_rb; rb += gridDim.x, ++rbi) {
        const int db = rbi & 1;
        if (rbi >= 2) mbar_wait(&dempty[db], ((rbi >> 1) - 1) & 1);
        umma::fence_after();
        const uint32_t dcol = tmem + kColD + static_cast<uint32_t>((2 * j + db) * nq);
        for (int st = j; st < n_st; st += n_iss) {
          const int ait = rbi * n_st + st;
          const int ab = ait % kUmmaABufs;
          mbar_wait(&afull[ab], (ait / kUmmaABufs) & 1);
          umma::fence_after();
          const uint32_t acol = tmem + kColA + ab * 64;
          // k chunk kc = core matrices 2kc, 2kc+1 (LBO 128 B apart); 8-query groups 8d apart
          const uint64_t bd0 = umma::sdesc_kmajor_noswz(xbase + static_cast<uint32_t>(st * kUmmaStageChunks * 256),
                                                        128, static_cast<uint32_t>(8 * d));
#pragma unroll
          for (int c = 0; c < kUmmaStageChunks; ++c)  // start address field: 16-byte units
            umma::mma_i8_ts(dcol, acol + 8 * c, bd0 + static_cast<uint64_t>(c * 16), idesc, (st != j) || (c != 0));
          umma::commit(&aempty[ab]);
        }
        umma::commit(&dfull[db]);
      }
    }
    __syncwarp();
  } else if (warp < kUmmaConvWarps) {
    // ===== converters (thread = TMEM lane = row within the block): int4
    // digits from the smem ring -> u8 -> the TMEM A-operand buffers. Warp w
    // may only touch TMEM lanes 32 (w % 4) ..; the kUmmaConvGroups
    // warpgroups split every stage's chunks so each SM sub-partition has
    // several converter warps to hide LDS / STTM latency.
    constexpr int kCpg = (kUmmaStageChunks + kUmmaConvGroups - 1) / kUmmaConvGroups;  // max chunks per group
    const int wl = warp & 3, grp = warp >> 2;
    const int c0 = grp * kUmmaStageChunks / kUmmaConvGroups, c1 = (grp + 1) * kUmmaStageChunks / kUmmaConvGroups;
    const uint32_t lane_off = static_cast<uint32_t>(32 * wl) << 16;
    int slot = 0, sphase = 0, ab = 0, aphase = 0, ait = 0;
    for (int64_t rb = blockIdx.x; rb < n_rb; rb += gridDim.x) {
      for (int st = 0; st < n_st; ++st, ++ait) {
        mbar_wait(&full[slot], sphase);
        const uint4* src = reinterpret_cast<const uint4*>(ring + static_cast<size_t>(slot) * kUmmaStageBytes) +
                           (c0 * kUmmaRows + 32 * wl + lane);
        uint4 v[kCpg];
#pragma unroll
        for (int c = 0; c < kCpg; ++c)
          if (c0 + c < c1) v[c] = src[c * kUmmaRows];
        umma::mbar_arrive(&empty[slot]);  // the slot's bytes are in registers
        if (++slot == stages) { slot = 0; sphase ^= 1; }
        if (ait >= kUmmaABufs) mbar_wait(&aempty[ab], aphase ^ 1);
        umma::fence_after();
        const uint32_t acol = tmem + lane_off + kColA + ab * 64 + 8 * c0;
#pragma unroll
        for (int c = 0; c < kCpg; ++c) {
          if (c0 + c >= c1) break;
          const uint32_t w4[4] = {v[c].x, v[c].y, v[c].z, v[c].w};
          uint32_t r[8];
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            r[2 * j] = w4[j] & 0x0F0F0F0Fu;
            r[2 * j + 1] = (w4[j] >> 4) & 0x0F0F0F0Fu;
          }
          umma::st_32x32b_x8(acol + 8 * c, r);
        }
        umma::wait_st();
        umma::fence_before();
        umma::mbar_arrive(&afull[ab]);
        if (++ab == kUmmaABufs) { ab = 0; aphase ^= 1; }
      }
    }
  } else {
    // ===== epilogue (warp w reads TMEM lanes 32 (w % 4) ..): accumulators
    // -> scale, phi -> scores [q][row]. With two warpgroups, group eg takes
    // the row blocks rbi % 2 == eg, i.e. accumulator buffer db = eg.
    // The per-row-block work is a dependent scalar chain in 4 warps, and the
    // last block's epilogue is the kernel's tail, so it is kept short: the
    // per-query constants come from shared memory (two broadcast LDS.128 per
    // 4 queries, no shuffles or selects), the row's scale is fetched before
    // the accumulator wait, the partial sums are read two at a time, and the
    // store address is a running pointer (ncu, cfg3 B=32: the epilogue warps
    // were busy 88 % of the kernel, ~6.8 us per row block, before this).
    griddep_wait();  // scores / sx / sum(xq) of this call: after the producer grids
    const int ew = (warp - kUmmaEpiWarp) & 3, eg = (warp - kUmmaEpiWarp) >> 2;
    const uint32_t lane_off = static_cast<uint32_t>(32 * ew) << 16;
    float* s_qsx = reinterpret_cast<float*>(smem + UmmaSmem::qc_off(stages, nq, d));
    int* s_qs8 = reinterpret_cast<int*>(s_qsx + 64);
    {
      const int et = tid - 32 * kUmmaEpiWarp;
      if (et < 64) {
        s_qsx[et] = et < nb ? sx[et] : 0.0f;
        s_qs8[et] = et < nb ? 8 * sumxq[et] : 0;
      }
      asm volatile("bar.sync 1, %0;" ::"r"(128 * kUmmaEpiGroups) : "memory");
    }
    // scores kept in L2 for the selector up to 32 queries (32 MB at V=256000);
    // beyond, evict-last rows would crowd each other out
    const uint64_t pol_s = nb <= 32 ? l2_policy_evict_last() : l2_policy_evict_normal();
    (void)pol_s;
    auto store = [&](float* p, float v) {
#if HIRE_UMMA_L2
      st_hint_f32(p, v, pol_s);
#else
      *p = v;
#endif
    };
    int rbi = 0;
    for (int64_t rb = blockIdx.x; rb < n_rb; rb += gridDim.x, ++rbi) {
      if (rbi % kUmmaEpiGroups != eg) continue;
      const int db = rbi & 1;
      const int64_t row = rb * kUmmaRows + 32 * ew + lane;
      const float sc = row < rows ? scales[row] : 0.0f;  // in flight during the accumulator wait
      mbar_wait(&dfull[db], (rbi >> 1) & 1);
      umma::fence_after();
      for (int q0 = 0; q0 < nq; q0 += 16) {
        uint32_t acc[16];
        const uint32_t t0 = tmem + lane_off + kColD + db * nq + q0;
        umma::ld_32x32b_x16(t0, acc);
        if (n_iss > 1) {  // the other issuers' partial sums (n_iss is 1, 2 or 4)
          uint32_t p1[16];
          umma::ld_32x32b_x16(t0 + 2 * nq, p1);
          umma::wait_ld();
#pragma unroll
          for (int e = 0; e < 16; ++e) acc[e] += p1[e];
          if (n_iss > 2) {
            uint32_t p2[16];
            umma::ld_32x32b_x16(t0 + 4 * nq, p1);
            umma::ld_32x32b_x16(t0 + 6 * nq, p2);
            umma::wait_ld();
#pragma unroll
            for (int e = 0; e < 16; ++e) acc[e] += p1[e] + p2[e];
          }
        } else {
          umma::wait_ld();
        }
        if (q0 + 16 >= nq) {
          umma::fence_before();
          umma::mbar_arrive(&dempty[db]);
        }
        const int jn = nb - q0;  // queries of this block that exist (may be <= 0: padding)
        if (row < rows && jn > 0) {
          float* p = scores + static_cast<int64_t>(q0) * score_stride + row;
#pragma unroll
          for (int j4 = 0; j4 < 16; j4 += 4) {
            const float4 sx4 = *reinterpret_cast<const float4*>(s_qsx + q0 + j4);
            const int4 s84 = *reinterpret_cast<const int4*>(s_qs8 + q0 + j4);
            const float sxv[4] = {sx4.x, sx4.y, sx4.z, sx4.w};
            const int s8v[4] = {s84.x, s84.y, s84.z, s84.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const int j = j4 + e;
              if (j < jn) {
                const int aint = static_cast<int>(acc[j]) - s8v[e];
                const float cs = __fmul_rn(sc, sxv[e]);
                const float z = __fmul_rn(static_cast<float>(aint), cs);
                store(p, phi == kIdentity ? z : apply_phi(phi, z));
              }
              p += score_stride;
            }
          }
        }
      }
    }
  }
  griddep_launch();
  umma::fence_before();
  __syncthreads();
  if (warp == kUmmaMmaWarp) {
    umma::fence_after();
    umma::tmem_dealloc(tmem, kTmemCols);
  }
}

}  // namespace hire_dev
