// exact.cuh — row-gather exact recompute (K4), dense exact scores (K8) and
// the sparse FFN down-projection (K6).
//
// Reference semantics:
//   column_score  linalg.hpp:140-146 (every exact value goes through it;
//                 hire.hpp:71-72, ffn.hpp:125-131, ffn.hpp:165)
//   matvec        linalg.hpp:148-154
//   ffn_apply_groups ffn.hpp:154-171: out[i] += act_j * V_j[i], j ascending
//
// fast   : one warp per row, 128-bit loads, fp32 FMA per lane in column
//          order, fixed butterfly tree (common.cuh warp_sum_f32). The same
//          routine serves the gather recompute and the dense exact pass, so
//          HiRE values equal dense values bit for bit on the GPU — the
//          reference's own design rule (linalg.hpp:137-139).
// strict : one thread per row, ascending columns, __fmul_rn/__fadd_rn —
//          bit-identical to the reference's sequential fp32 loop.
#pragma once
#include "common.cuh"

namespace hire_dev {

template <typename T>
struct Vec16;
// E consecutive fp32 values of x from shared memory as 128-bit loads (the
// scalar form compiles to E LDS.32 with a 4*E-byte lane stride — an E-way
// bank conflict on every load).
template <int E>
__device__ __forceinline__ void load_x_vec(const float* p, float* out) {
#pragma unroll
  for (int q = 0; q < E / 4; ++q) {
    const float4 v = *reinterpret_cast<const float4*>(p + 4 * q);
    out[4 * q] = v.x; out[4 * q + 1] = v.y; out[4 * q + 2] = v.z; out[4 * q + 3] = v.w;
  }
}

template <>
struct Vec16<__nv_bfloat16> {
  static constexpr int kElems = 8;
  __device__ __forceinline__ static void expand(uint4 u, float* f) {
    f[0] = bf16_lo(u.x); f[1] = bf16_hi(u.x); f[2] = bf16_lo(u.y); f[3] = bf16_hi(u.y);
    f[4] = bf16_lo(u.z); f[5] = bf16_hi(u.z); f[6] = bf16_lo(u.w); f[7] = bf16_hi(u.w);
  }
};
template <>
struct Vec16<float> {
  static constexpr int kElems = 4;
  __device__ __forceinline__ static void expand(uint4 u, float* f) {
    f[0] = __uint_as_float(u.x); f[1] = __uint_as_float(u.y);
    f[2] = __uint_as_float(u.z); f[3] = __uint_as_float(u.w);
  }
};

// grid = (tiles, B); 8 warps per CTA; warp-strided over the n_cand rows of
// query b. cand == nullptr means row i itself (dense exact, K8).
template <typename T, int CPL>
__global__ void __launch_bounds__(256, (CPL >= 16 ? 1 : 2)) recompute_fast(
    const T* __restrict__ w, int d, const uint32_t* __restrict__ cand, int64_t cand_stride,
    int n_cand, const float* __restrict__ x, int phi, float* __restrict__ out,
    int64_t out_stride) {
  hire_dev::griddep_wait();
  KTrace kt_(kKtRecompute);
  extern __shared__ __align__(16) unsigned char smem[];
  float* s_x = reinterpret_cast<float*>(smem);
  constexpr int E = Vec16<T>::kElems;
  const int b = blockIdx.y;
  block_copy(s_x, x + static_cast<int64_t>(b) * d, d);
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int64_t pitch_vec = static_cast<int64_t>(d) / E;  // 16-byte vectors per row
  // long rows (CPL >= 16, one CTA/SM): the next row's loads are issued
  // before this row's arithmetic (two rows in flight per warp); the
  // arithmetic per lane is unchanged (same chunks, same fmaf order)
  constexpr bool kPrefetch = CPL >= 16;
  const int step = gridDim.x * 8;
  auto row_ptr = [&](int i) {
    const int64_t row = cand ? cand[b * cand_stride + i] : i;
    return reinterpret_cast<const uint4*>(w) + row * pitch_vec;
  };
  uint4 nv[kPrefetch ? CPL : 1];
  if (kPrefetch && blockIdx.x * 8 + wid < n_cand) {
    const uint4* rp = row_ptr(blockIdx.x * 8 + wid);
#pragma unroll
    for (int c = 0; c < (kPrefetch ? CPL : 1); ++c) nv[c] = ldg_stream(rp + lane + 32 * c);
  }
#pragma unroll 1
  for (int i = blockIdx.x * 8 + wid; i < n_cand; i += step) {
    uint4 v[CPL];
    if constexpr (kPrefetch) {
#pragma unroll
      for (int c = 0; c < CPL; ++c) v[c] = nv[(kPrefetch ? c : 0)];
      if (i + step < n_cand) {
        const uint4* rn = row_ptr(i + step);
#pragma unroll
        for (int c = 0; c < (kPrefetch ? CPL : 1); ++c) nv[c] = ldg_stream(rn + lane + 32 * c);
      }
    } else {
      const uint4* rp = row_ptr(i);
#pragma unroll
      for (int c = 0; c < CPL; ++c) v[c] = ldg_stream(rp + lane + 32 * c);
    }
    float acc = 0.0f;
#pragma unroll
    for (int c = 0; c < CPL; ++c) {
      float f[E], xv[E];
      Vec16<T>::expand(v[c], f);
      load_x_vec<E>(s_x + (lane + 32 * c) * E, xv);
#pragma unroll
      for (int e = 0; e < E; ++e) acc = fmaf(f[e], xv[e], acc);
    }
    acc = warp_sum_f32(acc);
    if (lane == 0) out[b * out_stride + i] = apply_phi(phi, acc);
  }
  // late trigger: dependents launched at this kernel's start are packed onto
  // the first SMs that drain (several per-query CTAs of the final top-k on
  // one SM: cfg3 B=32 CTA durations 4.8 .. 9.9 us); launched at its end they
  // spread over the idle GPU
  hire_dev::griddep_launch();
}

// ---------------------------------------------------------------------
// K4U — batch-union gather recompute (the device counterpart of
// union_group_select's premise, ffn.hpp:237-253: a row selected by several
// inputs of the batch is fetched once). For batches whose candidate lists
// overlap heavily (FFN layers: B * k' >> rows) the per-query gather moves
// every row once per query that selected it through L2; here each unique row
// leaves L2 once.
//   U1 union_mark_kernel   rowmask[r] |= 1 << b for every candidate (b, r)
//   U2 union_dot_kernel    grid (CPL column slices, row tiles). A slice is 512
//        bytes of every row (one 16-byte vector per lane — the same lane /
//        column assignment as recompute_fast's chunk c). The CTA holds the
//        slice of x for all B queries in shared memory (B * 512/sizeof(T) * 4
//        bytes); a warp takes a row with a non-empty mask, loads its slice
//        once, and for each query of the mask does the lane FMAs in column
//        order and the fixed butterfly -> part[b][r][slice].
//   U3 union_gather_kernel out[b][j] = phi(sum over slices, ascending, of
//        part[b][cand[b][j]][slice]); clears rowmask (zero at rest).
// Fixed order, so deterministic and independent of the batch composition;
// the association differs from recompute_fast's (per-slice butterflies, then
// the slice sum), so values agree with the per-query path to fp32 rounding
// (~1e-7 relative), not bit for bit. Fast mode only.
//
// Experiments build only (negative result on B200, cfg2 shape, bf16): one
// FFN layer at B = 8 / 16 / 32 / 64 takes 39 / 50 / 62 / 90 us with the
// per-query gather and 50 / 66 / 90 / 149 us with this path. The per-query
// kernels already read each unique row from HBM once — L2 holds the layer
// (ncu, profiles/r02c_ffn_gather_dram_b*.csv: recompute_fast reads 18.6 MB
// from DRAM at B=8 for 18.9 MB of unique rows, 34.2 MB at B=64 for 33.5 MB,
// while L2 serves 40 / 242 MB) — and they amortise the butterfly and the loop
// overhead over a whole row (~24 instructions per 512-byte slice of a pair)
// where this kernel pays them per slice (73; ncu: 30.7 M warp instructions,
// short-scoreboard bound).
// ---------------------------------------------------------------------
#if HIRE_EXPERIMENTS
__global__ void __launch_bounds__(256) union_mark_kernel(const uint32_t* __restrict__ cand, int64_t cand_stride,
                                                         int n_cand, int B, unsigned long long* __restrict__ rowmask) {
  hire_dev::griddep_wait();
  hire_dev::griddep_launch();
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= static_cast<int64_t>(B) * n_cand) return;
  const int b = static_cast<int>(t / n_cand), j = static_cast<int>(t % n_cand);
  atomicOr(rowmask + cand[b * cand_stride + j], 1ull << b);
}

template <typename T>
__global__ void __launch_bounds__(256) union_dot_kernel(const T* __restrict__ w, int d, int64_t rows,
                                                        const unsigned long long* __restrict__ rowmask,
                                                        const float* __restrict__ x, int B, int rows_per_cta,
                                                        float* __restrict__ part) {
  constexpr int E = Vec16<T>::kElems;
  constexpr int DC = 32 * E;  // columns per slice
  extern __shared__ __align__(16) unsigned char smem[];
  float* s_x = reinterpret_cast<float*>(smem);  // [B][DC]
  hire_dev::griddep_wait();
  hire_dev::griddep_launch();
  KTrace kt_(kKtRecompute);
  const int ct = blockIdx.x, nct = gridDim.x;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < B * (DC / 4); i += blockDim.x) {
    const int b = i / (DC / 4), q = i % (DC / 4);
    reinterpret_cast<float4*>(s_x)[i] =
        *reinterpret_cast<const float4*>(x + static_cast<int64_t>(b) * d + static_cast<int64_t>(ct) * DC + 4 * q);
  }
  __syncthreads();
  const int64_t pitch_vec = static_cast<int64_t>(d) / E;
  const int64_t r0 = static_cast<int64_t>(blockIdx.y) * rows_per_cta;
  const int64_t r1 = min(rows, r0 + rows_per_cta);
  // two rows per warp in flight: the next row's mask and slice are fetched
  // before this row's arithmetic
  int64_t r = r0 + wid;
  unsigned long long m_next = r < r1 ? rowmask[r] : 0ull;
  uint4 v_next = make_uint4(0, 0, 0, 0);
  if (m_next) v_next = ldg_stream(reinterpret_cast<const uint4*>(w) + r * pitch_vec + static_cast<int64_t>(ct) * 32 + lane);
  for (; r < r1; r += 8) {
    unsigned long long m = m_next;
    const uint4 v = v_next;
    const int64_t rn = r + 8;
    m_next = rn < r1 ? rowmask[rn] : 0ull;
    if (m_next) v_next = ldg_stream(reinterpret_cast<const uint4*>(w) + rn * pitch_vec + static_cast<int64_t>(ct) * 32 + lane);
    if (!m) continue;
    float f[E];
    Vec16<T>::expand(v, f);
    while (m) {
      const int b = __ffsll(static_cast<long long>(m)) - 1;
      m &= m - 1ull;
      float xv[E];
      load_x_vec<E>(s_x + b * DC + lane * E, xv);
      float acc = 0.0f;
#pragma unroll
      for (int e = 0; e < E; ++e) acc = fmaf(f[e], xv[e], acc);
      acc = warp_sum_f32(acc);
      if (lane == 0) part[(static_cast<int64_t>(b) * rows + r) * nct + ct] = acc;
    }
  }
}

__global__ void __launch_bounds__(256) union_gather_kernel(const float* __restrict__ part, int64_t rows, int nct,
                                                           const uint32_t* __restrict__ cand, int64_t cand_stride,
                                                           int n_cand, int B, int phi, float* __restrict__ out,
                                                           int64_t out_stride, unsigned long long* __restrict__ rowmask) {
  hire_dev::griddep_wait();
  hire_dev::griddep_launch();
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= static_cast<int64_t>(B) * n_cand) return;
  const int b = static_cast<int>(t / n_cand), j = static_cast<int>(t % n_cand);
  const int64_t r = cand[b * cand_stride + j];
  const float* p = part + (static_cast<int64_t>(b) * rows + r) * nct;
  float acc = 0.0f;
  for (int c = 0; c < nct; ++c) acc = __fadd_rn(acc, __ldcg(p + c));
  out[b * out_stride + j] = apply_phi(phi, acc);
  rowmask[r] = 0ull;  // zero at rest (every selecting query writes the same zero)
}
#endif  // HIRE_EXPERIMENTS (K4U)

#if HIRE_EXPERIMENTS
// Same arithmetic as recompute_fast (lane chunk order, fmaf order, fixed
// butterfly -> bit-identical values), but the gathered rows are moved by
// the bulk-copy engine into shared memory (cp.async.bulk + mbarrier), so the
// bytes in flight are not bounded by registers. Each warp owns two groups
// of G row slots and alternates: while one group is consumed the other is
// in flight. A group is consumed chunk by chunk with each x chunk read once
// for all G rows (x is the larger smem stream: fp32 vs bf16 rows). x sits in
// shared memory split into low / high 16-byte halves of each lane chunk so
// the 128-bit reads are conflict-free. 4 warps, one CTA per SM.
template <typename T, int G>
__global__ void __launch_bounds__(128, 1) recompute_tma(
    const T* __restrict__ w, int d, const uint32_t* __restrict__ cand, int64_t cand_stride,
    int n_cand, const float* __restrict__ x, int phi, float* __restrict__ out, int64_t out_stride) {
  hire_dev::griddep_wait();
  hire_dev::griddep_launch();
  KTrace kt_(kKtRecompute);
  constexpr int NW = 4, S = 2 * G;
  constexpr int E = Vec16<T>::kElems;  // elements per 16-byte chunk
  extern __shared__ __align__(128) unsigned char smem[];
  const int b = blockIdx.y;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const unsigned row_bytes = static_cast<unsigned>(d) * sizeof(T);
  const int cpl = static_cast<int>(row_bytes / 512);
  const int nchunk = d / E;
  float* s_xa = reinterpret_cast<float*>(smem);            // [nchunk][min(E,4)]
  float* s_xb = s_xa + static_cast<size_t>(nchunk) * 4;    // [nchunk][4] (E == 8 only)
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + static_cast<size_t>(d) * 4);
  unsigned char* rows = smem + ((static_cast<size_t>(d) * 4 + NW * S * 8 + 127) & ~static_cast<size_t>(127));
  uint64_t* mybar = bars + wid * S;
  unsigned char* myrows = rows + static_cast<size_t>(wid) * S * row_bytes;
  if (lane == 0)
    for (int s = 0; s < S; ++s) mbar_init(&mybar[s], 1);
  fence_mbar_init();
  {
    const float* xb = x + static_cast<int64_t>(b) * d;
    for (int i = threadIdx.x; i < d; i += blockDim.x) {
      const int ch = i / E, e = i % E;
      if (E == 8) (e < 4 ? s_xa : s_xb)[ch * 4 + (e & 3)] = xb[i];
      else s_xa[i] = xb[i];
    }
  }
  __syncthreads();
  const int gw = blockIdx.x * NW + wid, nw = gridDim.x * NW;
  const int cnt = n_cand > gw ? (n_cand - gw + nw - 1) / nw : 0;  // rows of this warp: gw + k*nw
  auto issue = [&](int k, int s) {
    const int i = gw + k * nw;
    const int64_t row = cand ? static_cast<int64_t>(cand[b * cand_stride + i]) : i;
    mbar_arrive_expect_tx(&mybar[s], row_bytes);
    bulk_g2s(myrows + static_cast<size_t>(s) * row_bytes,
             reinterpret_cast<const unsigned char*>(w) + row * row_bytes, row_bytes, &mybar[s]);
  };
  const int ngroups = (cnt + G - 1) / G;
  if (lane == 0)
    for (int k = 0; k < S && k < cnt; ++k) issue(k, k);
  for (int gi = 0; gi < ngroups; ++gi) {
    const int half = gi & 1;
    const unsigned ph = static_cast<unsigned>((gi >> 1) & 1);
    const int k0 = gi * G;
    float acc[G];
#pragma unroll
    for (int r = 0; r < G; ++r) {
      acc[r] = 0.0f;
      if (k0 + r < cnt) mbar_wait(&mybar[half * G + r], ph);
    }
    const uint4* rp = reinterpret_cast<const uint4*>(myrows + static_cast<size_t>(half * G) * row_bytes);
    const int rstride = static_cast<int>(row_bytes / 16);
#pragma unroll 2
    for (int c = 0; c < cpl; ++c) {
      const int ch = lane + 32 * c;
      float xv[E];
      {
        const float4 a = *reinterpret_cast<const float4*>(s_xa + ch * 4);
        xv[0] = a.x; xv[1] = a.y; xv[2] = a.z; xv[3] = a.w;
        if (E == 8) {
          const float4 bq = *reinterpret_cast<const float4*>(s_xb + ch * 4);
          xv[4 % E] = bq.x; xv[5 % E] = bq.y; xv[6 % E] = bq.z; xv[7 % E] = bq.w;
        }
      }
#pragma unroll
      for (int r = 0; r < G; ++r) {
        float f[E];
        Vec16<T>::expand(rp[r * rstride + ch], f);
#pragma unroll
        for (int e = 0; e < E; ++e) acc[r] = fmaf(f[e], xv[e], acc[r]);
      }
    }
#pragma unroll
    for (int r = 0; r < G; ++r) {
      const float v = warp_sum_f32(acc[r]);
      if (lane == 0 && k0 + r < cnt) out[b * out_stride + gw + (k0 + r) * nw] = apply_phi(phi, v);
    }
    __syncwarp();
    if (lane == 0) {
      fence_proxy_async_smem();  // this group's reads precede its refill
#pragma unroll
      for (int r = 0; r < G; ++r)
        if (k0 + r + S < cnt) issue(k0 + r + S, half * G + r);
    }
  }
}
#endif  // HIRE_EXPERIMENTS

// strict / generic: one thread per row; any d.
template <typename T>
__global__ void __launch_bounds__(128) recompute_seq(
    const T* __restrict__ w, int d, const uint32_t* __restrict__ cand, int64_t cand_stride,
    int n_cand, const float* __restrict__ x, int phi, float* __restrict__ out,
    int64_t out_stride) {
  hire_dev::griddep_wait();
  hire_dev::LateTrigger late_trigger_;
  KTrace kt_(kKtRecompute);
  extern __shared__ __align__(16) unsigned char smem[];
  float* s_x = reinterpret_cast<float*>(smem);
  const int b = blockIdx.y;
  block_copy(s_x, x + static_cast<int64_t>(b) * d, d);
  __syncthreads();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_cand) return;
  const int64_t row = cand ? cand[b * cand_stride + i] : i;
  const T* rp = w + row * d;
  float acc = 0.0f;
  for (int c = 0; c < d; ++c) acc = __fadd_rn(acc, __fmul_rn(load_elem<T>(rp, c), s_x[c]));
  out[b * out_stride + i] = apply_phi(phi, acc);
}

// ---------------------------------------------------------------------
// K6 fast: split over selected units. grid = (n_chunks, B), 256 threads;
// chunk c sums units [c*CH, c*CH+CH) of query b (ascending) for all d
// columns; each thread owns 8 (bf16) / 4 (fp32) consecutive columns per
// pass. partial[b][c][d] is then reduced over c ascending (deterministic).
// ---------------------------------------------------------------------
template <typename T>
__global__ void __launch_bounds__(256) ffn_down_partial(
    const T* __restrict__ v, int d, const uint32_t* __restrict__ sel,
    const float* __restrict__ act, int64_t sel_stride, int n_sel, int ch,
    float* __restrict__ partial) {
  hire_dev::griddep_wait();
  hire_dev::LateTrigger late_trigger_;
  KTrace kt_(kKtDown);
  constexpr int E = Vec16<T>::kElems;
  const int c = blockIdx.x, b = blockIdx.y;
  const int lo = c * ch, hi = min(n_sel, lo + ch);
  const int64_t pitch_vec = d / E;
  float* pout = partial + (static_cast<int64_t>(b) * gridDim.x + c) * d;
  for (int col0 = threadIdx.x; col0 < pitch_vec; col0 += blockDim.x) {
    float acc[E];
#pragma unroll
    for (int e = 0; e < E; ++e) acc[e] = 0.0f;
    int j = lo;
    for (; j + 4 <= hi; j += 4) {
      uint4 u[4];
      float a[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int64_t row = sel[b * sel_stride + j + q];
        a[q] = act[b * sel_stride + j + q];
        u[q] = ldg_stream(reinterpret_cast<const uint4*>(v) + row * pitch_vec + col0);
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        float f[E];
        Vec16<T>::expand(u[q], f);
#pragma unroll
        for (int e = 0; e < E; ++e) acc[e] = fmaf(a[q], f[e], acc[e]);
      }
    }
    for (; j < hi; ++j) {
      const int64_t row = sel[b * sel_stride + j];
      const float a = act[b * sel_stride + j];
      float f[E];
      Vec16<T>::expand(ldg_stream(reinterpret_cast<const uint4*>(v) + row * pitch_vec + col0), f);
#pragma unroll
      for (int e = 0; e < E; ++e) acc[e] = fmaf(a, f[e], acc[e]);
    }
#pragma unroll
    for (int e = 0; e < E; ++e) pout[col0 * E + e] = acc[e];
  }
}

__global__ void __launch_bounds__(256) ffn_down_reduce(const float* __restrict__ partial,
                                                       int n_chunks, int d, int B,
                                                       float* __restrict__ out) {
  hire_dev::griddep_wait();
  hire_dev::griddep_launch();
  const int64_t id = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (id >= static_cast<int64_t>(B) * d) return;
  const int b = static_cast<int>(id / d), col = static_cast<int>(id % d);
  const float* p = partial + static_cast<int64_t>(b) * n_chunks * d + col;
  float s = 0.0f;
  for (int c = 0; c < n_chunks; ++c) s = __fadd_rn(s, p[static_cast<int64_t>(c) * d]);
  out[id] = s;
}

// strict: one thread per (column, query); units ascending; no contraction.
// Bit-identical to ffn.hpp:160-169 given identical activations.
template <typename T>
__global__ void __launch_bounds__(256) ffn_down_seq(const T* __restrict__ v, int d,
                                                    const uint32_t* __restrict__ sel,
                                                    const float* __restrict__ act,
                                                    int64_t sel_stride, int n_sel,
                                                    float* __restrict__ out) {
  hire_dev::griddep_wait();
  hire_dev::griddep_launch();
  const int col = blockIdx.x * blockDim.x + threadIdx.x, b = blockIdx.y;
  if (col >= d) return;
  float acc = 0.0f;
  for (int j = 0; j < n_sel; ++j) {
    const int64_t row = sel[b * sel_stride + j];
    acc = __fadd_rn(acc, __fmul_rn(act[b * sel_stride + j], load_elem<T>(v + row * d, col)));
  }
  out[static_cast<int64_t>(b) * d + col] = acc;
}

}  // namespace hire_dev
