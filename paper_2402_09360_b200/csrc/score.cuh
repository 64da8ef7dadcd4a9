// score.cuh — compressed-proxy scorers (K1 int4, K2 low-rank), the x
// quantiser for the integer mode and the on-device int4 proxy build (K9).
//
// Reference semantics being replaced:
//   ApproxScorer::scores  /root/reference/proj/include/hire/approx.hpp:382-411
//     quantized branch :395-403  s_j = phi(sum_i (code_ji*scale_j)*x_i)
//     low-rank branch  :477-496  t = Z1^T x ; s_j = phi(sum_q Z2[j,q] t_q)
//   quantize_int4       approx.hpp:49-65
//
// Device layouts:
//   int4 proxy  : uint8 [rows][pitch], pitch = round_up(ceil(d/2), 16);
//                 two codes per byte, low nibble = even column (the HIRQ
//                 packing of approx.hpp:551-564, one row per reference column)
//   scales      : fp32 [rows]
//   low-rank Z1 : T [r][d]   (reference z1 columns, byte-identical)
//   low-rank Z2 : T [rows][r] (row j = the r coefficients of output j)
#pragma once
#include "common.cuh"

namespace hire_dev {

// ---------------------------------------------------------------------
// Integer mode, step 0: quantise each query x[b] to int8 with the
// quantize_int4 rule widened to [-127,127] (approx.hpp:41-65):
//   sx = max|x| / 127 (1 if x == 0), xq_i = RHAZ(x_i / sx).
// Writes xq (natural order), xperm (xg_mode 0: dp4a order, see
// q4_score_fast_int8; xg_mode 1: the tcgen05 proxy's B-operand layout,
// xg_offset in score_umma.cuh, with CTAs b >= n_real writing the zero
// padding queries), sx and sum(xq). One CTA per query.
// ---------------------------------------------------------------------
__global__ void __launch_bounds__(256) prep_x_int8_kernel(
    const float* __restrict__ x, int d, int8_t* __restrict__ xq,
    int8_t* __restrict__ xperm, float* __restrict__ sx_out,
    int* __restrict__ sumxq_out, int xg_mode, int n_real) {
  hire_dev::griddep_wait();
  hire_dev::griddep_launch();
  KTrace kt_(kKtPrep);
  const int b = blockIdx.x;
  if (b >= n_real) {  // padding query of the grouped layout (xg_mode 1)
    for (int i = threadIdx.x * 16; i < d; i += blockDim.x * 16)
      *reinterpret_cast<int4*>(xperm + (static_cast<int64_t>(b) >> 3) * 8 * d + (i >> 4) * 128 + (b & 7) * 16) =
          make_int4(0, 0, 0, 0);
    return;
  }
  const float* xb = x + static_cast<int64_t>(b) * d;
  __shared__ float s_red[8];
  __shared__ int s_sum[8];
  // x stays in registers between the two passes (d <= 256 * kXR on the fast
  // path; longer vectors stream the remainder)
  constexpr int kXR = 32;
  float xr[kXR];
  float m = 0.0f;
#pragma unroll
  for (int r = 0; r < kXR; ++r) {
    const int i = threadIdx.x + r * 256;
    xr[r] = i < d ? xb[i] : 0.0f;
  }
#pragma unroll
  for (int r = 0; r < kXR; ++r) m = fmaxf(m, fabsf(xr[r]));
  for (int i = threadIdx.x + kXR * 256; i < d; i += blockDim.x) m = fmaxf(m, fabsf(xb[i]));
  m = warp_max_f32(m);
  if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x < 32) {
    float v = threadIdx.x < (blockDim.x >> 5) ? s_red[threadIdx.x] : 0.0f;
    v = warp_max_f32(v);
    if (threadIdx.x == 0) s_red[0] = v;
  }
  __syncthreads();
  const float maxabs = s_red[0];
  const float sx = maxabs > 0.0f ? __fdiv_rn(maxabs, 127.0f) : 1.0f;
  int local = 0;
#pragma unroll
  for (int r = 0; r < kXR; ++r) {
    const int i = threadIdx.x + r * 256;
    if (i >= d) break;
    const int q = rhaz_clamp(__fdiv_rn(xr[r], sx), 127);
    local += q;
    xq[static_cast<int64_t>(b) * d + i] = static_cast<int8_t>(q);
    if (xg_mode) {
      xperm[(static_cast<int64_t>(b) >> 3) * 8 * d + (i >> 4) * 128 + (b & 7) * 16 + (i & 15)] = static_cast<int8_t>(q);
    } else {
      const int g = i & ~7, j = i & 7;
      const int pos = g + ((j & 1) ? 4 : 0) + (j >> 1);
      xperm[static_cast<int64_t>(b) * d + pos] = static_cast<int8_t>(q);
    }
  }
  for (int i = threadIdx.x + kXR * 256; i < d; i += blockDim.x) {
    const int q = rhaz_clamp(__fdiv_rn(xb[i], sx), 127);
    local += q;
    xq[static_cast<int64_t>(b) * d + i] = static_cast<int8_t>(q);
    if (xg_mode) {
      xperm[(static_cast<int64_t>(b) >> 3) * 8 * d + (i >> 4) * 128 + (b & 7) * 16 + (i & 15)] = static_cast<int8_t>(q);
    } else {
      // dp4a order: within each 8-element word group, the 4 even elements
      // then the 4 odd elements (matches the lo/hi nibble extraction).
      const int g = i & ~7, j = i & 7;
      const int pos = g + ((j & 1) ? 4 : 0) + (j >> 1);
      xperm[static_cast<int64_t>(b) * d + pos] = static_cast<int8_t>(q);
    }
  }
  local = warp_sum_i32(local);
  if ((threadIdx.x & 31) == 0) s_sum[threadIdx.x >> 5] = local;
  __syncthreads();
  if (threadIdx.x == 0) {
    int s = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += s_sum[w];
    sumxq_out[b] = s;
    sx_out[b] = sx;
  }
}

// ---------------------------------------------------------------------
// K1, integer mode, fast path (d % 1024 == 0). One warp per row, two rows
// in flight per warp; each lane streams CPL 16-byte chunks (32 codes) of
// each row with 128-bit non-allocating loads and keeps the matching int8 x
// words of QB queries in registers for the whole kernel.
//   Offset trick: code c in [-7,7] is the two's-complement nibble n;
//   n ^ 8 == c + 8 in [1,15], so one XOR per word turns 8 nibbles into
//   unsigned digits; lo/hi masks give 4 bytes each, fed to dp4a against the
//   even/odd x bytes. sum((c+8)*xq) - 8*sum(xq) = sum(c*xq) exactly (int32).
//   score = phi(float(acc) * (scale_j * sx)) — the oracle's multiply order.
// ---------------------------------------------------------------------
template <int QB, int CPL>
__global__ void __launch_bounds__(256) q4_score_fast_int8(
    const uint8_t* __restrict__ wq, int64_t pitch, const float* __restrict__ scales,
    int64_t rows, int d, const int8_t* __restrict__ xperm,
    const float* __restrict__ sx, const int* __restrict__ sumxq, int phi,
    float* __restrict__ scores, int64_t score_stride) {
  hire_dev::griddep_wait();
  hire_dev::LateTrigger late_trigger_;
  KTrace kt_(kKtProxy);
  const int lane = threadIdx.x & 31;
  const int64_t warp = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;

  int xw[QB][CPL][8];
#pragma unroll
  for (int q = 0; q < QB; ++q)
#pragma unroll
    for (int c = 0; c < CPL; ++c) {
      const int4* p = reinterpret_cast<const int4*>(
          xperm + static_cast<int64_t>(q) * d + (lane + 32 * c) * 32);
      const int4 a = p[0], b = p[1];
      xw[q][c][0] = a.x; xw[q][c][1] = a.y; xw[q][c][2] = a.z; xw[q][c][3] = a.w;
      xw[q][c][4] = b.x; xw[q][c][5] = b.y; xw[q][c][6] = b.z; xw[q][c][7] = b.w;
    }
  float qsx[QB];
  int qsum[QB];
#pragma unroll
  for (int q = 0; q < QB; ++q) { qsx[q] = sx[q]; qsum[q] = sumxq[q]; }

  for (int64_t r0 = warp * 2; r0 < rows; r0 += nwarps * 2) {
    const bool has1 = r0 + 1 < rows;
    uint4 w[2][CPL];
#pragma unroll
    for (int c = 0; c < CPL; ++c) {
      w[0][c] = ldg_stream(wq + r0 * pitch + (lane + 32 * c) * 16);
      w[1][c] = has1 ? ldg_stream(wq + (r0 + 1) * pitch + (lane + 32 * c) * 16)
                     : make_uint4(0x88888888u, 0x88888888u, 0x88888888u, 0x88888888u);
    }
    int acc[2][QB];
#pragma unroll
    for (int rr = 0; rr < 2; ++rr) {
#pragma unroll
      for (int q = 0; q < QB; ++q) acc[rr][q] = 0;
#pragma unroll
      for (int c = 0; c < CPL; ++c) {
        const uint32_t words[4] = {w[rr][c].x, w[rr][c].y, w[rr][c].z, w[rr][c].w};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const uint32_t u = words[k] ^ 0x88888888u;
          const int lo = static_cast<int>(u & 0x0F0F0F0Fu);
          const int hi = static_cast<int>((u >> 4) & 0x0F0F0F0Fu);
#pragma unroll
          for (int q = 0; q < QB; ++q) {
            acc[rr][q] = __dp4a(lo, xw[q][c][2 * k], acc[rr][q]);
            acc[rr][q] = __dp4a(hi, xw[q][c][2 * k + 1], acc[rr][q]);
          }
        }
      }
#pragma unroll
      for (int q = 0; q < QB; ++q) acc[rr][q] = warp_sum_i32(acc[rr][q]);
    }
    // lanes 0..2*QB-1 write one (row, query) each
#pragma unroll
    for (int rr = 0; rr < 2; ++rr)
#pragma unroll
      for (int q = 0; q < QB; ++q)
        if (lane == rr * QB + q && (rr == 0 || has1)) {
          const int a = acc[rr][q] - 8 * qsum[q];
          const float cs = __fmul_rn(scales[r0 + rr], qsx[q]);
          scores[static_cast<int64_t>(q) * score_stride + r0 + rr] =
              apply_phi(phi, __fmul_rn(static_cast<float>(a), cs));
        }
  }
}

// ---------------------------------------------------------------------
// K1, fp32-x mode (the reference's own scorer, approx.hpp:395-403), fast
// path: one query per pass, x in registers, nibble -> fp32 through the
// 2^23 magic constant (exact), fp32 FMA per code, x-chunk partial sums
// reduced by the fixed warp tree, then one multiply by scale_j. Values
// differ from the reference's sequential sum by rounding only (near-tie
// tolerance); the strict kernel below is bit-exact.
// ---------------------------------------------------------------------
template <int CPL>
__global__ void __launch_bounds__(256) q4_score_fast_fpx(
    const uint8_t* __restrict__ wq, int64_t pitch, const float* __restrict__ scales,
    int64_t rows, int d, const float* __restrict__ x, int phi,
    float* __restrict__ scores) {
  hire_dev::griddep_wait();
  hire_dev::LateTrigger late_trigger_;
  KTrace kt_(kKtProxy);
  const int lane = threadIdx.x & 31;
  const int64_t warp = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  float xr[CPL][32];
#pragma unroll
  for (int c = 0; c < CPL; ++c) {
    const float4* p = reinterpret_cast<const float4*>(x + (lane + 32 * c) * 32);
#pragma unroll
    for (int v = 0; v < 8; ++v) {
      const float4 f = p[v];
      xr[c][4 * v] = f.x; xr[c][4 * v + 1] = f.y; xr[c][4 * v + 2] = f.z; xr[c][4 * v + 3] = f.w;
    }
  }
  for (int64_t r = warp; r < rows; r += nwarps) {
    uint4 w[CPL];
#pragma unroll
    for (int c = 0; c < CPL; ++c) w[c] = ldg_stream(wq + r * pitch + (lane + 32 * c) * 16);
    float acc = 0.0f;
#pragma unroll
    for (int c = 0; c < CPL; ++c) {
      const uint32_t words[4] = {w[c].x, w[c].y, w[c].z, w[c].w};
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint32_t u = words[k] ^ 0x88888888u;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float cf = __fsub_rn(__uint_as_float(0x4B000000u | ((u >> (4 * j)) & 0xFu)), 8388616.0f);
          acc = fmaf(cf, xr[c][8 * k + j], acc);
        }
      }
    }
    acc = warp_sum_f32(acc);
    if (lane == 0) scores[r] = apply_phi(phi, __fmul_rn(acc, scales[r]));
  }
}

// ---------------------------------------------------------------------
// K1, generic / strict path: one thread per row, columns in ascending order.
//   fp32-x : acc = acc + (code*scale)*x_i, no contraction — bit-identical to
//            approx.hpp:398-402.
//   int8   : exact int32 sum, then the integer-mode epilogue.
// Any d; x (and xq) for the query staged in shared memory (broadcast reads).
// ---------------------------------------------------------------------
__global__ void __launch_bounds__(128) q4_score_seq(
    const uint8_t* __restrict__ wq, int64_t pitch, const float* __restrict__ scales,
    int64_t rows, int d, const float* __restrict__ x, const int8_t* __restrict__ xq,
    const float* __restrict__ sx, int int8_mode, int phi, float* __restrict__ scores,
    int64_t score_stride) {
  hire_dev::griddep_wait();
  hire_dev::LateTrigger late_trigger_;
  KTrace kt_(kKtProxy);
  extern __shared__ __align__(16) unsigned char smem[];
  float* s_x = reinterpret_cast<float*>(smem);
  int8_t* s_xq = reinterpret_cast<int8_t*>(smem + static_cast<size_t>(d) * 4);
  const int b = blockIdx.y;
  for (int i = threadIdx.x; i < d; i += blockDim.x) {
    if (int8_mode) s_xq[i] = xq[static_cast<int64_t>(b) * d + i];
    else s_x[i] = x[static_cast<int64_t>(b) * d + i];
  }
  __syncthreads();
  const int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r >= rows) return;
  const uint8_t* row = wq + r * pitch;
  const float scale = scales[r];
  if (int8_mode) {
    int acc = 0;
    for (int i0 = 0; i0 < d; i0 += 32) {
      const uint4 v = *reinterpret_cast<const uint4*>(row + i0 / 2);
      const uint32_t words[4] = {v.x, v.y, v.z, v.w};
      for (int j = 0; j < 32 && i0 + j < d; ++j) {
        const uint32_t nib = (words[j >> 3] >> (4 * (j & 7))) & 0xFu;
        const int c = static_cast<int>(nib ^ 8u) - 8;
        acc += c * s_xq[i0 + j];
      }
    }
    const float cs = __fmul_rn(scale, sx[b]);
    scores[static_cast<int64_t>(b) * score_stride + r] =
        apply_phi(phi, __fmul_rn(static_cast<float>(acc), cs));
  } else {
    float acc = 0.0f;
    for (int i0 = 0; i0 < d; i0 += 32) {
      const uint4 v = *reinterpret_cast<const uint4*>(row + i0 / 2);
      const uint32_t words[4] = {v.x, v.y, v.z, v.w};
      for (int j = 0; j < 32 && i0 + j < d; ++j) {
        const uint32_t nib = (words[j >> 3] >> (4 * (j & 7))) & 0xFu;
        const float c = static_cast<float>(static_cast<int>(nib ^ 8u) - 8);
        acc = __fadd_rn(acc, __fmul_rn(__fmul_rn(c, scale), s_x[i0 + j]));
      }
    }
    scores[static_cast<int64_t>(b) * score_stride + r] = apply_phi(phi, acc);
  }
}

// ---------------------------------------------------------------------
// K9 — int4 proxy build on the device (approx.hpp:49-65): per row absmax,
// scale = absmax/7 (IEEE division, 1 for a zero row), code = RHAZ(w/scale)
// clamped to [-7,7], packed low nibble first. One warp per row.
// ---------------------------------------------------------------------
template <typename T>
__global__ void __launch_bounds__(256) quantize_q4_kernel(
    const T* __restrict__ w, int64_t rows, int d, uint8_t* __restrict__ wq, int64_t pitch,
    float* __restrict__ scales) {
  hire_dev::griddep_wait();
  hire_dev::griddep_launch();
  const int lane = threadIdx.x & 31;
  const int64_t r = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  if (r >= rows) return;
  const T* row = w + r * d;
  float m = 0.0f;
  for (int i = lane; i < d; i += 32) m = fmaxf(m, fabsf(load_elem<T>(row, i)));
  m = warp_max_f32(m);
  const float scale = m > 0.0f ? __fdiv_rn(m, 7.0f) : 1.0f;
  if (lane == 0) scales[r] = scale;
  uint8_t* out = wq + r * pitch;
  // each lane packs 8 consecutive codes into one 32-bit word
  for (int g = lane * 8; g < static_cast<int>(pitch) * 2; g += 256) {
    uint32_t word = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int i = g + j;
      if (i < d) {
        const int c = rhaz_clamp(__fdiv_rn(load_elem<T>(row, i), scale), 7);
        word |= (static_cast<uint32_t>(c) & 0xFu) << (4 * j);
      }
    }
    if (g / 2 + 3 < pitch) *reinterpret_cast<uint32_t*>(out + g / 2) = word;
    else
      for (int j = 0; j < 4 && g / 2 + j < pitch; ++j) out[g / 2 + j] = (word >> (8 * j)) & 0xFF;
  }
}

// ---------------------------------------------------------------------
// K2 — low-rank proxy, step 1: t[b][q] = sum_i Z1[q][i] * x[b][i].
//   fast  : one warp per (q, b), fixed butterfly tree.
//   strict: one thread per (q, b), ascending i, no contraction (bit-exact
//           with approx.hpp:483-488).
// ---------------------------------------------------------------------
template <typename T>
__global__ void __launch_bounds__(256) lr_t_kernel(const T* __restrict__ z1, int r, int d,
                                                   const float* __restrict__ x, int B,
                                                   int strict, float* __restrict__ t) {
  hire_dev::griddep_wait();
  hire_dev::griddep_launch();
  KTrace kt_(kKtLrT);
  if (strict) {
    const int id = blockIdx.x * blockDim.x + threadIdx.x;
    if (id >= r * B) return;
    const int q = id % r, b = id / r;
    const T* zr = z1 + static_cast<int64_t>(q) * d;
    const float* xb = x + static_cast<int64_t>(b) * d;
    float acc = 0.0f;
    for (int i = 0; i < d; ++i) acc = __fadd_rn(acc, __fmul_rn(load_elem<T>(zr, i), xb[i]));
    t[static_cast<int64_t>(b) * r + q] = acc;
    return;
  }
  const int lane = threadIdx.x & 31;
  const int id = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (id >= r * B) return;
  const int q = id % r, b = id / r;
  const T* zr = z1 + static_cast<int64_t>(q) * d;
  const float* xb = x + static_cast<int64_t>(b) * d;
  float acc = 0.0f;
  for (int i = lane; i < d; i += 32) acc = fmaf(load_elem<T>(zr, i), xb[i], acc);
  acc = warp_sum_f32(acc);
  if (lane == 0) t[static_cast<int64_t>(b) * r + q] = acc;
}

// ---------------------------------------------------------------------
// K2 step 2: s[b][j] = phi(sum_q Z2[j][q] * t[b][q]), q ascending — one
// thread per row, the whole row in registers, all queries' t in shared
// memory (broadcast). strict: __fmul_rn/__fadd_rn (bit-exact with
// approx.hpp:489-494); fast: fmaf in the same order.
// ---------------------------------------------------------------------
template <typename T, int R, bool STRICT>
__global__ void __launch_bounds__(128) lr_score_kernel(
    const T* __restrict__ z2, int64_t rows, const float* __restrict__ t, int B, int phi,
    float* __restrict__ scores, int64_t score_stride) {
  hire_dev::griddep_wait();
  hire_dev::griddep_launch();
  KTrace kt_(kKtLrScore);
  extern __shared__ __align__(16) unsigned char smem[];
  float* s_t = reinterpret_cast<float*>(smem);
  block_copy(s_t, t, R * B);
  __syncthreads();
  const int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= rows) return;
  float z[R];
  const T* row = z2 + j * R;
  if constexpr (sizeof(T) == 2) {
#pragma unroll
    for (int v = 0; v < R / 8; ++v) {
      const uint4 u = *reinterpret_cast<const uint4*>(row + 8 * v);
      z[8 * v + 0] = bf16_lo(u.x); z[8 * v + 1] = bf16_hi(u.x);
      z[8 * v + 2] = bf16_lo(u.y); z[8 * v + 3] = bf16_hi(u.y);
      z[8 * v + 4] = bf16_lo(u.z); z[8 * v + 5] = bf16_hi(u.z);
      z[8 * v + 6] = bf16_lo(u.w); z[8 * v + 7] = bf16_hi(u.w);
    }
  } else {
#pragma unroll
    for (int v = 0; v < R / 4; ++v) {
      const float4 u = *reinterpret_cast<const float4*>(row + 4 * v);
      z[4 * v] = u.x; z[4 * v + 1] = u.y; z[4 * v + 2] = u.z; z[4 * v + 3] = u.w;
    }
  }
  for (int b = 0; b < B; ++b) {
    const float* tb = s_t + b * R;
    float acc = 0.0f;
#pragma unroll
    for (int q = 0; q < R; ++q) {
      if constexpr (STRICT) acc = __fadd_rn(acc, __fmul_rn(z[q], tb[q]));
      else acc = fmaf(z[q], tb[q], acc);
    }
    scores[static_cast<int64_t>(b) * score_stride + j] = apply_phi(phi, acc);
  }
}

// ---------------------------------------------------------------------
// K2 step 1, fast: t[b][q] = sum_i Z1[q][i] x[b][i]. grid (r, ceil(B/4)),
// 256 threads; each thread owns 8-element chunks i = 8(tid + 256 j) and up
// to 4 queries; all loads issued up front; fixed-order reduction
// (per-thread chunk order, butterfly, warps in order) -> deterministic.
// ---------------------------------------------------------------------
template <typename T>
__global__ void __launch_bounds__(256) lr_t_fast(const T* __restrict__ z1, int d,
                                                 const float* __restrict__ x, int B, int r,
                                                 float* __restrict__ t) {
  hire_dev::griddep_wait();
  hire_dev::griddep_launch();
  KTrace kt_(kKtLrT);
  __shared__ float s_part[8][4];
  const int q = blockIdx.x, b0 = blockIdx.y * 4;
  const int nb = min(4, B - b0);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const T* zr = z1 + static_cast<int64_t>(q) * d;
  float acc[4] = {0.f, 0.f, 0.f, 0.f};
  for (int ch = threadIdx.x; ch < d / 8; ch += 256) {
    float zf[8];
    if constexpr (sizeof(T) == 2) {
      const uint4 u = *reinterpret_cast<const uint4*>(zr + 8 * ch);
      zf[0] = bf16_lo(u.x); zf[1] = bf16_hi(u.x); zf[2] = bf16_lo(u.y); zf[3] = bf16_hi(u.y);
      zf[4] = bf16_lo(u.z); zf[5] = bf16_hi(u.z); zf[6] = bf16_lo(u.w); zf[7] = bf16_hi(u.w);
    } else {
      const float4 u0 = *reinterpret_cast<const float4*>(zr + 8 * ch);
      const float4 u1 = *reinterpret_cast<const float4*>(zr + 8 * ch + 4);
      zf[0] = u0.x; zf[1] = u0.y; zf[2] = u0.z; zf[3] = u0.w;
      zf[4] = u1.x; zf[5] = u1.y; zf[6] = u1.z; zf[7] = u1.w;
    }
#pragma unroll
    for (int bb = 0; bb < 4; ++bb) {
      if (bb < nb) {
        const float* xb = x + static_cast<int64_t>(b0 + bb) * d + 8 * ch;
        const float4 x0 = *reinterpret_cast<const float4*>(xb);
        const float4 x1 = *reinterpret_cast<const float4*>(xb + 4);
        acc[bb] = fmaf(zf[0], x0.x, acc[bb]); acc[bb] = fmaf(zf[1], x0.y, acc[bb]);
        acc[bb] = fmaf(zf[2], x0.z, acc[bb]); acc[bb] = fmaf(zf[3], x0.w, acc[bb]);
        acc[bb] = fmaf(zf[4], x1.x, acc[bb]); acc[bb] = fmaf(zf[5], x1.y, acc[bb]);
        acc[bb] = fmaf(zf[6], x1.z, acc[bb]); acc[bb] = fmaf(zf[7], x1.w, acc[bb]);
      }
    }
  }
#pragma unroll
  for (int bb = 0; bb < 4; ++bb) {
    const float v = warp_sum_f32(acc[bb]);
    if (lane == 0) s_part[wid][bb] = v;
  }
  __syncthreads();
  if (threadIdx.x < nb) {
    float v = 0.0f;
#pragma unroll
    for (int w8 = 0; w8 < 8; ++w8) v += s_part[w8][threadIdx.x];
    t[static_cast<int64_t>(b0 + threadIdx.x) * r + q] = v;
  }
}

// ---------------------------------------------------------------------
// K2 step 2 on the tensor cores: s[b][j] = phi(sum_q Z2[j][q] t[b][q]).
// mma.sync m16n8k16 bf16 -> fp32. t is split exactly into three bf16 terms
// (hi + mid + lo carry its 24 bits); a bf16 Z2 operand is exact, an fp32 Z2
// is split the same way and the six terms above 2^-24 relative are summed.
// Every product is exact in fp32; only the accumulation order differs from
// the sequential reference (fast mode, within tolerance).
// The k order inside each 32-wide block is permuted consistently for A and
// B so that one 16-byte load per row and block feeds two k-steps:
// lane (g, c) holds row elements 8c..8c+7 of the block; k-step s takes
// elements 4s, 4s+1 as logical k 2c, 2c+1 and 4s+2, 4s+3 as 2c+8, 2c+9.
// One warp per 16-row tile (grid-stride), NTN n-tiles of 8 queries per pass.
// ---------------------------------------------------------------------
__device__ __forceinline__ void mma_bf16(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                         uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

__device__ __forceinline__ void split3_bf16(float v, __nv_bfloat16* o) {
  const __nv_bfloat16 h = __float2bfloat16_rn(v);
  const float r1 = v - __bfloat162float(h);
  const __nv_bfloat16 m = __float2bfloat16_rn(r1);
  const float r2 = r1 - __bfloat162float(m);
  o[0] = h;
  o[1] = m;
  o[2] = __float2bfloat16_rn(r2);
}

__device__ __forceinline__ uint32_t pack_bf16(__nv_bfloat16 lo, __nv_bfloat16 hi) {
  return static_cast<uint32_t>(__bfloat16_as_ushort(lo)) | (static_cast<uint32_t>(__bfloat16_as_ushort(hi)) << 16);
}

constexpr int kLrThreads = 256;

template <typename T, int R>
struct LrTile {
  static constexpr int KB = R / 32;
  static constexpr int NL = sizeof(T) == 2 ? 1 : 2;  // 16-byte loads per row and k block
  uint4 u[KB][2][NL];
  __device__ __forceinline__ void load(const T* z2, int64_t rows, int64_t tile, int g, int c) {
#pragma unroll
    for (int kb = 0; kb < KB; ++kb)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int64_t rr = tile * 16 + g + 8 * h;
#pragma unroll
        for (int l = 0; l < NL; ++l)
          u[kb][h][l] = rr < rows ? ldg_stream(z2 + rr * R + kb * 32 + 8 * c + 4 * l) : make_uint4(0, 0, 0, 0);
      }
  }
};

// NTN n-tiles (<= 8 * NTN queries of the batch, starting at query b0) per
// launch; the B fragments of all (n-tile, k-step, split) live in registers
// for the whole kernel, the NTN accumulator chains interleave.
template <typename T, int R, int NTN>
__global__ void __launch_bounds__(kLrThreads) lr_score_mma(
    const T* __restrict__ z2, int64_t rows, const float* __restrict__ t, int B, int b0, int phi,
    float* __restrict__ scores, int64_t score_stride) {
  constexpr int KB = R / 32;                       // 32-wide k blocks
  constexpr int NS = sizeof(T) == 2 ? 1 : 3;       // A splits
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int g = lane >> 2, c = lane & 3;
  const int64_t tiles = (rows + 15) / 16;
  const int64_t tstride = static_cast<int64_t>(gridDim.x) * (kLrThreads / 32);
  int64_t tile = static_cast<int64_t>(blockIdx.x) * (kLrThreads / 32) + wid;
  // Z2 is not produced by the previous kernel: start streaming the first
  // tile before the programmatic-dependency wait
  LrTile<T, R> cur;
  if (tile < tiles) cur.load(z2, rows, tile, g, c);
  hire_dev::griddep_wait();
  hire_dev::griddep_launch();
  KTrace kt_(kKtLrScore);
  const int nb = min(B - b0, 8 * NTN);
  // t split once per CTA into shared memory in fragment order:
  // s_bf[nt][kb][s2][p][lane] = {pack(t[q][k0], t[q][k0+1]), pack(t[q][k0+2], t[q][k0+3])},
  // q = 8 nt + g, k0 = kb*32 + 8c + 4 s2
  __shared__ uint2 s_bf[NTN][KB][2][3][32];
  for (int i = threadIdx.x; i < NTN * KB * 2 * 32; i += kLrThreads) {
    const int ln = i & 31, s2 = (i >> 5) & 1, kb = (i >> 6) % KB, nt = (i >> 6) / KB;
    const int q = 8 * nt + (ln >> 2);
    const int k0 = kb * 32 + 8 * (ln & 3) + 4 * s2;
    __nv_bfloat16 sp[4][3];
#pragma unroll
    for (int e = 0; e < 4; ++e) split3_bf16(q < nb ? t[static_cast<int64_t>(b0 + q) * R + k0 + e] : 0.0f, sp[e]);
#pragma unroll
    for (int p = 0; p < 3; ++p)
      s_bf[nt][kb][s2][p][ln] = make_uint2(pack_bf16(sp[0][p], sp[1][p]), pack_bf16(sp[2][p], sp[3][p]));
  }
  __syncthreads();
  for (; tile < tiles; tile += tstride) {
    LrTile<T, R> nxt;
    if (tile + tstride < tiles) nxt.load(z2, rows, tile + tstride, g, c);  // next tile in flight
    uint32_t a[KB][NS][2][4];  // [kb][split][row half][bf16 pairs]
#pragma unroll
    for (int kb = 0; kb < KB; ++kb) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        if constexpr (sizeof(T) == 2) {
          const uint4 u = cur.u[kb][h][0];
          a[kb][0][h][0] = u.x; a[kb][0][h][1] = u.y; a[kb][0][h][2] = u.z; a[kb][0][h][3] = u.w;
        } else {
          const uint4 u0 = cur.u[kb][h][0], u1 = cur.u[kb][h][NS > 1 ? 1 : 0];
          const float e[8] = {__uint_as_float(u0.x), __uint_as_float(u0.y), __uint_as_float(u0.z),
                              __uint_as_float(u0.w), __uint_as_float(u1.x), __uint_as_float(u1.y),
                              __uint_as_float(u1.z), __uint_as_float(u1.w)};
          __nv_bfloat16 sp[8][3];
#pragma unroll
          for (int q = 0; q < 8; ++q) split3_bf16(e[q], sp[q]);
#pragma unroll
          for (int p = 0; p < NS; ++p)
#pragma unroll
            for (int w = 0; w < 4; ++w) a[kb][p][h][w] = pack_bf16(sp[2 * w][p], sp[2 * w + 1][p]);
        }
      }
    }
    float acc[NTN][4];
#pragma unroll
    for (int nt = 0; nt < NTN; ++nt) acc[nt][0] = acc[nt][1] = acc[nt][2] = acc[nt][3] = 0.f;
#pragma unroll
    for (int kb = 0; kb < KB; ++kb)
#pragma unroll
      for (int s2 = 0; s2 < 2; ++s2)
#pragma unroll
        for (int pa = 0; pa < NS; ++pa)
#pragma unroll
          for (int pb = 0; pb < 3; ++pb) {
            if (pa + pb > 2) continue;  // terms below 2^-24 relative
#pragma unroll
            for (int nt = 0; nt < NTN; ++nt) {
              const uint2 bq = s_bf[nt][kb][s2][pb][lane];
              mma_bf16(acc[nt], a[kb][pa][0][2 * s2], a[kb][pa][1][2 * s2], a[kb][pa][0][2 * s2 + 1],
                       a[kb][pa][1][2 * s2 + 1], bq.x, bq.y);
            }
          }
    const int64_t r0 = tile * 16 + g, r1 = r0 + 8;
#pragma unroll
    for (int nt = 0; nt < NTN; ++nt) {
      const int q0 = nt * 8 + 2 * c;
      float* o0 = scores + static_cast<int64_t>(b0 + q0) * score_stride;
      if (q0 < nb) {
        if (r0 < rows) o0[r0] = apply_phi(phi, acc[nt][0]);
        if (r1 < rows) o0[r1] = apply_phi(phi, acc[nt][2]);
      }
      if (q0 + 1 < nb) {
        if (r0 < rows) o0[score_stride + r0] = apply_phi(phi, acc[nt][1]);
        if (r1 < rows) o0[score_stride + r1] = apply_phi(phi, acc[nt][3]);
      }
    }
    cur = nxt;
  }
}

// Generic-rank fallback (any r): same arithmetic, row streamed from memory.
template <typename T, bool STRICT>
__global__ void __launch_bounds__(128) lr_score_generic(
    const T* __restrict__ z2, int64_t rows, int r, const float* __restrict__ t, int B, int phi,
    float* __restrict__ scores, int64_t score_stride) {
  hire_dev::griddep_wait();
  hire_dev::griddep_launch();
  KTrace kt_(kKtLrScore);
  extern __shared__ __align__(16) unsigned char smem[];
  float* s_t = reinterpret_cast<float*>(smem);
  block_copy(s_t, t, r * B);
  __syncthreads();
  const int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= rows) return;
  const T* row = z2 + j * r;
  for (int b = 0; b < B; ++b) {
    const float* tb = s_t + b * r;
    float acc = 0.0f;
    for (int q = 0; q < r; ++q) {
      const float zq = load_elem<T>(row, q);
      if constexpr (STRICT) acc = __fadd_rn(acc, __fmul_rn(zq, tb[q]));
      else acc = fmaf(zq, tb[q], acc);
    }
    scores[static_cast<int64_t>(b) * score_stride + j] = apply_phi(phi, acc);
  }
}

}  // namespace hire_dev

namespace hire_dev {


// ---------------------------------------------------------------------
// MMA-tiled int4 layout for the tensor-core proxy (K1-mma). For row-block
// rb (16 rows) and k-block kb (64 columns), 512 bytes; lane l (g = l>>2,
// t = l&3) owns bytes [16l, 16l+16) = words w0..w3 with, for k-tile
// j = w>>1 and half h = w&1:
//   low  nibble of byte p = code(row 16rb+g,   col 64kb + 32j + 16h + 4t + p)
//   high nibble of byte p = code(row 16rb+g+8, col 64kb + 32j + 16h + 4t + p)
// i.e. after (w ^ 0x88888888) the lo/hi masks are exactly the m16n8k32
// A-fragment registers {a0,a1} (h=0) and {a2,a3} (h=1) of k-tile j, offset
// by +8 (unsigned digits 1..15). One 128-bit load per lane feeds 2 MMAs.
// ---------------------------------------------------------------------
__global__ void q4_to_mma_layout(const uint8_t* __restrict__ wq, int64_t pitch, int64_t rows,
                                 int d, uint32_t* __restrict__ out, int64_t n_words) {
  // No early launch_dependents: the proxy kernels that follow stream their
  // first weight tiles BEFORE their griddepcontrol.wait (independent
  // prologue), so the layout they read must be complete when they start.
  hire_dev::griddep_wait();
  const int64_t id = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (id >= n_words) return;
  const int nkb = d / 64;
  const int w = static_cast<int>(id & 3);
  const int lane = static_cast<int>((id >> 2) & 31);
  const int64_t blk = id >> 7;
  const int64_t rb = blk / nkb, kb = blk % nkb;
  const int g = lane >> 2, t = lane & 3;
  const int j = w >> 1, h = w & 1;
  uint32_t word = 0;
#pragma unroll
  for (int p = 0; p < 4; ++p) {
    const int64_t col = kb * 64 + 32 * j + 16 * h + 4 * t + p;
#pragma unroll
    for (int hi = 0; hi < 2; ++hi) {
      const int64_t row = rb * 16 + g + 8 * hi;
      uint32_t nib = 0;
      if (row < rows) {
        const uint8_t byte = wq[row * pitch + col / 2];
        nib = (col & 1) ? (byte >> 4) : (byte & 0xF);
      }
      word |= nib << (8 * p + 4 * hi);
    }
  }
  out[id] = word;
}

__device__ __forceinline__ void mma_u8s8(int (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2,
                                         uint32_t a3, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k32.row.col.s32.u8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

// ---------------------------------------------------------------------
// K1 integer mode on the tensor cores: int4 (as u8 digits c+8) x int8 x
// -> int32, mma.sync m16n8k32. NT n-tiles of 8 queries. A CTA of 8 warps
// owns 8/KS row-blocks; the KS warps of a row-block split its k range and
// their int32 accumulators are summed exactly through shared memory.
// Persistent over row-block groups; x (int8, natural order, padded rows)
// staged in shared memory once per CTA. Exact: identical integers to the
// dp4a path and the oracle.
// ---------------------------------------------------------------------
template <int NT, int KS>
__global__ void __launch_bounds__(256) q4_score_mma(
    const uint4* __restrict__ wmma, int64_t rows, int d, const float* __restrict__ scales,
    const int8_t* __restrict__ xq, const float* __restrict__ sx, const int* __restrict__ sumxq,
    int B, int phi, float* __restrict__ scores, int64_t score_stride) {
  extern __shared__ __align__(16) unsigned char smem[];
  constexpr int RB_PER_CTA = 8 / KS;
  const int xs = d + 16;  // padded query stride (bank spread)
  int8_t* s_x = reinterpret_cast<int8_t*>(smem);
  int* s_acc = reinterpret_cast<int*>(smem + static_cast<size_t>(NT) * 8 * xs);  // [8 warps][NT][4][32]
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int nkb = d / 64;
  const int64_t n_rb = (rows + 15) / 16;
  const int rb_local = wid / KS, ks = wid % KS;
  const int kb0 = ks * nkb / KS, kb1 = (ks + 1) * nkb / KS;

  // prologue independent of the producer kernel: first weight loads
  int64_t rb = static_cast<int64_t>(blockIdx.x) * RB_PER_CTA + rb_local;
  const int64_t rb_stride = static_cast<int64_t>(gridDim.x) * RB_PER_CTA;
  constexpr int U = 4;
  uint4 a[U];
  if (rb < n_rb) {
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (kb0 + u < kb1) a[u] = ldg_stream(wmma + ((rb * nkb + kb0 + u) * 32 + lane));
  }
  griddep_wait();  // x quantisation (prep_x_int8_kernel) is complete
  LateTrigger late_trigger_;
  KTrace kt_(kKtProxy);
  for (int i = threadIdx.x; i < NT * 8 * (d / 16); i += blockDim.x) {
    const int n = i / (d / 16), c = i % (d / 16);
    int4 v = make_int4(0, 0, 0, 0);
    if (n < B) v = *reinterpret_cast<const int4*>(xq + static_cast<int64_t>(n) * d + c * 16);
    *reinterpret_cast<int4*>(s_x + n * xs + c * 16) = v;
  }
  __syncthreads();

  for (int64_t rb_base = static_cast<int64_t>(blockIdx.x) * RB_PER_CTA; rb_base < n_rb; rb_base += rb_stride) {
    rb = rb_base + rb_local;
    int acc[NT][4];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) acc[nt][0] = acc[nt][1] = acc[nt][2] = acc[nt][3] = 0;
    // the two row scales of this lane: in flight during the k loop (loaded at
    // their use they stalled the epilogue on an L2 round trip per row block)
    float rs_lo = 0.0f, rs_hi = 0.0f;
    if (ks == 0 && rb < n_rb) {
      const int64_t r0 = rb * 16 + g;
      if (r0 < rows) rs_lo = scales[r0];
      if (r0 + 8 < rows) rs_hi = scales[r0 + 8];
    }
    if (rb < n_rb) {
      for (int kb = kb0; kb < kb1; kb += U) {
        uint4 nxt[U];
#pragma unroll
        for (int u = 0; u < U; ++u)
          if (kb + U + u < kb1) nxt[u] = ldg_stream(wmma + ((rb * nkb + kb + U + u) * 32 + lane));
#pragma unroll
        for (int u = 0; u < U; ++u) {
          if (kb + u >= kb1) break;
          const uint32_t w4[4] = {a[u].x, a[u].y, a[u].z, a[u].w};
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
        for (int u = 0; u < U; ++u) a[u] = nxt[u];
      }
    }
    // next row-block's first loads (software pipeline across row-blocks)
    const int64_t rbn = rb + rb_stride;
    if (rbn < n_rb) {
#pragma unroll
      for (int u = 0; u < U; ++u)
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
    if (ks == 0 && rb < n_rb) {
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int64_t row = rb * 16 + g + ((e & 2) ? 8 : 0);
          const int n = nt * 8 + 2 * t + (e & 1);
          if (row < rows && n < B) {
            const int aint = acc[nt][e] - 8 * sumxq[n];
            const float cs = __fmul_rn((e & 2) ? rs_hi : rs_lo, sx[n]);
            scores[static_cast<int64_t>(n) * score_stride + row] =
                apply_phi(phi, __fmul_rn(static_cast<float>(aint), cs));
          }
        }
    }
  }
  if (g_ktrace) {  // spread of CTA end times (debug timeline)
    __syncthreads();
    if (threadIdx.x == 0) {
      atomicMin(&g_ktrace[54], gtimer());
      atomicMax(&g_ktrace[55], gtimer());
    }
  }
}

}  // namespace hire_dev
