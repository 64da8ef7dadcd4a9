// common.cuh — shared device helpers for the HiRE sm_100a kernels.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

// Kernels kept only as measured negative results (DESIGN.md "What B200
// taught this design") are compiled in with -DHIRE_EXPERIMENTS=1; the
// product library leaves them out.
#ifndef HIRE_EXPERIMENTS
#define HIRE_EXPERIMENTS 0
#endif

namespace hire_dev {

constexpr int kWarp = 32;

enum Phi : int { kIdentity = 0, kRelu = 1, kSqRelu = 2 };

// linalg.hpp:31-38 (apply_activation).
__device__ __forceinline__ float apply_phi(int phi, float z) {
  if (phi == kRelu) return z > 0.0f ? z : 0.0f;
  if (phi == kSqRelu) return z > 0.0f ? __fmul_rn(z, z) : 0.0f;
  return z;
}

// ---------------------------------------------------------------------
// Rank keys. The reference orders every selection by value descending,
// ties by ascending index (linalg.hpp:129-133, `va != vb` so -0 == +0).
// A 64-bit key = orderable(value) << 32 | (0xFFFFFFFF - index) turns that
// total order into plain unsigned '>' : larger key ranks first. Key 0 never
// encodes a real (non-NaN) score and is used as padding.
// ---------------------------------------------------------------------
__host__ __device__ __forceinline__ uint32_t ord_of(float v) {
  uint32_t u;
#ifdef __CUDA_ARCH__
  u = __float_as_uint(v);
#else
  __builtin_memcpy(&u, &v, 4);
#endif
  if (u == 0x80000000u) u = 0;  // -0.0 ranks equal to +0.0
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

__host__ __device__ __forceinline__ float value_of_ord(uint32_t o) {
  const uint32_t u = (o & 0x80000000u) ? (o & 0x7FFFFFFFu) : ~o;
#ifdef __CUDA_ARCH__
  return __uint_as_float(u);
#else
  float f;
  __builtin_memcpy(&f, &u, 4);
  return f;
#endif
}

__host__ __device__ __forceinline__ uint64_t make_key(float v, uint32_t idx) {
  return (static_cast<uint64_t>(ord_of(v)) << 32) | (0xFFFFFFFFu - idx);
}
__host__ __device__ __forceinline__ uint32_t key_index(uint64_t k) {
  return 0xFFFFFFFFu - static_cast<uint32_t>(k);
}
__host__ __device__ __forceinline__ float key_value(uint64_t k) {
  return value_of_ord(static_cast<uint32_t>(k >> 32));
}

// ------------------------------------------- programmatic dependent launch --
// Every kernel is launched with programmatic stream serialization: it may be
// scheduled while its predecessor drains, and waits here (griddepcontrol
// .wait) before touching anything the predecessor wrote. launch_dependents
// lets the next kernel in the chain get scheduled early.
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void griddep_launch() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
// Wide kernels (a CTA wave over the whole GPU) trigger their dependents when
// they finish, not when they start: dependents launched early are packed onto
// the first SMs that drain, and the small per-query kernels that follow (one
// CTA per query, barrier- and shuffle-bound) then share an SM (measured: cfg3
// B=32 final top-k CTAs 4.8 .. 9.9 us packed, 4.7 .. 5.5 us spread). Narrow
// kernels trigger at once, so the wide kernel after them is resident early.
struct LateTrigger {
  __device__ __forceinline__ ~LateTrigger() { griddep_launch(); }
};

// ------------------------------------------------- kernel timeline trace --
// Debug aid (hire_debug_ktrace): when g_ktrace is set, thread 0 of every CTA
// records min(start) / max(end) %globaltimer per kernel id.
__device__ unsigned long long* g_ktrace = nullptr;
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
struct KTrace {
  int id;
  __device__ __forceinline__ explicit KTrace(int i) : id(i) {
    unsigned long long* t = g_ktrace;
    if (t && threadIdx.x == 0) atomicMin(t + 2 * id, gtimer());
  }
  __device__ __forceinline__ ~KTrace() {
    unsigned long long* t = g_ktrace;
    if (t && threadIdx.x == 0) atomicMax(t + 2 * id + 1, gtimer());
  }
};
enum KtId { kKtPivot = 0, kKtWindow = 1, kKtWindowSel = 2, kKtEmit = 3, kKtFinal = 4, kKtRecompute = 5,
            kKtProxy = 6, kKtGather = 7, kKtPrep = 8, kKtLrT = 9, kKtLrScore = 10, kKtDown = 11,
            kKtNum = 32 };

// ------------------------------------------------ cross-CTA flag access --
// Polling with ld.acquire costs an L1 invalidate (CCTL.IVALL) per probe;
// spin with relaxed loads and fence once after the flag is seen.
__device__ __forceinline__ unsigned ld_relaxed_gpu(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_gpu(unsigned* p, unsigned v) {
  asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void fence_acq_rel_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }

// ------------------------------------------- bulk async copies (TMA 1D) --
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
// make mbarrier inits visible to the async proxy (TMA completes on them)
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
// order this thread's generic-proxy smem accesses before later async-proxy ones
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
// global -> shared bulk copy (bytes % 16 == 0, both 16-B aligned), completes on bar
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// bulk L2 prefetch of [src, src + bytes) (bytes % 16 == 0, 16-B aligned)
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned phase) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}

// --------------------------------------------------------------- loads --
// Weight streams (proxy codes, gathered rows): no L1 allocation.
// HIRE_L2_HINT=1 adds an L2 evict-first policy (measured slower on B200).
#ifndef HIRE_L2_HINT
#define HIRE_L2_HINT 0  // measured: slower proxy stream, no downstream gain (kept opt-in)
#endif
__device__ __forceinline__ uint4 ldg_stream(const void* p) {
  uint4 r;
#if HIRE_L2_HINT
  asm("{\n\t.reg .b64 pol;\n\t"
      "createpolicy.fractional.L2::evict_first.b64 pol, 1.0;\n\t"
      "ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], pol;\n\t}"
      : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
      : "l"(p));
#else
  asm("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
#endif
  return r;
}

__device__ __forceinline__ float bf16_lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf16_hi(uint32_t w) { return __uint_as_float(w & 0xFFFF0000u); }

// ------------------------------------------------- block staging copies --
// Global -> shared copies with U loads in flight per thread (a plain
// `for (i = tid; ...) dst[i] = src[i]` loop serialises one L2/HBM latency
// per iteration because each store waits for its load).
template <int U = 8, typename T, typename F>
__device__ __forceinline__ void block_copy_tf(T* __restrict__ dst, int n, F load) {
  for (int i0 = threadIdx.x; i0 < n; i0 += static_cast<int>(blockDim.x) * U) {
    T v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i = i0 + u * static_cast<int>(blockDim.x);
      if (i < n) v[u] = load(i);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i = i0 + u * static_cast<int>(blockDim.x);
      if (i < n) dst[i] = v[u];
    }
  }
}
template <int U = 8, typename T>
__device__ __forceinline__ void block_copy(T* __restrict__ dst, const T* __restrict__ src, int n) {
  block_copy_tf<U, T>(dst, n, [&](int i) { return src[i]; });
}
template <int U = 8, typename T>
__device__ __forceinline__ void block_copy_cg(T* __restrict__ dst, const T* __restrict__ src, int n) {
  block_copy_tf<U, T>(dst, n, [&](int i) { return __ldcg(src + i); });
}

// ------------------------------------------------------ warp reductions --
__device__ __forceinline__ int warp_sum_i32(int v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Fixed butterfly tree: identical association on every call, every launch
// configuration — so every exact-score producer that uses it (gather
// recompute, dense exact, FFN activations) yields bit-identical values.
__device__ __forceinline__ float warp_sum_f32(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = __fadd_rn(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

__device__ __forceinline__ float warp_max_f32(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

__device__ __forceinline__ uint64_t warp_max_u64(uint64_t v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const uint64_t w = __shfl_xor_sync(0xffffffffu, v, o);
    v = w > v ? w : v;
  }
  return v;
}

template <typename T>
__device__ __forceinline__ float load_elem(const T* p, int64_t i);
template <>
__device__ __forceinline__ float load_elem<float>(const float* p, int64_t i) { return p[i]; }
template <>
__device__ __forceinline__ float load_elem<__nv_bfloat16>(const __nv_bfloat16* p, int64_t i) {
  return __bfloat162float(p[i]);
}

// Round half away from zero, clamped — approx.hpp:41-45. `v + 0.5f` is one
// IEEE fp32 add exactly as on the host.
__device__ __forceinline__ int rhaz_clamp(float v, int lim) {
  const float r = v >= 0.0f ? floorf(__fadd_rn(v, 0.5f)) : ceilf(__fsub_rn(v, 0.5f));
  int c = static_cast<int>(r);
  return c < -lim ? -lim : (c > lim ? lim : c);
}

}  // namespace hire_dev
