// gather_bench.cuh — device side of the group-gather microbenchmark
// (reference gather_bench.hpp:71-152): the source buffer filled with the
// reference Rng's Gaussian stream (rng.hpp:20-61), a group gather (one CTA
// per selected group, 128-bit copies) and a contiguous copy of the same
// bytes, and the reference's FNV-1a checksum per group.
#pragma once
#include <cstdint>

#include "common.cuh"

namespace hire_dev {

__host__ __device__ __forceinline__ uint64_t rng_mix64(uint64_t seed, uint64_t counter) {
  uint64_t z = seed + counter * 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

// element i of Rng(seed).next_gaussian_f() stream: pair p = i / 2 uses the
// uniforms of counters 2p + 1, 2p + 2; even i = the cosine member, odd i =
// the cached sine member
__global__ void gb_fill_kernel(float* __restrict__ src, int64_t n, uint64_t seed) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint64_t p = static_cast<uint64_t>(i >> 1);
  const double u1 = static_cast<double>(rng_mix64(seed, 2 * p + 1) >> 11) * 0x1.0p-53;
  const double u2 = static_cast<double>(rng_mix64(seed, 2 * p + 2) >> 11) * 0x1.0p-53;
  const double radius = sqrt(-2.0 * log1p(-u1));
  const double angle = 2.0 * 3.141592653589793238462643383279502884 * u2;
  src[i] = static_cast<float>((i & 1) ? radius * sin(angle) : radius * cos(angle));
}

// dst[i] = group ids[i] of src, group_elems floats: a flat grid-stride over
// the selected 16-byte vectors (every group spread over many threads,
// consecutive threads on consecutive vectors of a group)
__global__ void gb_gather_kernel(const float* __restrict__ src, const uint32_t* __restrict__ ids, int64_t n_sel,
                                 int64_t group_elems, float* __restrict__ dst) {
  if ((group_elems & 3) == 0) {
    const int64_t ge4 = group_elems / 4, n4 = n_sel * ge4;
    const float4* s4 = reinterpret_cast<const float4*>(src);
    float4* d4 = reinterpret_cast<float4*>(dst);
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n4;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
      const int64_t gi = i / ge4, e = i - gi * ge4;
      d4[i] = __ldcs(s4 + static_cast<int64_t>(ids[gi]) * ge4 + e);
    }
  } else {
    const int64_t n = n_sel * group_elems;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
      const int64_t gi = i / group_elems, e = i - gi * group_elems;
      dst[i] = src[static_cast<int64_t>(ids[gi]) * group_elems + e];
    }
  }
}

// the dense baseline: one contiguous copy of the same byte count
__global__ void gb_copy_kernel(const float4* __restrict__ src, float4* __restrict__ dst, int64_t n4) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n4;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    dst[i] = __ldcs(src + i);
}

// FNV-1a over the float bits of each group (gather_bench.hpp:52-61)
__global__ void gb_checksum_kernel(const float* __restrict__ buf, const uint32_t* __restrict__ ids, int64_t n_sel,
                                   int64_t group_elems, uint64_t* __restrict__ out) {
  const int64_t gi = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (gi >= n_sel) return;
  const float* a = buf + (ids ? static_cast<int64_t>(ids[gi]) : gi) * group_elems;
  uint64_t h = 0xCBF29CE484222325ULL;
  for (int64_t e = 0; e < group_elems; ++e) h = (h ^ __float_as_uint(a[e])) * 0x100000001B3ULL;
  out[gi] = h;
}

}  // namespace hire_dev
