// Probe: issue rate of tcgen05.mma kind::i8 (M=128) with A in TMEM (TS) or
// in shared memory (SS), B in shared memory, for N = 16..64, with and
// without a tcgen05.commit every 8 MMAs. One CTA per SM, all SMs; prints
// cycles per MMA. Informs score_umma.cuh's pipeline design.
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -o probe_umma_rate probe_umma_rate.cu
#include <cstdio>
#include <vector>

#include "../../paper_2402_09360_b200/csrc/umma.cuh"

using namespace hire_dev;

__device__ __forceinline__ void mma_i8_ss(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                          uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, {%5, %6, %7, %8}, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(acc), "r"(0u), "r"(0u), "r"(0u), "r"(0u)
      : "memory");
}

// mode 0: TS, one commit at the end; 1: TS, commit every 8 and wait for the
// commit 4 groups back; 2: SS one commit; 3: SS commit every 8 + wait 4 back
__global__ void rate(int N, int n_mma, int mode, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t taddr_s;
  __shared__ __align__(8) uint64_t bars[4];
  const int t = threadIdx.x, w = t / 32;
  for (int i = t; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = i * 2654435761u;
  if (w == 0) {
    umma::tmem_alloc(&taddr_s, 512);
    umma::tmem_relinquish();
  }
  if (t == 0) {
    for (int i = 0; i < 4; ++i) mbar_init(&bars[i], 1);
    fence_mbar_init();
  }
  fence_proxy_async_smem();
  umma::fence_before();
  __syncthreads();
  umma::fence_after();
  const uint32_t tm = taddr_s;
  if (mode >= 4) {  // 4: (mode-3) issuer warps, TS, one commit each
    const int nw = mode - 3;
    if (w < nw && (t & 31) == 0) {
      const uint32_t idesc = umma::idesc_i8(128, N, false, true);
      const uint32_t base = smem_u32(sm);
      long long t0 = clock64();
      for (int i = 0; i < n_mma / nw; ++i) {
        const int kc = i & 15;
        const uint64_t bd = umma::sdesc_kmajor_noswz(base + 32768 + (kc & 7) * 256, 128, 8 * 2048 / 8);
        umma::mma_i8_ts(tm + 256 + 64 * w, tm + 8 * (kc & 31), bd, idesc, i > 0);
      }
      umma::commit(&bars[w]);
      mbar_wait(&bars[w], 0);
      long long t1 = clock64();
      if (blockIdx.x == 0 && w == 0) out[0] = t1 - t0;
    }
  } else if (t == 0) {
    const uint32_t idesc = umma::idesc_i8(128, N, false, true);
    const uint32_t base = smem_u32(sm);
    long long t0 = clock64();
    int grp = 0;
    for (int i = 0; i < n_mma; ++i) {
      const int kc = i & 15;
      const uint64_t bd = umma::sdesc_kmajor_noswz(base + 32768 + (kc & 7) * 256, 128, 8 * 2048 / 8);
      if (mode < 2) {
        umma::mma_i8_ts(tm + 256, tm + 8 * (kc & 31), bd, idesc, i > 0);
      } else {
        const uint64_t ad = umma::sdesc_kmajor_noswz(base + kc * 256, 128, 4096);
        mma_i8_ss(tm + 256, ad, bd, idesc, i > 0);
      }
      if ((mode & 1) && (i & 7) == 7) {
        umma::commit(&bars[grp & 3]);
        if (grp >= 3) mbar_wait(&bars[(grp - 3) & 3], ((grp - 3) >> 2) & 1);
        ++grp;
      }
    }
    umma::commit(&bars[grp & 3]);
    mbar_wait(&bars[grp & 3], (grp >> 2) & 1);
    long long t1 = clock64();
    if (blockIdx.x == 0) out[0] = t1 - t0;
  }
  umma::fence_before();
  __syncthreads();
  if (w == 0) umma::tmem_dealloc(tm, 512);
}

int main() {
  long long* d;
  cudaMalloc(&d, 8);
  cudaFuncSetAttribute(rate, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  const int n = 4096;
  for (int mode = 0; mode < 8; ++mode)
    for (int N : {16, 32, 64}) {
      rate<<<148, 128, 64 * 1024>>>(N, n, mode, d);
      cudaError_t e = cudaDeviceSynchronize();
      long long c = 0;
      cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
      printf("mode=%d (%s, %s) N=%3d: %.1f cycles per MMA (%s)\n", mode, mode < 2 || mode >= 4 ? "A in TMEM" : "A in smem",
             mode >= 4 ? "several issuer warps" : (mode & 1) ? "commit/8 + wait 4 back" : "one commit", N,
             double(c) / n, cudaGetErrorString(e));
      if (e != cudaSuccess) return 1;
    }
  return 0;
}
