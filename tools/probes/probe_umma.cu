// Probe: tcgen05.mma kind::i8 with A (u8) in TMEM and B (s8) in shared
// memory (K-major, no swizzle), D s32 in TMEM. Checks the operand layouts
// the q4 UMMA proxy kernel relies on against a CPU product, for N = 8..64.
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -o probe_umma probe_umma.cu
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../../paper_2402_09360_b200/csrc/umma.cuh"

using namespace hire_dev;

__global__ void probe(const uint8_t* A, const int8_t* Bm, int32_t* D, int K, int N, int a_signed) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t taddr_s;
  __shared__ __align__(8) uint64_t bar;
  const int t = threadIdx.x, w = t / 32;
  // B -> core-matrix layout: offset(n,k) = (k/16)*(N*16) + (n/8)*128 + (n%8)*16 + k%16
  for (int i = t; i < N * K; i += blockDim.x) {
    const int n = i / K, k = i % K;
    sm[(k / 16) * (N * 16) + (n / 8) * 128 + (n % 8) * 16 + (k % 16)] = static_cast<uint8_t>(Bm[i]);
  }
  if (w == 0) {
    umma::tmem_alloc(&taddr_s, 256);
    umma::tmem_relinquish();
  }
  if (t == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  fence_proxy_async_smem();  // generic smem writes -> async proxy (MMA reads)
  umma::fence_before();
  __syncthreads();
  umma::fence_after();
  const uint32_t tm = taddr_s;
  // A row t -> lane t: column c holds bytes A[t][4c .. 4c+3]
  const uint32_t lane_base = static_cast<uint32_t>(32 * w) << 16;
  for (int c0 = 0; c0 < K / 4; c0 += 8) {
    uint32_t r[8];
    for (int j = 0; j < 8; ++j) {
      const uint8_t* p = A + static_cast<size_t>(t) * K + 4 * (c0 + j);
      r[j] = p[0] | (p[1] << 8) | (p[2] << 16) | (p[3] << 24);
    }
    umma::st_32x32b_x8(tm + lane_base + c0, r);
  }
  umma::wait_st();
  umma::fence_before();
  __syncthreads();
  if (t == 0) {
    umma::fence_after();
    const uint32_t idesc = umma::idesc_i8(128, N, a_signed != 0, true);
    const uint32_t sbase = smem_u32(sm);
    for (int s = 0; s < K / 32; ++s) {
      const uint64_t bd = umma::sdesc_kmajor_noswz(sbase + 2 * s * N * 16, N * 16, 128);
      umma::mma_i8_ts(tm + 128, tm + 8 * s, bd, idesc, s > 0);
    }
    umma::commit(&bar);
  }
  mbar_wait(&bar, 0);
  umma::fence_after();
  for (int c0 = 0; c0 < N; c0 += 8) {
    uint32_t r[8];
    umma::ld_32x32b_x8(tm + lane_base + 128 + c0, r);
    umma::wait_ld();
    for (int j = 0; j < 8; ++j) D[t * N + c0 + j] = static_cast<int32_t>(r[j]);
  }
  umma::fence_before();
  __syncthreads();
  if (w == 0) umma::tmem_dealloc(tm, 256);
}

int main() {
  const int K = 256;
  int bad_total = 0;
  for (int a_signed = 0; a_signed < 2; ++a_signed)
    for (int N : {8, 16, 32, 48, 64}) {
      std::vector<uint8_t> A(128 * K);
      std::vector<int8_t> Bm(N * K);
      srand(N * 7 + a_signed);
      for (auto& v : A) v = a_signed ? static_cast<uint8_t>(static_cast<int8_t>(rand() % 15 - 7)) : rand() % 16;
      for (auto& v : Bm) v = static_cast<int8_t>(rand() % 255 - 127);
      uint8_t* dA;
      int8_t* dB;
      int32_t* dD;
      cudaMalloc(&dA, A.size());
      cudaMalloc(&dB, Bm.size());
      cudaMalloc(&dD, 128 * N * 4);
      cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice);
      cudaMemcpy(dB, Bm.data(), Bm.size(), cudaMemcpyHostToDevice);
      cudaMemset(dD, 0, 128 * N * 4);
      const int smem = N * K;
      cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
      probe<<<1, 128, smem>>>(dA, dB, dD, K, N, a_signed);
      cudaError_t e = cudaDeviceSynchronize();
      std::vector<int32_t> D(128 * N);
      cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
      int bad = 0;
      for (int m = 0; m < 128; ++m)
        for (int n = 0; n < N; ++n) {
          int64_t s = 0;
          for (int k = 0; k < K; ++k)
            s += (a_signed ? static_cast<int>(static_cast<int8_t>(A[m * K + k])) : static_cast<int>(A[m * K + k])) *
                 static_cast<int>(Bm[n * K + k]);
          if (s != D[m * N + n]) {
            if (bad < 4) printf("  m=%d n=%d got %d want %lld\n", m, n, D[m * N + n], (long long)s);
            ++bad;
          }
        }
      printf("a_signed=%d N=%d: %s, %d mismatches of %d\n", a_signed, N, cudaGetErrorString(e), bad, 128 * N);
      bad_total += bad + (e != cudaSuccess);
      cudaFree(dA);
      cudaFree(dB);
      cudaFree(dD);
      if (e != cudaSuccess) return 2;
    }
  printf(bad_total ? "PROBE FAIL\n" : "PROBE OK\n");
  return bad_total ? 1 : 0;
}
