// Throughput probes for the K2-TC building blocks on B200: back-to-back tcgen05.mma
// (kind::tf32, M=128, A in TMEM, B K-major smem) for several N, and tcgen05.st x8 / ld x16.
#include <cstdio>
#include <cstdint>
#include "../../paper_2402_14118_b200/csrc/tc_ptx.cuh"
using namespace mmmcu;

__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile("{\n\t.reg .pred P1;\n\telect.sync _|P1, 0xffffffff;\n\tselp.b32 %0, 1, 0, P1;\n\t}" : "=r"(pred));
  return pred != 0;
}
__global__ void k_mma_warp_rate(int n_mma, int N, long long* cycles) {
  __shared__ __align__(1024) uint8_t sB[8192];
  __shared__ uint64_t bar;
  __shared__ uint32_t tb;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 8192 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sB)[i] = 0x3f800000u;
  if (warp == 0) tc::tmem_alloc(&tb, 512);
  if (tid == 0) { tc::mbar_init(&bar, 1); tc::fence_mbar_init(); }
  tc::fence_async_smem();
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t base = tb;
  if (warp == 0) {
    const uint32_t idesc = tc::idesc_tf32_m128(N);
    const uint64_t desc = tc::smem_desc(tc::smem_u32(sB), (N / 8) * 128, 128);
    long long t0 = clock64();
    for (int i = 0; i < n_mma; ++i) {
      const uint32_t d = base + (uint32_t)((i % 8) * 16);
      const uint32_t a = base + 256 + (uint32_t)(i % 16) * 8;
      if (elect_one()) tc::mma_tf32_ts(d, a, desc, idesc, 1);
      __syncwarp();
    }
    if (elect_one()) tc::mma_commit(&bar);
    __syncwarp();
    tc::mbar_wait(&bar, 0);
    long long t1 = clock64();
    if (tid == 0) cycles[0] = t1 - t0;
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(base, 512);
}

__global__ void k_mma_rate(int n_mma, int N, long long* cycles, int same_d) {
  __shared__ __align__(1024) uint8_t sB[8192];
  __shared__ uint64_t bar;
  __shared__ uint32_t tb;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 8192 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sB)[i] = 0x3f800000u;
  if (warp == 0) tc::tmem_alloc(&tb, 512);
  if (tid == 0) { tc::mbar_init(&bar, 1); tc::fence_mbar_init(); }
  tc::fence_async_smem();
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t base = tb;
  if (tid == 0) {
    const uint32_t idesc = tc::idesc_tf32_m128(N);
    const uint64_t desc = tc::smem_desc(tc::smem_u32(sB), (N / 8) * 128, 128);
    long long t0 = clock64();
    if (same_d >= 2) {
      const int nd = same_d == 2 ? 4 : same_d == 3 ? 16 : 1;  // distinct accumulators (N=16 apart)
      for (int i = 0; i < n_mma; i += 16) {
#pragma unroll
        for (int u = 0; u < 16; ++u) tc::mma_tf32_ts(base + (u % nd) * 16, base + 256 + u * 8, desc, idesc, 1);
      }
    } else {
    for (int i = 0; i < n_mma; ++i) {
      const uint32_t d = same_d ? base : base + (uint32_t)((i % 8) * N) % 256;
      tc::mma_tf32_ts(d, base + 256 + (i % 16) * 8, desc, idesc, 1);
    }
    }
    tc::mma_commit(&bar);
    tc::mbar_wait(&bar, 0);
    long long t1 = clock64();
    cycles[0] = t1 - t0;
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(base, 512);
}

__device__ __forceinline__ void mma_tf32_ss(uint32_t d_taddr, uint64_t a_desc, uint64_t b_desc, uint32_t idesc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 1, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_taddr), "l"(a_desc),
               "l"(b_desc), "r"(idesc) : "memory");
}
__device__ __forceinline__ void mma_f16_ss(uint32_t d_taddr, uint64_t a_desc, uint64_t b_desc, uint32_t idesc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 1, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_taddr), "l"(a_desc),
               "l"(b_desc), "r"(idesc) : "memory");
}
__global__ void k_mma_ss_rate(int n_mma, int N, long long* cycles, int kind) {
  __shared__ __align__(1024) uint8_t sA[4096 * 4];
  __shared__ __align__(1024) uint8_t sB[8192];
  __shared__ uint64_t bar;
  __shared__ uint32_t tb;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 4096; i += blockDim.x) reinterpret_cast<uint32_t*>(sA)[i] = 0x3f800000u;
  for (int i = tid; i < 8192 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sB)[i] = 0x3f800000u;
  if (warp == 0) tc::tmem_alloc(&tb, 512);
  if (tid == 0) { tc::mbar_init(&bar, 1); tc::fence_mbar_init(); }
  tc::fence_async_smem();
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t base = tb;
  if (tid == 0) {
    uint32_t idesc = tc::idesc_tf32_m128(N);
    if (kind == 1) idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((128u >> 4) << 24);  // bf16
    const uint64_t adesc = tc::smem_desc(tc::smem_u32(sA), 2048, 128);
    const uint64_t bdesc = tc::smem_desc(tc::smem_u32(sB), (N / 8) * 128, 128);
    long long t0 = clock64();
    for (int i = 0; i < n_mma; ++i) {
      const uint32_t d = base + (uint32_t)((i % 2) * 256);
      if (kind == 0) mma_tf32_ss(d, adesc, bdesc, idesc);
      else mma_f16_ss(d, adesc, bdesc, idesc);
    }
    tc::mma_commit(&bar);
    tc::mbar_wait(&bar, 0);
    long long t1 = clock64();
    cycles[0] = t1 - t0;
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(base, 512);
}

__global__ void k_st_rate(int n, long long* cycles) {
  __shared__ uint32_t tb;
  const int tid = threadIdx.x, warp = tid >> 5;
  if (warp == 0) tc::tmem_alloc(&tb, 512);
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t base = tb + ((uint32_t)(32 * (warp & 3)) << 16);
  uint32_t v[8] = {1, 2, 3, 4, 5, 6, 7, 8};
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    tc::tmem_st8(base + (i % 64) * 8, v);
    if ((i & 3) == 3) tc::tmem_st_wait();
  }
  tc::tmem_st_wait();
  long long t1 = clock64();
  if (tid == 0) cycles[1] = t1 - t0;
  uint32_t w[16];
  t0 = clock64();
  for (int i = 0; i < n; ++i) {
    tc::tmem_ld16(base + (i % 32) * 16, w);
    tc::tmem_ld_wait();
    v[0] += w[i & 15];
  }
  t1 = clock64();
  if (tid == 0) cycles[2] = t1 - t0;
  if (v[0] == 12345) cycles[3] = 1;
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(tb, 512);
}

int main() {
  long long* d; cudaMalloc(&d, 64); long long h[8];
  for (int N : {16, 32, 64, 128, 192, 256}) for (int same : {4, 2, 3}) {
    k_mma_rate<<<1, 128>>>(4096, N, d, same);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost);
    printf("mma tf32 M128 N%3d same_d=%d: %s %.1f cycles/MMA (ideal %.1f)\n", N, same, cudaGetErrorString(e), h[0] / 4096.0, 128.0 * N * 8 / 2048);
  }
  for (int N : {16, 32, 64, 128, 256}) {
    k_mma_warp_rate<<<1, 128>>>(4096, N, d);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost);
    printf("mma TS warp-converged+elect N%3d: %s %.1f cycles/MMA (ideal %.1f)\n", N, cudaGetErrorString(e), h[0] / 4096.0, 128.0 * N * 8 / 2048);
  }
  for (int kind : {0, 1}) for (int N : {16, 64, 128, 256}) {
    k_mma_ss_rate<<<1, 128>>>(4096, N, d, kind);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost);
    printf("mma SS %s M128 N%3d: %s %.1f cycles/MMA (ideal %.1f)\n", kind ? "bf16 K16" : "tf32 K8", N, cudaGetErrorString(e), h[0] / 4096.0, 128.0 * N * 8 / 2048);
  }
  for (int warps : {4, 8}) {
    k_st_rate<<<1, 32 * warps>>>(4096, d);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, d, 32, cudaMemcpyDeviceToHost);
    printf("warps=%d: tcgen05.st x8 (+wait every 4): %.1f cycles each per warp; tcgen05.ld x16 + wait: %.1f cycles (%s)\n", warps, h[1] / 4096.0, h[2] / 4096.0, cudaGetErrorString(e));
  }
  return 0;
}
