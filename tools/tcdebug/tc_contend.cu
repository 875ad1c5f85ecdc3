// Does anything else running on the SM slow down back-to-back tcgen05.mma (kind::tf32, M=128,
// A in TMEM, B K-major in smem)?  mode bits: 1 = 4 warps tcgen05.st into TMEM continuously,
// 2 = 4 warps write shared memory continuously (STS.128), 4 = 4 warps read shared memory.
#include <cstdio>
#include <cstdint>
#include "../../paper_2402_14118_b200/csrc/tc_ptx.cuh"
using namespace mmmcu;

__global__ void k(int n_mma, int N, int lbo, int sbo, int mode, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* sB = sm;                  // 32 KB
  float4* sX = reinterpret_cast<float4*>(sm + 32768);  // 64 KB scratch for the smem traffic warps
  __shared__ uint64_t bar;
  __shared__ uint64_t cbar[8];
  __shared__ uint32_t tb;
  __shared__ volatile int stop;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 32768 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sB)[i] = 0x3f800000u;
  if (warp == 0) tc::tmem_alloc(&tb, 512);
  if (tid == 0) { tc::mbar_init(&bar, 1); for (int q = 0; q < 8; ++q) tc::mbar_init(&cbar[q], 1); tc::fence_mbar_init(); stop = 0; }
  tc::fence_async_smem();
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t base = tb;
  if (warp == 4) {
    if ((tid & 31) == 0) {
      const uint32_t idesc = tc::idesc_tf32_m128(N);
      const uint64_t desc = tc::smem_desc(tc::smem_u32(sB), lbo, sbo);
      long long t0 = clock64();
      for (int i = 0; i < n_mma; ++i) {
        tc::mma_tf32_ts(base, base + 384 + (i % 8) * 16, desc, idesc, 1);
        if ((mode & 8) && i % 3 == 2) tc::mma_commit(&cbar[(i / 3) % 8]);
        if ((mode & 16) && i % 3 == 2) asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      }
      tc::mma_commit(&bar);
      tc::mbar_wait(&bar, 0);
      out[0] = clock64() - t0;
      stop = 1;
    }
    __syncwarp();
  } else {
    const uint32_t lane_off = (uint32_t)(32 * warp) << 16;
    uint32_t v[8] = {1, 2, 3, 4, 5, 6, 7, 8};
    float4 acc = make_float4(0, 0, 0, 0);
    int i = 0;
    while (!stop) {
      if (mode & 1) {
        tc::tmem_st8(base + lane_off + 384 + (i % 16) * 8, v);
        tc::tmem_st_wait();
      }
      if (mode & 2) {
#pragma unroll
        for (int u = 0; u < 8; ++u) sX[(i * 8 + u) % 4096 * 0 + ((tid + 128 * u) % 4096)] = make_float4(i, u, 0, 0);
      }
      if (mode & 4) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const float4 x = sX[(tid + 128 * u + i) % 4096];
          acc.x += x.x;
        }
      }
      ++i;
    }
    if (acc.x == 1234.5f) out[1] = 1;
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(base, 512);
}

int main() {
  long long* d; cudaMalloc(&d, 64); long long h[2];
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 98304);
  struct Cfg { int N, lbo, sbo; } cfgs[] = {{192, 128, 256}, {256, 128, 256}, {192, 3072, 128}, {256, 4096, 128}};
  for (auto c : cfgs)
    for (int mode : {0, 7, 8, 16, 24, 31}) {
      k<<<1, 160, 98304>>>(3000, c.N, c.lbo, c.sbo, mode, d);
      cudaError_t e = cudaDeviceSynchronize();
      cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost);
      printf("N=%d lbo=%d sbo=%d mode=%d: %.1f cycles/MMA (ideal %.0f) %s\n", c.N, c.lbo, c.sbo, mode, h[0] / 3000.0,
             c.N / 2.0, cudaGetErrorString(e));
    }
  return 0;
}
