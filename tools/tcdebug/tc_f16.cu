// kind::f16 probe (A fp16 in TMEM, B fp16 K-major in smem): checks the TMEM A-operand packing
// (two k per 32-bit column) and the smem descriptor for 16-bit K-major B, then times back-to-back
// MMAs (f16 M128 N192 K16 vs tf32 M128 N192 K8) for the fp16-split K2-TC design.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cmath>
#include <cuda_fp16.h>
#include "../../paper_2402_14118_b200/csrc/tc_ptx.cuh"
using namespace mmmcu;

__host__ __device__ constexpr uint32_t idesc_f16_m128(uint32_t n) {
  return (1u << 4) | (0u << 7) | (0u << 10) | ((n >> 3) << 17) | ((128u >> 4) << 24);
}
__device__ __forceinline__ void mma_f16_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
      "r"(a), "l"(b), "r"(idesc), "r"(acc) : "memory");
}

// variant 0: TMEM col c = k 2c (low half) | k 2c+1 (high half); variant 1: swapped halves
__global__ void k_probe(const float* A, const float* B, float* D, int variant, int N) {
  __shared__ __align__(1024) uint8_t sB[16 * 256 * 2];
  __shared__ uint64_t bar;
  __shared__ uint32_t tb;
  const int tid = threadIdx.x, warp = tid >> 5;
  if (warp == 0) tc::tmem_alloc(&tb, 512);
  if (tid == 0) { tc::mbar_init(&bar, 1); tc::fence_mbar_init(); }
  const int lbo = (N / 8) * 128;
  for (int e = tid; e < 16 * N; e += blockDim.x) {
    const int k = e / N, n = e % N;
    const int off = (n % 8) * 16 + (n / 8) * 128 + (k / 8) * lbo + (k % 8) * 2;
    *reinterpret_cast<__half*>(sB + off) = __float2half_rn(B[k * N + n]);
  }
  tc::fence_async_smem();
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t base = tb;
  const uint32_t lane_base = (uint32_t)(32 * warp) << 16;
  uint32_t a[8];
  for (int c = 0; c < 8; ++c) {
    const uint32_t lo = __half_as_ushort(__float2half_rn(A[tid * 16 + 2 * c]));
    const uint32_t hi = __half_as_ushort(__float2half_rn(A[tid * 16 + 2 * c + 1]));
    a[c] = variant == 0 ? (lo | (hi << 16)) : (hi | (lo << 16));
  }
  tc::tmem_st8(base + lane_base + 256, a);
  tc::tmem_st_wait();
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) {
    tc::fence_after_sync();
    if (tc::elect_one()) {
      const uint64_t desc = tc::smem_desc(tc::smem_u32(sB), lbo, 128);
      mma_f16_ts(base, base + 256, desc, idesc_f16_m128(N), 0);
      tc::mma_commit(&bar);
    }
    __syncwarp();
  }
  tc::mbar_wait(&bar, 0);
  tc::fence_after_sync();
  for (int c0 = 0; c0 < N; c0 += 16) {
    uint32_t v[16];
    tc::tmem_ld16(base + lane_base + c0, v);
    tc::tmem_ld_wait();
    for (int n = 0; n < 16; ++n) D[tid * N + c0 + n] = __uint_as_float(v[n]);
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(base, 512);
}

// rate: one CTA per SM, one elected thread issues `iters` x 3 MMAs (N=192) back to back
__global__ void k_rate(int kind, int iters, unsigned long long* out) {
  __shared__ __align__(1024) uint8_t sB[192 * 16 * 2 * 2];
  __shared__ uint64_t bar;
  __shared__ uint32_t tb;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int e = tid; e < (int)sizeof(sB) / 4; e += blockDim.x) reinterpret_cast<uint32_t*>(sB)[e] = 0x3c003c00u;
  if (warp == 0) tc::tmem_alloc(&tb, 512);
  if (tid == 0) { tc::mbar_init(&bar, 1); tc::fence_mbar_init(); }
  tc::fence_async_smem();
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t base = tb;
  if (warp == 0) {
    const long long t0 = clock64();
    if (tc::elect_one()) {
      const uint64_t desc = tc::smem_desc(tc::smem_u32(sB), 24 * 128, 128);
      for (int i = 0; i < iters; ++i) {
        for (int u = 0; u < 3; ++u) {
          if (kind == 0) mma_f16_ts(base, base + 384 + 8 * u, desc, idesc_f16_m128(192), i + u > 0);
          else tc::mma_tf32_ts(base, base + 384 + 8 * u, desc, tc::idesc_tf32_m128(192), i + u > 0);
        }
      }
      tc::mma_commit(&bar);
    }
    __syncwarp();
    tc::mbar_wait(&bar, 0);
    const long long t1 = clock64();
    if (tid == 0) out[blockIdx.x] = (unsigned long long)(t1 - t0);
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(base, 512);
}

int main() {
  for (int N : {16, 192}) {
    float *hA = new float[128 * 16], *hB = new float[16 * N], *hD = new float[128 * N], *ref = new float[128 * N];
    srand(1);
    for (int i = 0; i < 128 * 16; ++i) hA[i] = (float)(rand() % 7 - 3);
    for (int i = 0; i < 16 * N; ++i) hB[i] = (float)(rand() % 5 - 2);
    for (int m = 0; m < 128; ++m)
      for (int n = 0; n < N; ++n) {
        float s = 0;
        for (int k = 0; k < 16; ++k) s += hA[m * 16 + k] * hB[k * N + n];
        ref[m * N + n] = s;
      }
    float *dA, *dB, *dD;
    cudaMalloc(&dA, 128 * 16 * 4); cudaMalloc(&dB, 16 * N * 4); cudaMalloc(&dD, 128 * N * 4);
    cudaMemcpy(dA, hA, 128 * 16 * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, hB, 16 * N * 4, cudaMemcpyHostToDevice);
    for (int variant = 0; variant < 2; ++variant) {
      cudaMemset(dD, 0, 128 * N * 4);
      k_probe<<<1, 128>>>(dA, dB, dD, variant, N);
      cudaError_t e = cudaDeviceSynchronize();
      cudaMemcpy(hD, dD, 128 * N * 4, cudaMemcpyDeviceToHost);
      double err = 0; int bad = 0;
      for (int i = 0; i < 128 * N; ++i) { double d = fabs(hD[i] - ref[i]); if (d > 1e-3) ++bad; if (d > err) err = d; }
      printf("N=%d variant %d: %s maxerr=%g bad=%d  D[0][0..3]=%g %g %g %g ref=%g %g %g %g\n", N, variant,
             cudaGetErrorString(e), err, bad, hD[0], hD[1], hD[2], hD[3], ref[0], ref[1], ref[2], ref[3]);
      fflush(stdout);
      if (e != cudaSuccess) return 1;
    }
  }
  unsigned long long* dout;
  cudaMalloc(&dout, 148 * 8);
  unsigned long long h[148];
  for (int kind = 0; kind < 2; ++kind) {
    const int iters = 2000;
    k_rate<<<148, 128>>>(kind, iters, dout);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, dout, sizeof h, cudaMemcpyDeviceToHost);
    double s = 0;
    for (int i = 0; i < 148; ++i) s += h[i];
    printf("%s N=192: %s  %.1f cycles per MMA (148 CTAs)\n", kind == 0 ? "f16 K=16" : "tf32 K=8", cudaGetErrorString(e),
           s / 148 / (3.0 * iters));
  }
  return 0;
}
