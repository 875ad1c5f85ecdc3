// Single-MMA layout probe for tcgen05.mma kind::tf32 (A in TMEM, B in smem): checks the
// TMEM A-operand and smem-descriptor conventions used by K2-TC against a host product.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cmath>
#include "../../paper_2402_14118_b200/csrc/tc_ptx.cuh"
using namespace mmmcu;

// variant 0: B MN-major, element (k,n) at (n/4)*SBO + (k%8)*16 + (n%4)*4, SBO=128, LBO=512
// variant 1: B K-major,  element (n,k) at (n%8)*16 + (n/8)*SBO + (k/4)*LBO + (k%4)*4, SBO=128, LBO=256
// variant 2: B MN-major with LBO/SBO swapped in the descriptor
// variant 3: B K-major with LBO/SBO swapped in the descriptor
__global__ void k_probe(const float* A, const float* B, float* D, int variant, int N) {
  __shared__ __align__(1024) uint8_t sB[4096];
  __shared__ uint64_t bar;
  __shared__ uint32_t tb;
  const int tid = threadIdx.x, warp = tid >> 5;
  if (warp == 0) tc::tmem_alloc(&tb, 64);
  if (tid == 0) { tc::mbar_init(&bar, 1); tc::fence_mbar_init(); }
  // B into smem
  for (int e = tid; e < 8 * N; e += blockDim.x) {
    const int k = e / N, n = e % N;
    int off;
    if (variant == 0 || variant == 2) off = (n / 4) * 128 + (k % 8) * 16 + (n % 4) * 4;
    else off = (n % 8) * 16 + (n / 8) * 128 + (k / 4) * (N / 8) * 128 + (k % 4) * 4;
    *reinterpret_cast<float*>(sB + off) = B[k * N + n];
  }
  tc::fence_async_smem();
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t base = tb;
  const uint32_t lane_base = (uint32_t)(32 * warp) << 16;
  // A (row = tid) into TMEM columns 32..39; D at columns 0..N-1 zeroed
  uint32_t a[8], z[8] = {0,0,0,0,0,0,0,0};
  for (int k = 0; k < 8; ++k) a[k] = __float_as_uint(A[tid * 8 + k]);
  tc::tmem_st8(base + lane_base + 32, a);
  for (int c = 0; c < N; c += 8) tc::tmem_st8(base + lane_base + c, z);
  tc::tmem_st_wait();
  tc::fence_before_sync();
  __syncthreads();
  if (tid == 0) {
    tc::fence_after_sync();
    uint64_t desc;
    const uint32_t sa = tc::smem_u32(sB);
    if (variant == 0) desc = tc::smem_desc(sa, 512, 128);
    else if (variant == 1) desc = tc::smem_desc(sa, (N / 8) * 128, 128);
    else if (variant == 2) desc = tc::smem_desc(sa, 128, 512);
    else desc = tc::smem_desc(sa, 128, (N / 8) * 128);
    uint32_t idesc = tc::idesc_tf32_m128(N);
    if (variant == 1 || variant == 3) idesc &= ~(1u << 16);  // B K-major
    tc::mma_tf32_ts(base, base + 32, desc, idesc, 1);
    tc::mma_commit(&bar);
  }
  tc::mbar_wait(&bar, 0);
  tc::fence_after_sync();
  uint32_t v[16];
  tc::tmem_ld16(base + lane_base, v);
  tc::tmem_ld_wait();
  for (int n = 0; n < N && n < 16; ++n) D[tid * N + n] = __uint_as_float(v[n]);
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(base, 64);
}

int main() {
  const int N = 16;
  float hA[128 * 8], hB[8 * N], hD[128 * N], ref[128 * N];
  srand(1);
  for (int i = 0; i < 128 * 8; ++i) hA[i] = (float)(rand() % 7 - 3);
  for (int i = 0; i < 8 * N; ++i) hB[i] = (float)(rand() % 5 - 2);
  for (int m = 0; m < 128; ++m)
    for (int n = 0; n < N; ++n) {
      float s = 0;
      for (int k = 0; k < 8; ++k) s += hA[m * 8 + k] * hB[k * N + n];
      ref[m * N + n] = s;
    }
  float *dA, *dB, *dD;
  cudaMalloc(&dA, sizeof hA); cudaMalloc(&dB, sizeof hB); cudaMalloc(&dD, sizeof hD);
  cudaMemcpy(dA, hA, sizeof hA, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB, sizeof hB, cudaMemcpyHostToDevice);
  for (int variant = 0; variant < 4; ++variant) {
    cudaMemset(dD, 0, sizeof hD);
    k_probe<<<1, 128>>>(dA, dB, dD, variant, N);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(hD, dD, sizeof hD, cudaMemcpyDeviceToHost);
    double err = 0; int bad = 0;
    for (int i = 0; i < 128 * N; ++i) { double d = fabs(hD[i] - ref[i]); if (d > 1e-3) ++bad; if (d > err) err = d; }
    printf("variant %d: %s maxerr=%g bad=%d  D[0][0..3]=%g %g %g %g ref=%g %g %g %g\n", variant, cudaGetErrorString(e),
           err, bad, hD[0], hD[1], hD[2], hD[3], ref[0], ref[1], ref[2], ref[3]);
    if (e != cudaSuccess) return 1;
  }
  return 0;
}
