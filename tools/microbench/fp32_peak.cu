// FP32 SIMT peak + shared-memory bandwidth microbenchmarks for the roofline
// denominators that MEASURED_PEAKS.json does not carry (SURVEY.md §7 hard part 7).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
  unsigned long long ra = *reinterpret_cast<unsigned long long*>(&a);
  unsigned long long rb = *reinterpret_cast<unsigned long long*>(&b);
  unsigned long long rc = *reinterpret_cast<unsigned long long*>(&c);
  unsigned long long rd;
  asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(rd) : "l"(ra), "l"(rb), "l"(rc));
  return *reinterpret_cast<float2*>(&rd);
}

template <int NCH>
__global__ void k_ffma2(float* out, int iters, float s) {
  float2 acc[NCH];
#pragma unroll
  for (int i = 0; i < NCH; ++i) acc[i] = make_float2(threadIdx.x * 1e-3f + i, i * 0.5f);
  float2 a = make_float2(s, s * 0.999f), b = make_float2(0.9999f, 1.0001f);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NCH; ++i) acc[i] = ffma2(acc[i], a, b);
  }
  float r = 0.f;
#pragma unroll
  for (int i = 0; i < NCH; ++i) r += acc[i].x + acc[i].y;
  if (r == 1234.5f) out[threadIdx.x] = r;
}

template <int NCH>
__global__ void k_ffma(float* out, int iters, float s) {
  float acc[NCH];
#pragma unroll
  for (int i = 0; i < NCH; ++i) acc[i] = threadIdx.x * 1e-3f + i;
  float a = s, b = 0.9999f;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NCH; ++i) acc[i] = fmaf(acc[i], a, b);
  }
  float r = 0.f;
#pragma unroll
  for (int i = 0; i < NCH; ++i) r += acc[i];
  if (r == 1234.5f) out[threadIdx.x] = r;
}

// smem: mode 0 = every lane a distinct conflict-free 16B chunk; 1 = broadcast (all lanes same
// address); 2 = random row per lane (row stride 1 KB), fixed column chunk rotated per lane
__global__ void k_lds(float* out, int iters, int mode, const uint32_t* rnd) {
  __shared__ float4 sm[2048];  // 32 KB: 16 rows x 128 chunks
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) sm[i] = make_float4(i, i + 1, i + 2, i + 3);
  __syncthreads();
  float4 acc = make_float4(0, 0, 0, 0);
  uint32_t lane = threadIdx.x & 31;
  uint32_t r = rnd[(blockIdx.x * blockDim.x + threadIdx.x) & 4095];
  for (int it = 0; it < iters; ++it) {
    uint32_t idx;
    if (mode == 0) idx = (threadIdx.x + it * 32) & 2047;
    else if (mode == 1) idx = (it * 8) & 2047;
    else if (mode == 2) { r = r * 1664525u + 1013904223u; idx = (((r >> 10) & 15) * 128 + ((lane + it * 8) & 127)) & 2047; }
    else { r = r * 1664525u + 1013904223u; idx = (r >> 12) & 2047; }
    float4 v = sm[idx];
    acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
  }
  if (acc.x + acc.y + acc.z + acc.w == 1234.5f) out[threadIdx.x] = acc.x;
}

int main() {
  float* out; CK(cudaMalloc(&out, 4096 * 4));
  uint32_t* rnd; CK(cudaMalloc(&rnd, 4096 * 4));
  uint32_t h[4096]; for (int i = 0; i < 4096; ++i) h[i] = i * 2654435761u;
  CK(cudaMemcpy(rnd, h, sizeof h, cudaMemcpyHostToDevice));
  int sms; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 20000;
  for (int rep = 0; rep < 2; ++rep) {
    for (int bpsm : {2, 4, 8}) {
      int blocks = sms * bpsm, threads = 256;
      k_ffma2<8><<<blocks, threads>>>(out, 100, 1.0001f);
      cudaEventRecord(e0);
      k_ffma2<8><<<blocks, threads>>>(out, iters, 1.0001f);
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double flops = 2.0 * 2 * 8 * (double)iters * blocks * threads;
      printf("ffma2 blocks/SM=%d: %.2f TFLOP/s (%.3f ms)\n", bpsm, flops / ms / 1e9, ms);
      k_ffma<16><<<blocks, threads>>>(out, 100, 1.0001f);
      cudaEventRecord(e0);
      k_ffma<16><<<blocks, threads>>>(out, iters, 1.0001f);
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      cudaEventElapsedTime(&ms, e0, e1);
      flops = 2.0 * 16 * (double)iters * blocks * threads;
      printf("ffma  blocks/SM=%d: %.2f TFLOP/s (%.3f ms)\n", bpsm, flops / ms / 1e9, ms);
    }
  }
  cudaFuncSetAttribute(k_lds, cudaFuncAttributeMaxDynamicSharedMemorySize, 0);
  for (int mode = 0; mode < 4; ++mode) {
    int blocks = sms, threads = 1024;
    k_lds<<<blocks, threads>>>(out, 100, mode, rnd);
    cudaEventRecord(e0);
    k_lds<<<blocks, threads>>>(out, iters, mode, rnd);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double lds = (double)iters * blocks * threads / 32;  // warp-level LDS.128 instructions
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    printf("lds128 mode=%d: %.3f ms, %.2f warp-LDS128/ns/SM, %.1f B/clk/SM at %d MHz (logical bytes)\n",
           mode, ms, lds / ms / 1e6 / sms, lds * 512 / (ms * 1e-3) / sms / (clk * 1e3), clk / 1000);
  }
  CK(cudaGetLastError());
  return 0;
}
