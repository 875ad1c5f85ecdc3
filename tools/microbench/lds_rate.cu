// Shared-memory load instruction throughput per SM on B200 (sm_100a): how many warp-level
// LDS.{32,64,128} per clock for conflict-free, broadcast and random patterns.  Sizes the
// SIMT masked-GEMM inner loops.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

template <typename T, int MODE>
__global__ void k(float* out, int iters, uint32_t seed) {
  __shared__ float4 sm[2048];  // 32 KB
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) sm[i] = make_float4(i, i + 1, i + 2, i + 3);
  __syncthreads();
  const T* s = reinterpret_cast<const T*>(sm);
  const uint32_t n = 32768 / sizeof(T);
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t r = seed ^ (threadIdx.x * 2654435761u);
  T acc[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) acc[u] = s[u];
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      uint32_t idx;
      if (MODE == 0) idx = (warp * 256 + u * 32 + lane + it * 8) & (n - 1);          // conflict-free
      else if (MODE == 1) idx = (warp * 64 + u * 8 + it) & (n - 1);                  // broadcast
      else { r = r * 1664525u + 1013904223u; idx = (r >> 8) & (n - 1); }           // random
      T v = s[idx];
      if constexpr (sizeof(T) == 4) acc[u] += v;
      else if constexpr (sizeof(T) == 8) { acc[u].x += v.x; acc[u].y += v.y; }
      else { acc[u].x += v.x; acc[u].y += v.y; acc[u].z += v.z; acc[u].w += v.w; }
    }
  }
  float t = 0;
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    if constexpr (sizeof(T) == 4) t += acc[u];
    else t += acc[u].x;
  }
  if (t == 1234.5f) out[threadIdx.x] = t;
}

template <typename T, int MODE>
int run(const char* name, int sms) {
  float* out; CK(cudaMalloc(&out, 4096 * 4));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 4000, threads = 1024, blocks = sms * 2;
  k<T, MODE><<<blocks, threads>>>(out, 10, 1);
  cudaEventRecord(e0);
  k<T, MODE><<<blocks, threads>>>(out, iters, 1);
  cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double wl = 8.0 * iters * blocks * threads / 32;
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double per_clk = wl / (ms * 1e-3) / sms / (clk * 1e3);
  printf("%-22s %.3f ms  %.3f warp-LDS/clk/SM  %.1f B/clk/SM (logical, at max clk %d MHz)\n", name, ms,
         per_clk, per_clk * 32 * sizeof(T), clk / 1000);
  cudaFree(out);
  return 0;
}

int main() {
  int sms; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  for (int rep = 0; rep < 2; ++rep) {
    run<float, 0>("lds32 conflict-free", sms);
    run<float, 1>("lds32 broadcast", sms);
    run<float, 2>("lds32 random", sms);
    run<float2, 0>("lds64 conflict-free", sms);
    run<float2, 1>("lds64 broadcast", sms);
    run<float2, 2>("lds64 random", sms);
    run<float4, 0>("lds128 conflict-free", sms);
    run<float4, 1>("lds128 broadcast", sms);
    run<float4, 2>("lds128 random", sms);
  }
  return 0;
}
