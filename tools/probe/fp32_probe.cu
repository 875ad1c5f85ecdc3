// FP32 SIMT peak probe (measurement tool, not product): the roofline denominator that
// MEASURED_PEAKS.json lacks (SURVEY.md §7 hard part 7).  Independent FFMA chains, 8 CTAs of
// 256 threads per SM; returns TFLOP/s measured with CUDA events.  Loaded by bench.py.
#include <cuda_runtime.h>
#include <cstdint>

template <int NCH>
__global__ void __launch_bounds__(256) k_ffma(float* out, int iters, float s) {
  float acc[NCH];
#pragma unroll
  for (int i = 0; i < NCH; ++i) acc[i] = threadIdx.x * 1e-3f + i;
  const float a = s, b = 0.9999f;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NCH; ++i) acc[i] = fmaf(acc[i], a, b);
  }
  float r = 0.f;
#pragma unroll
  for (int i = 0; i < NCH; ++i) r += acc[i];
  if (r == 1234.5f) out[threadIdx.x] = r;
}

extern "C" double probe_fp32_tflops(int device, int iters) {
  if (cudaSetDevice(device) != cudaSuccess) return -1.0;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  float* out = nullptr;
  if (cudaMalloc(&out, 4096 * sizeof(float)) != cudaSuccess) return -1.0;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int blocks = sms * 8, threads = 256;
  k_ffma<16><<<blocks, threads>>>(out, 64, 1.0001f);
  double best = 0.0;
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0);
    k_ffma<16><<<blocks, threads>>>(out, iters, 1.0001f);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    const double tf = 2.0 * 16 * (double)iters * blocks * threads / (ms * 1e-3) / 1e12;
    if (tf > best) best = tf;
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(out);
  return cudaGetLastError() == cudaSuccess ? best : -1.0;
}
