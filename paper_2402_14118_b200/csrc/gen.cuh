// Device generator for the BASELINE.json synthetic inputs.
//
// Built on the reference's counter hash (rng.hpp:8-26: mix64 / hash_coords / unit_double),
// a pure function of (seed, stream, i, j), so any grid decomposition produces the same
// matrix.  Uniform values and all masks are integer hashing plus exact double arithmetic
// and match the oracle's orc_gen_iid bit for bit; the normal modes go through the device
// double log1p/cos (<= 1 ulp from glibc), rounded to fp32 once.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace mmmcu {

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

__host__ __device__ __forceinline__ uint64_t hash_coords(uint64_t seed, uint64_t a, uint64_t b, uint64_t c) {
  uint64_t h = mix64(seed ^ 0x7fb5d329728ea185ULL);
  h = mix64(h ^ a);
  h = mix64(h ^ b);
  return mix64(h ^ c);
}

__device__ __forceinline__ double unit_double(uint64_t x) { return __dmul_rn(__ull2double_rn(x >> 11), 0x1.0p-53); }

// value_kind 0 uniform[-1,1], 1 N(0, sigma), 2 ReLU(N(0,1) - thresh)
// mask_kind  0 none, 1 element zero w.p. p (stream 1), 2 aligned block zero w.p. p (stream 4)
__global__ void k_generate(float* __restrict__ out, int64_t rows, int64_t cols, int64_t ld, int64_t row0, uint64_t seed,
                           int value_kind, double sigma, double thresh, int mask_kind, double p, int64_t block) {
  const int64_t total = rows * ld;
  const double two_pi = 6.283185307179586476925286766559;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = row0 + t / ld, j = t % ld;
    float v = 0.0f;
    if (j < cols) {
      bool zero = false;
      if (mask_kind == 1) zero = unit_double(hash_coords(seed, 1, (uint64_t)i, (uint64_t)j)) < p;
      else if (mask_kind == 2) zero = unit_double(hash_coords(seed, 4, (uint64_t)i, (uint64_t)(j / block))) < p;
      if (!zero) {
        const double u1 = unit_double(hash_coords(seed, 2, (uint64_t)i, (uint64_t)j));
        if (value_kind == 0) {
          v = __double2float_rn(__dsub_rn(__dmul_rn(2.0, u1), 1.0));
        } else {
          const double u2 = unit_double(hash_coords(seed, 3, (uint64_t)i, (uint64_t)j));
          const double rad = sqrt(__dmul_rn(-2.0, log1p(-u1)));
          const double g = __dmul_rn(rad, cos(__dmul_rn(two_pi, u2)));
          if (value_kind == 1) {
            v = __double2float_rn(__dmul_rn(sigma, g));
          } else {
            const double d = __dsub_rn(g, thresh);
            v = d > 0.0 ? __double2float_rn(d) : 0.0f;
          }
        }
      }
    }
    out[t] = v;
  }
}

}  // namespace mmmcu
