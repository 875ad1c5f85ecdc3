// KG — the lane-general, dtype-general plan and multiply: any valid
// LaneConfig {W, P, V} (group width G = W*V in {1, 2, 4, ..., 64}, P in [1, 16], region
// width R = G*P; matrix.hpp:31-44, kernel_table.cpp:64-92) and both reference dtypes
// (f32, f64; matrix.hpp:13-26).  The f32 default lane {8, 8, 1} keeps the fused K1/K2
// kernels; every other (dtype, lane) runs these:
//
//   kg_abits<T>    A bitmap (uint32 [M][ceil(K/32)], LSB-first, as K1) + per-row / per-32-row
//                  non-zero counts, one ballot per (row, 32 columns); the CSR then reuses
//                  K1's k1_csr over the same bitmap.
//   kg_codes<T>    B pattern codes, uint16 [K][ldb/R]: bit (P-1-j) <-> group j of the region
//                  has a non-zero (MSB first over all P bits: kernel_table.cpp:19 for the high
//                  8 groups, :86-88 chains the low P-8 groups the same way).
//   kg_bcounts     per B row: Σ popcount(code), # codes != 0 (the WorkCounters factors).
//   kg_mul<T, D>   C += A*B on 64 x 64 C tiles: per C element the ascending-k fma chain of
//                  exactly the terms the reference kernel table forms — a_ik != 0 and the
//                  code bit of (k, group of j) set (kernel_table.cpp:12-28: a set group FMAs
//                  all G of its elements, zero b included; an unset group is untouched) — so
//                  C is bit-identical to the reference for every dtype and lane.  D = dense:
//                  multiply_simple (every term).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "k1_preprocess.cuh"

namespace mmmcu {

// one warp per (row, 32-column word): lane l tests column 32w + l
template <typename T>
__global__ void __launch_bounds__(256) kg_abits(const T* __restrict__ A, int64_t M, int64_t K, int64_t lda,
                                                uint32_t* __restrict__ abits, int64_t kw, uint32_t* __restrict__ arow,
                                                uint32_t* __restrict__ tile_sum) {
  const int lane = threadIdx.x & 31;
  const int64_t w = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5), i = blockIdx.y;
  if (w >= kw) return;
  const int64_t col = 32 * w + lane;
  const bool nz = col < K && A[i * lda + col] != T(0);
  const uint32_t m = __ballot_sync(0xffffffffu, nz);
  if (lane == 0) {
    abits[i * kw + w] = m;
    if (m) {
      atomicAdd(&arow[i], (uint32_t)__popc(m));
      atomicAdd(&tile_sum[i / kK1Rows], (uint32_t)__popc(m));
    }
  }
}

// exclusive prefix of the 32-row tile counts (the CSR's row_ptr base), one CTA
__global__ void __launch_bounds__(256) kg_tile_prefix(const uint32_t* __restrict__ tile_sum, int64_t n,
                                                      int64_t* __restrict__ out) {
  k1_block_exclusive_scan(tile_sum, n, 0, out);
}

// thread per (k, region)
template <typename T>
__global__ void kg_codes(const T* __restrict__ B, int64_t K, int64_t ldb, int64_t nreg, int G, int P,
                         uint16_t* __restrict__ codes) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= K * nreg) return;
  const int64_t k = t / nreg, r = t % nreg;
  const T* reg = B + k * ldb + r * (int64_t)G * P;
  uint32_t code = 0;
  for (int j = 0; j < P; ++j) {
    bool nz = false;
    for (int l = 0; l < G; ++l) nz |= reg[j * G + l] != T(0);
    code = (code << 1) | (nz ? 1u : 0u);
  }
  codes[t] = (uint16_t)code;
}

// thread per B row: Σ popcount(code), # non-zero codes
__global__ void kg_bcounts(const uint16_t* __restrict__ codes, int64_t K, int64_t nreg, uint32_t* __restrict__ bpop,
                           uint32_t* __restrict__ bnz) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= K) return;
  uint32_t pop = 0, nz = 0;
  for (int64_t r = 0; r < nreg; ++r) {
    const uint32_t c = codes[k * nreg + r];
    pop += __popc(c);
    nz += c != 0u;
  }
  bpop[k] = pop;
  bnz[k] = nz;
}

// Exact WorkCounters from the per-column A counts and per-row B factors:
// out = {inv, lanes (Σ acol·G·bpop), skipped, zero regions, nnzA}; one CTA of 1024 threads.
__global__ void __launch_bounds__(1024) kg_counters(const uint32_t* __restrict__ acol, const uint32_t* __restrict__ bpop,
                                                    const uint32_t* __restrict__ bnz, int64_t K, int64_t M, int64_t nreg,
                                                    int G, unsigned long long* __restrict__ out) {
  unsigned long long s[4] = {0, 0, 0, 0};
  for (int64_t k = threadIdx.x; k < K; k += blockDim.x) {
    const unsigned long long a = acol[k], p = bpop[k], n = bnz[k];
    s[0] += a * n;
    s[1] += a * (unsigned long long)G * p;
    s[2] += a * ((unsigned long long)nreg - n);
    s[3] += a;
  }
  __shared__ unsigned long long red[32][4];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    unsigned long long v = s[q];
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) red[warp][q] = v;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long v[4] = {0, 0, 0, 0};
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w)
      for (int q = 0; q < 4; ++q) v[q] += red[w][q];
    out[0] = v[0];
    out[1] = v[1];
    out[2] = (unsigned long long)(M * K) - v[3];
    out[3] = v[2];
    out[4] = v[3];
  }
}

// plan totals over the codes: out[5] = Σ popcount, out[6] = # zero codes (plan_stats)
__global__ void __launch_bounds__(1024) kg_plan_totals(const uint32_t* __restrict__ bpop, const uint32_t* __restrict__ bnz,
                                                       int64_t K, int64_t nreg, unsigned long long* __restrict__ out) {
  unsigned long long p = 0, z = 0;
  for (int64_t k = threadIdx.x; k < K; k += blockDim.x) {
    p += bpop[k];
    z += (unsigned long long)nreg - bnz[k];
  }
  __shared__ unsigned long long red[32][2];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    p += __shfl_xor_sync(0xffffffffu, p, o);
    z += __shfl_xor_sync(0xffffffffu, z, o);
  }
  if (lane == 0) {
    red[warp][0] = p;
    red[warp][1] = z;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long a = 0, b = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
      a += red[w][0];
      b += red[w][1];
    }
    out[5] = a;
    out[6] = b;
  }
}

// C (M x ncols, ldc) += A * B over 64 x 64 C tiles, 256 threads of 4 x 4 elements, k in
// chunks of 16 staged in shared memory together with the chunk's 64-column code-bit masks.
// DENSE: every term (multiply_simple).  ncols: B's padded width for the masked multiply (the
// reference's regions cover the padding), N for multiply_simple.
constexpr int kKgTile = 64, kKgChunk = 16;
template <typename T, bool DENSE>
__global__ void __launch_bounds__(256) kg_mul(const T* __restrict__ A, int64_t lda, const T* __restrict__ B,
                                              int64_t ldb, T* __restrict__ C, int64_t ldc, int64_t M, int64_t K,
                                              int64_t ncols, const uint16_t* __restrict__ codes, int64_t nreg, int G,
                                              int P) {
  __shared__ T sa[kKgChunk][kKgTile];  // A^T chunk: sa[kk][row]
  __shared__ T sb[kKgChunk][kKgTile];
  __shared__ uint32_t sm[kKgChunk][2];  // code bit of (k, column) for the tile's 64 columns
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const int64_t m0 = (int64_t)blockIdx.y * kKgTile, n0 = (int64_t)blockIdx.x * kKgTile;
  T acc[4][4];
#pragma unroll
  for (int r = 0; r < 4; ++r)
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int64_t i = m0 + 4 * ty + r, j = n0 + 4 * tx + c;
      acc[r][c] = (i < M && j < ncols) ? C[i * ldc + j] : T(0);
    }
  const int R = G * P;
  for (int64_t k0 = 0; k0 < K; k0 += kKgChunk) {
    for (int e = tid; e < kKgChunk * kKgTile; e += 256) {
      const int kk = e % kKgChunk, row = e / kKgChunk;  // A: consecutive threads walk k (coalesced rows)
      const int64_t i = m0 + row, k = k0 + kk;
      sa[kk][row] = (i < M && k < K) ? A[i * lda + k] : T(0);
      const int kb = e / kKgTile, col = e % kKgTile;
      const int64_t kq = k0 + kb, j = n0 + col;
      sb[kb][col] = (kq < K && j < ncols) ? B[kq * ldb + j] : T(0);
    }
    if (!DENSE) {
      // warp w: masks of k rows w and w + 8, 32 columns per ballot
      const int lane = tid & 31, w = tid >> 5;
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        const int kk = w + 8 * (h >> 1), half = h & 1;
        const int64_t k = k0 + kk, j = n0 + 32 * half + lane;
        bool bit = false;
        if (k < K && j < ncols) {
          const int64_t r = j / R, jg = (j % R) / G;
          bit = (codes[k * nreg + r] >> (P - 1 - jg)) & 1u;
        }
        const uint32_t m = __ballot_sync(0xffffffffu, bit);
        if (lane == 0) sm[kk][half] = m;
      }
    }
    __syncthreads();
    const int kn = (int)(K - k0 < kKgChunk ? K - k0 : kKgChunk);
    for (int kk = 0; kk < kn; ++kk) {
      T a[4], b[4];
#pragma unroll
      for (int r = 0; r < 4; ++r) a[r] = sa[kk][4 * ty + r];
#pragma unroll
      for (int c = 0; c < 4; ++c) b[c] = sb[kk][4 * tx + c];
      const uint32_t mb = DENSE ? 0xFu : (sm[kk][tx >> 3] >> (4 * (tx & 7))) & 0xFu;
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int c = 0; c < 4; ++c)
          if (DENSE || (a[r] != T(0) && ((mb >> c) & 1u))) acc[r][c] = fma(a[r], b[c], acc[r][c]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int r = 0; r < 4; ++r)
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int64_t i = m0 + 4 * ty + r, j = n0 + 4 * tx + c;
      if (i < M && j < ncols) C[i * ldc + j] = acc[r][c];
    }
}

}  // namespace mmmcu
