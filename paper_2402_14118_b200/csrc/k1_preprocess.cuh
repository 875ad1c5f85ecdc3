// K1 — one-pass sparsity-map preprocessing on sm_100a.
//
// Replaces SPEC preprocess_b / preprocess_a (PAPER Fig. 9 and Fig. 11,
// PAPER.md:398-413, :446-458).  Everything here is HBM-bound integer work: each operand
// element is read exactly once with 16-byte coalesced loads, zero tests are exact float
// compares (`!= 0.0f`, never flushed: see SURVEY.md §7 hard part 3), and the masks are
// assembled with warp shuffles / ballots instead of per-element branches.
//
// Outputs (context-owned device memory, layouts documented in DESIGN.md):
//   abits   uint32 [M][kw]          A non-zero bitmap, bit b of word w <-> column 32w+b
//   arow    uint32 [M]              non-zeros per A row
//   acol    uint32 [K]              non-zeros per A column (for the exact WorkCounters)
//   row_ptr int64  [M+1], cols      per-row ascending index lists (CSR), ballot/popc + scan
//   codes   uint8  [K][nreg]        B pattern codes, bit 7-j <-> 8-column group j (MSB first,
//                                   kernel_table.cpp:19) == the BPlan codes
//   bgrp    uint32 [ngrp][kw]       B group k-bitmaps: bit (k%32) of word k/32 of group g set
//                                   iff B[k, 8g:8g+8] has a non-zero (transposed block masks)
//   bpop    uint32 [K]              Σ popcount(codes[k][:])   (lane ops per A non-zero / 8)
//   bnz     uint32 [K]              # codes != 0 in row k     (kernel invocations per A nz)
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace mmmcu {

constexpr int kK1Threads = 256;  // 8 warps; each thread owns 4 consecutive columns
constexpr int kK1Cols = 4 * kK1Threads;  // 1024 columns per CTA tile
constexpr int kK1Rows = 32;              // rows per CTA tile (one 32-bit k-word for B)

__device__ __forceinline__ float4 ldg_stream(const float* p) {
  float4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(p));
  return v;
}

// Exact zero test; +0 and -0 are zero, NaN and denormals are not (matrix.hpp:152, :174).
__device__ __forceinline__ uint32_t nz4(float4 v) {
  return (uint32_t)(v.x != 0.0f) | ((uint32_t)(v.y != 0.0f) << 1) | ((uint32_t)(v.z != 0.0f) << 2) |
         ((uint32_t)(v.w != 0.0f) << 3);
}

// --------------------------------------------------------------------------- A pass
// grid (ceil(K/1024), ceil(M/32)); thread t owns columns c = 1024*bx + 4t .. +3 and walks
// 32 rows.  lanes 8q..8q+7 of a warp hold the 32 columns of one bitmap word.
__global__ void __launch_bounds__(kK1Threads)
k1_a_pass(const float* __restrict__ A, int64_t M, int64_t K, int64_t lda, uint32_t* __restrict__ abits,
          int64_t kw, uint32_t* __restrict__ arow, uint32_t* __restrict__ acol) {
  const int lane = threadIdx.x & 31;
  const int64_t c = (int64_t)blockIdx.x * kK1Cols + 4 * threadIdx.x;
  const int64_t r0 = (int64_t)blockIdx.y * kK1Rows;
  const bool col_ok = c < K;
  // valid-column mask of this thread's 4 columns (K need not be a multiple of 4)
  const uint32_t vmask = col_ok ? (K - c >= 4 ? 0xFu : ((1u << (K - c)) - 1u)) : 0u;
  uint32_t ccount[4] = {0, 0, 0, 0};
  const int64_t rend = min(r0 + kK1Rows, M);
#pragma unroll 4
  for (int64_t i = r0; i < rend; ++i) {
    uint32_t nib = 0;
    if (col_ok) nib = nz4(ldg_stream(A + i * lda + c)) & vmask;
#pragma unroll
    for (int q = 0; q < 4; ++q) ccount[q] += (nib >> q) & 1u;
    uint32_t word = nib << (4 * (lane & 7));
    word |= __shfl_xor_sync(0xffffffffu, word, 1);
    word |= __shfl_xor_sync(0xffffffffu, word, 2);
    word |= __shfl_xor_sync(0xffffffffu, word, 4);
    uint32_t cnt = __popc(nib);
    cnt += __shfl_xor_sync(0xffffffffu, cnt, 1);
    cnt += __shfl_xor_sync(0xffffffffu, cnt, 2);
    cnt += __shfl_xor_sync(0xffffffffu, cnt, 4);
    cnt += __shfl_xor_sync(0xffffffffu, cnt, 8);
    cnt += __shfl_xor_sync(0xffffffffu, cnt, 16);
    if ((lane & 7) == 0 && col_ok) abits[i * kw + (c >> 5)] = word;
    if (lane == 0 && cnt) atomicAdd(&arow[i], cnt);
  }
  if (col_ok) {
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if (ccount[q]) atomicAdd(&acol[c + q], ccount[q]);
  }
}

// --------------------------------------------------------------------------- B pass
// grid (ceil(ldb/1024), ceil(K/32)); thread t owns columns c = 1024*bx + 4t .. +3 of the
// padded row (ldb is a multiple of 64, padding is zero) and walks the 32 rows of one
// k-word.  Lane pairs form 8-column groups; 16 lanes form one 64-column region (code).
__global__ void __launch_bounds__(kK1Threads)
k1_b_pass(const float* __restrict__ B, int64_t K, int64_t ldb, uint8_t* __restrict__ codes, int64_t nreg,
          uint32_t* __restrict__ bgrp, int64_t kw, uint32_t* __restrict__ bpop, uint32_t* __restrict__ bnz,
          unsigned long long* __restrict__ slice_nz) {
  const int lane = threadIdx.x & 31;
  const int64_t c = (int64_t)blockIdx.x * kK1Cols + 4 * threadIdx.x;
  const int64_t kw_idx = blockIdx.y;
  const int64_t k0 = kw_idx * 32;
  const bool col_ok = c < ldb;
  uint32_t gword = 0;  // group k-bitmap word over the 32 rows
  uint32_t slices = 0;  // (k, 16-column slice) pairs with a non-zero, counted by lane%4==0
  const int64_t kend = min(k0 + 32, K);
#pragma unroll 4
  for (int64_t k = k0; k < kend; ++k) {
    uint32_t any = 0;
    if (col_ok) any = nz4(ldg_stream(B + k * ldb + c)) != 0u;
    any |= __shfl_xor_sync(0xffffffffu, any, 1);  // 8-column group
    gword |= any << (uint32_t)(k - k0);
    const uint32_t sibling = __shfl_xor_sync(0xffffffffu, any, 2);  // other group of the slice
    if ((lane & 3) == 0 && col_ok) slices += any | sibling;
    // region code: group j = (lane & 15) >> 1 -> bit 7 - j (MSB first)
    uint32_t code = any << (7 - ((lane & 15) >> 1));
    code |= __shfl_xor_sync(0xffffffffu, code, 2);
    code |= __shfl_xor_sync(0xffffffffu, code, 4);
    code |= __shfl_xor_sync(0xffffffffu, code, 8);
    uint32_t pop = ((lane & 15) == 0 && col_ok) ? __popc(code) : 0u;
    uint32_t nzc = ((lane & 15) == 0 && col_ok) ? (uint32_t)(code != 0) : 0u;
    pop += __shfl_xor_sync(0xffffffffu, pop, 16);
    nzc += __shfl_xor_sync(0xffffffffu, nzc, 16);
    if ((lane & 15) == 0 && col_ok) codes[k * nreg + (c >> 6)] = (uint8_t)code;
    if (lane == 0) {
      if (pop) atomicAdd(&bpop[k], pop);
      if (nzc) atomicAdd(&bnz[k], nzc);
    }
  }
  if ((lane & 1) == 0 && col_ok) bgrp[(c >> 3) * kw + kw_idx] = gword;
#pragma unroll
  for (int o = 16; o; o >>= 1) slices += __shfl_xor_sync(0xffffffffu, slices, o);
  if (lane == 0 && slices) atomicAdd(slice_nz, (unsigned long long)slices);
}

// ------------------------------------------------------------------ row_ptr (scan)
// Single CTA exclusive scan of arow -> row_ptr[0..M]; M up to a few million rows.
__global__ void __launch_bounds__(1024) k1_scan_rows(const uint32_t* __restrict__ arow, int64_t M,
                                                     int64_t* __restrict__ row_ptr) {
  __shared__ int64_t warp_sums[32];
  __shared__ int64_t carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int64_t base = 0; base < M; base += 1024) {
    const int64_t i = base + threadIdx.x;
    int64_t v = i < M ? (int64_t)arow[i] : 0;
    int64_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int64_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) warp_sums[warp] = x;
    __syncthreads();
    if (warp == 0) {
      int64_t s = warp_sums[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        int64_t y = __shfl_up_sync(0xffffffffu, s, o);
        if (lane >= o) s += y;
      }
      warp_sums[lane] = s;  // inclusive over warps
    }
    __syncthreads();
    const int64_t before = carry + (warp ? warp_sums[warp - 1] : 0) + x - v;
    if (i < M) row_ptr[i] = before;
    __syncthreads();
    if (threadIdx.x == 1023) carry = before + v;
    __syncthreads();
  }
  if (threadIdx.x == 0) row_ptr[M] = carry;
}

// --------------------------------------------------------------- CSR index lists
// One warp per row: popc of each bitmap word, warp prefix sum, then each lane expands its
// word's set bits into ascending column indices.  Reads only the bitmap (no second pass
// over A).  Index type: uint16 when K <= 65536, else uint32.
template <typename Idx>
__global__ void __launch_bounds__(256) k1_csr(const uint32_t* __restrict__ abits, int64_t M, int64_t kw,
                                              const int64_t* __restrict__ row_ptr, Idx* __restrict__ cols) {
  const int lane = threadIdx.x & 31;
  const int64_t row = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (row >= M) return;
  int64_t out = row_ptr[row];
  const uint32_t* bits = abits + row * kw;
  for (int64_t w0 = 0; w0 < kw; w0 += 32) {
    const int64_t w = w0 + lane;
    uint32_t word = w < kw ? bits[w] : 0u;
    uint32_t n = __popc(word);
    uint32_t x = n;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    int64_t pos = out + x - n;
    while (word) {
      const int b = __ffs(word) - 1;
      word &= word - 1;
      cols[pos++] = (Idx)(w * 32 + b);
    }
    out += __shfl_sync(0xffffffffu, x, 31);
  }
}

// ---------------------------------------------------------------- counters + stats
// Exact WorkCounters of the coming multiply and plan_stats:
//   lane_fma_ops  = Σ_k acol[k] * 8 * bpop[k]
//   invocations   = Σ_k acol[k] * bnz[k]
//   zero regions  = Σ_k acol[k] * (nreg - bnz[k])
//   rows_skipped  = M*K - Σ_k acol[k]
//   stats         = Σ_k bpop[k], Σ_k (nreg - bnz[k])
// out: u64[8] = {inv, lanes, skipped, zreg, nnzA, pop_total, zero_codes, span}
//   span: K2-SIMT mask granularity, from the cost model of DESIGN.md (K2 variants):
//   16-column slices cost ~41 issue slots per non-zero (k, slice), 8-column groups ~23 per
//   non-zero (k, group); pick the cheaper (slice_nz[0] = # non-zero (k, slice) pairs).
__global__ void __launch_bounds__(1024) k1_finalize(const uint32_t* __restrict__ acol, const uint32_t* __restrict__ bpop,
                                                    const uint32_t* __restrict__ bnz, int64_t K, int64_t M,
                                                    int64_t nreg, int has_a, int has_b,
                                                    const unsigned long long* __restrict__ slice_nz,
                                                    unsigned long long* __restrict__ out) {
  unsigned long long s[6] = {0, 0, 0, 0, 0, 0};
  for (int64_t k = threadIdx.x; k < K; k += blockDim.x) {
    const unsigned long long a = has_a ? acol[k] : 0ull;
    const unsigned long long p = has_b ? bpop[k] : 0ull;
    const unsigned long long z = has_b ? (unsigned long long)(nreg - (int64_t)bnz[k]) : 0ull;
    const unsigned long long n = has_b ? bnz[k] : 0ull;
    s[0] += a * n;
    s[1] += a * 8ull * p;
    s[2] += a * z;
    s[3] += a;
    s[4] += p;
    s[5] += z;
  }
  __shared__ unsigned long long red[32][6];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int q = 0; q < 6; ++q) {
    unsigned long long v = s[q];
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) red[warp][q] = v;
  }
  __syncthreads();
  if (threadIdx.x < 6) {
    unsigned long long v = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) v += red[w][threadIdx.x];
    red[0][threadIdx.x] = v;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    out[0] = red[0][0];
    out[1] = red[0][1];
    out[2] = (unsigned long long)(M * K) - red[0][3];
    out[3] = red[0][2];
    out[4] = red[0][3];
    out[5] = red[0][4];
    out[6] = red[0][5];
    out[7] = (has_b && 41ull * slice_nz[0] > 23ull * red[0][4]) ? 8ull : 16ull;
  }
}

// ------------------------------------------------------------ ABlockIndex export
// SPEC ABlockIndex from the bitmap (export path, not the hot path): segment s of the
// block-major enumeration -> count = popc(byte), offsets = set-bit positions.
__global__ void k1_ablock_export(const uint32_t* __restrict__ abits, int64_t M, int64_t K, int64_t kw,
                                 int64_t block_dim, int64_t n_bc, uint8_t* __restrict__ counts,
                                 uint8_t* __restrict__ offsets) {
  // one thread per (row, 8-segment); segment index computed block-major
  const int64_t nseg_row = (K + 7) / 8;
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= M * nseg_row) return;
  const int64_t i = t / nseg_row, sg = t % nseg_row;
  const int64_t k0 = sg * 8;
  const int64_t bi = i / block_dim, bk = k0 / block_dim;
  const int64_t rows_in_br = min(block_dim, M - bi * block_dim);
  const int64_t segs_full_block = block_dim / 8;
  // segments before block (bi, bk): all earlier block rows, then earlier blocks in this row
  const int64_t before_br = bi * block_dim * nseg_row;
  const int64_t before_bc = rows_in_br * bk * segs_full_block;
  const int64_t width_bk = min(block_dim, K - bk * block_dim);
  const int64_t segs_this_block = (width_bk + 7) / 8;
  const int64_t s = before_br + before_bc + (i - bi * block_dim) * segs_this_block + (k0 - bk * block_dim) / 8;
  const uint32_t byte = (abits[i * kw + (k0 >> 5)] >> (k0 & 31)) & 0xFFu;
  const uint32_t cnt = __popc(byte);
  counts[s] = (uint8_t)cnt;
  uint8_t off[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) off[q] = 0xFF;
  if (cnt != 8) {
    uint32_t b = byte;
    int n = 0;
    while (b) {
      const int p = __ffs(b) - 1;
      b &= b - 1;
      off[n++] = (uint8_t)p;
    }
  }
#pragma unroll
  for (int q = 0; q < 8; ++q) offsets[8 * s + q] = off[q];
  (void)n_bc;
}

}  // namespace mmmcu
