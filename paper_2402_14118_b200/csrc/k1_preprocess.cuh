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
constexpr int kTcTileN = 192;            // K2-TC C tile width (columns)

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

// Zero-initialised per-plan scratch (one cudaMemsetAsync per preprocess):
//   za = arow[M] | acol[K] | tile_sum[M/32];  zb = slice_nz (u64) | bpop[K] | bnz[K]
struct K1Scratch {
  uint32_t* arow;
  uint32_t* acol;
  uint32_t* tile_sum;     // [ceil(M/32)] non-zeros per 32-row tile (zeroed)
  int64_t* tile_prefix;   // [ceil(M/32) + 1] exclusive prefix of tile_sum (written by the last CTA)
  uint32_t* bpop;
  uint32_t* bnz;
  unsigned long long* slice_nz;
  unsigned int* done;
  // K2-TC operands (nullptr when the TC path is not prepared)
  float* at;              // A^T per 128-row tile: at[(rt * kpad + k) * 128 + (i % 128)], zero padded
  int64_t kpad;           // K rounded up to 32
  int64_t m_at;           // M rounded up to 128
  uint32_t* tlive;        // [n_tc][kw] live-k mask per kTcTileN-column TC tile: bit kk of word c
                          // set iff B[32c + kk, tile columns] has a non-zero (zeroed, atomicOr)
  int64_t n_tb;           // 256-column tiles of B (K2-SIMT records)
  int64_t n_tc;           // kTcTileN-column tiles of B (K2-TC)
  int choose;             // AUTO: pick K2-SIMT vs K2-TC from the cost model (both operand sets built)
  // K2-SIMT operand: raw non-zero B block rows per (256-column tile, chunk)
  uint32_t* row_cnt;      // [n_tb][kw] non-zero (k, 16-column slice) rows (zeroed)
  int64_t* row_off;       // [n_tb * kw + 1] exclusive prefix of (row_cnt + 3 header rows), 64-byte units
};

// --------------------------------------------------------------------------- A tile
// Tile (tx, ty): columns 1024*tx + 4t .. +3 for thread t, rows 32*ty .. +31.  Lanes
// 8q..8q+7 of a warp hold the 32 columns of one bitmap word.  Rows are processed 8 at a
// time so eight 16-byte loads per thread are in flight before the first shuffle.
__device__ __forceinline__ void k1_a_tile(const float* __restrict__ A, int64_t M, int64_t K, int64_t lda,
                                          uint32_t* __restrict__ abits, int64_t kw, const K1Scratch& z, int64_t tx,
                                          int64_t ty) {
  const int lane = threadIdx.x & 31;
  const int64_t c = tx * kK1Cols + 4 * threadIdx.x;
  const int64_t r0 = ty * kK1Rows;
  const bool col_ok = c < K;
  const uint32_t vmask = col_ok ? (K - c >= 4 ? 0xFu : ((1u << (K - c)) - 1u)) : 0u;
  uint32_t ccount[4] = {0, 0, 0, 0};
  uint32_t warp_total = 0;
  const int64_t rend = min(r0 + kK1Rows, M);
  // with the TC operand enabled, rows run to the 128-row tile boundary (zeros past M)
  const int64_t rend_at = z.at ? min(r0 + kK1Rows, z.m_at) : rend;
  const bool at_ok = z.at != nullptr && c < z.kpad;
  for (int64_t rb = r0; rb < rend_at; rb += 8) {
    float4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u)
      v[u] = (col_ok && rb + u < rend) ? ldg_stream(A + (rb + u) * lda + c) : make_float4(0.f, 0.f, 0.f, 0.f);
    if (at_ok) {
      // A^T tile row k = c+q holds rows rb..rb+7 at offset rb % 128: two 16-byte stores
      const int64_t rt = rb >> 7;
      float* dst = z.at + (rt * z.kpad + c) * 128 + (rb & 127);
      const float e[4][8] = {{v[0].x, v[1].x, v[2].x, v[3].x, v[4].x, v[5].x, v[6].x, v[7].x},
                             {v[0].y, v[1].y, v[2].y, v[3].y, v[4].y, v[5].y, v[6].y, v[7].y},
                             {v[0].z, v[1].z, v[2].z, v[3].z, v[4].z, v[5].z, v[6].z, v[7].z},
                             {v[0].w, v[1].w, v[2].w, v[3].w, v[4].w, v[5].w, v[6].w, v[7].w}};
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        float4* d4 = reinterpret_cast<float4*>(dst + q * 128);
        d4[0] = make_float4(e[q][0], e[q][1], e[q][2], e[q][3]);
        d4[1] = make_float4(e[q][4], e[q][5], e[q][6], e[q][7]);
      }
    }
    if (rb >= rend) continue;
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int64_t i = rb + u;
      const uint32_t nib = nz4(v[u]) & vmask;
#pragma unroll
      for (int q = 0; q < 4; ++q) ccount[q] += (nib >> q) & 1u;
      uint32_t word = nib << (4 * (lane & 7));
      word |= __shfl_xor_sync(0xffffffffu, word, 1);
      word |= __shfl_xor_sync(0xffffffffu, word, 2);
      word |= __shfl_xor_sync(0xffffffffu, word, 4);
      uint32_t cnt = __popc(word);  // per 32-column word; lanes 8q hold distinct words
      cnt = (lane & 7) == 0 ? cnt : 0u;
      cnt += __shfl_xor_sync(0xffffffffu, cnt, 8);
      cnt += __shfl_xor_sync(0xffffffffu, cnt, 16);
      if (i < rend) {
        if ((lane & 7) == 0 && col_ok) abits[i * kw + (c >> 5)] = word;
        if (lane == 0 && cnt) atomicAdd(&z.arow[i], cnt);
        warp_total += cnt;
      }
    }
  }
  if (lane == 0 && warp_total) atomicAdd(&z.tile_sum[ty], warp_total);
  if (col_ok) {
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if (ccount[q]) atomicAdd(&z.acol[c + q], ccount[q]);
  }
}

// --------------------------------------------------------------------------- B tile
// Tile (tx, kw_idx): columns 1024*tx + 4t .. +3 of the padded row (ldb is a multiple of
// 64, padding is zero) over the 32 rows of one k-word.  Lane pairs form 8-column groups;
// 16 lanes form one 64-column region (code).
__device__ __forceinline__ void k1_b_tile(const float* __restrict__ B, int64_t K, int64_t ldb,
                                          uint8_t* __restrict__ codes, int64_t nreg, uint32_t* __restrict__ bgrp,
                                          int64_t kw, const K1Scratch& z, int64_t tx, int64_t kw_idx) {
  const int lane = threadIdx.x & 31;
  const int64_t c = tx * kK1Cols + 4 * threadIdx.x;
  const int64_t k0 = kw_idx * 32;
  const bool col_ok = c < ldb;
  uint32_t gword = 0;   // group k-bitmap word over the 32 rows
  uint32_t slices = 0;  // (k, 16-column slice) pairs with a non-zero, counted by lane%4==0
  const int64_t kend = min(k0 + 32, K);
  for (int64_t kb = k0; kb < kend; kb += 8) {
    float4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u)
      v[u] = (col_ok && kb + u < kend) ? ldg_stream(B + (kb + u) * ldb + c) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int64_t k = kb + u;
      uint32_t any = nz4(v[u]) != 0u;
      any |= __shfl_xor_sync(0xffffffffu, any, 1);  // 8-column group
      gword |= any << (uint32_t)(k - k0);
      const uint32_t sibling = __shfl_xor_sync(0xffffffffu, any, 2);  // other group of the slice
      if ((lane & 3) == 0 && col_ok && k < kend) slices += any | sibling;
      // region code: group j = (lane & 15) >> 1 -> bit 7 - j (MSB first)
      uint32_t code = any << (7 - ((lane & 15) >> 1));
      code |= __shfl_xor_sync(0xffffffffu, code, 2);
      code |= __shfl_xor_sync(0xffffffffu, code, 4);
      code |= __shfl_xor_sync(0xffffffffu, code, 8);
      uint32_t pop = ((lane & 15) == 0 && col_ok) ? __popc(code) : 0u;
      uint32_t nzc = ((lane & 15) == 0 && col_ok) ? (uint32_t)(code != 0) : 0u;
      pop += __shfl_xor_sync(0xffffffffu, pop, 16);
      nzc += __shfl_xor_sync(0xffffffffu, nzc, 16);
      if (k < kend) {
        if ((lane & 15) == 0 && col_ok) codes[k * nreg + (c >> 6)] = (uint8_t)code;
        if (lane == 0) {
          if (pop) atomicAdd(&z.bpop[k], pop);
          if (nzc) atomicAdd(&z.bnz[k], nzc);
        }
      }
    }
  }
  if ((lane & 1) == 0 && col_ok) bgrp[(c >> 3) * kw + kw_idx] = gword;
#pragma unroll
  for (int o = 16; o; o >>= 1) slices += __shfl_xor_sync(0xffffffffu, slices, o);
  if (lane == 0 && slices) atomicAdd(z.slice_nz, (unsigned long long)slices);
  if (z.row_cnt) {
    // K2-SIMT rows of this chunk: one 64-byte row per non-zero (k, 16-column slice)
    const uint32_t smask = gword | __shfl_xor_sync(0xffffffffu, gword, 2);
    uint32_t rows = ((lane & 3) == 0 && col_ok) ? (uint32_t)__popc(smask) : 0u;
#pragma unroll
    for (int o = 16; o; o >>= 1) rows += __shfl_xor_sync(0xffffffffu, rows, o);
    const int64_t c_warp = tx * kK1Cols + 128 * (threadIdx.x >> 5);
    if (lane == 0 && rows && c_warp < ldb) atomicAdd(&z.row_cnt[(c_warp >> 8) * kw + kw_idx], rows);
  }
  if (z.tlive) {
    // K2-TC live k of this chunk: OR of the group k-masks per TC tile; a warp's 128
    // columns touch at most two 192-column tiles (a lane's 4 columns lie in one)
    const int64_t t_lane = c / kTcTileN;
    const int64_t t0 = __shfl_sync(0xffffffffu, t_lane, 0);
    uint32_t w0 = (col_ok && t_lane == t0) ? gword : 0u;
    uint32_t w1 = (col_ok && t_lane != t0) ? gword : 0u;
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      w0 |= __shfl_xor_sync(0xffffffffu, w0, o);
      w1 |= __shfl_xor_sync(0xffffffffu, w1, o);
    }
    if (lane == 0 && w0) atomicOr(&z.tlive[t0 * kw + kw_idx], w0);
    if (lane == 0 && w1) atomicOr(&z.tlive[(t0 + 1) * kw + kw_idx], w1);
  }
}

__device__ void k1_finalize_block(const uint32_t* __restrict__ acol, const uint32_t* __restrict__ bpop,
                                  const uint32_t* __restrict__ bnz, int64_t K, int64_t M, int64_t nreg, int has_a,
                                  int has_b, const unsigned long long* __restrict__ slice_nz,
                                  unsigned long long* __restrict__ out);

// AUTO path choice (stats[7] := 32 for K2-TC, else the K2-SIMT span stays): estimated
// SM-cycles of each path from the plan, constants measured on B200 (K2 choice):
//   K2-SIMT = records * 1158 + row tiles * (span 16: 26 * slice_nz | span 8: 17.5 * pop)
//             records = row tiles * 256-column tiles * 32-k chunks
//   K2-TC   = row tiles * Σ_tiles (24200 + 784 * stages), stages = ceil(live k / 16)
//   + K1 packing traffic at 0.0433 SM-cycles per byte (HBM): K2-SIMT rows 2 x 64 B per
//     non-zero (k, slice); K2-TC step images 3 x 768 B per live (k, tile);
//   each divided by min(148 SMs, its CTA count).
__device__ void k1_choose_path(const K1Scratch& z, int64_t M, int64_t kw, unsigned long long* __restrict__ out) {
  __shared__ unsigned long long s_stage[kK1Threads / 32], s_live[kK1Threads / 32];
  unsigned long long st = 0, live = 0;
  for (int64_t tb = threadIdx.x; tb < z.n_tc; tb += blockDim.x) {
    unsigned long long n = 0;
    for (int64_t c = 0; c < kw; ++c) n += __popc(z.tlive[tb * kw + c]);
    live += n;
    st += (n + 15) / 16;
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    st += __shfl_xor_sync(0xffffffffu, st, o);
    live += __shfl_xor_sync(0xffffffffu, live, o);
  }
  if (lane == 0) {
    s_stage[warp] = st;
    s_live[warp] = live;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long stages = 0, lv = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
      stages += s_stage[w];
      lv += s_live[w];
    }
    const double rt = (double)((M + 127) / 128);
    const double span = (double)out[7];
    const double slice_nz = (double)z.slice_nz[0], pop = (double)out[5];
    const double simt = rt * (double)z.n_tb * (double)kw * 1158.0 + rt * (span == 16.0 ? 26.0 * slice_nz : 17.5 * pop) +
                        0.0433 * 128.0 * slice_nz;
    const double tc = rt * (24200.0 * (double)z.n_tc + 784.0 * (double)stages) + 0.0433 * 3.0 * 768.0 * (double)lv;
    // time ~ work / min(SMs, CTAs): short operands leave SMs idle
    const double par_simt = fmin(148.0, rt * (double)z.n_tb), par_tc = fmin(148.0, rt * (double)z.n_tc);
    if (tc / par_tc < simt / par_simt) out[7] = 32ull;
  }
  __syncthreads();
}

// Block-wide exclusive scan of (cnt[t] + add) -> out[0..n] (out[n] = total); one CTA.
__device__ void k1_block_exclusive_scan(const uint32_t* __restrict__ cnt, int64_t n, uint32_t add,
                                        int64_t* __restrict__ out) {
  __shared__ int64_t carry;
  __shared__ int64_t wsum[kK1Threads / 32];
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int64_t base = 0; base < n; base += kK1Threads) {
    const int64_t t = base + threadIdx.x;
    const int64_t v = t < n ? (int64_t)cnt[t] + add : 0;
    int64_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) wsum[warp] = x;
    __syncthreads();
    int64_t before = carry;
    for (int w = 0; w < warp; ++w) before += wsum[w];
    if (t < n) out[t] = before + x - v;
    __syncthreads();
    if (threadIdx.x == kK1Threads - 1) carry = before + x;
    __syncthreads();
  }
  if (threadIdx.x == 0) out[n] = carry;
  __syncthreads();
}

// ------------------------------------------------------------------ fused K1 pass
// One launch: CTAs [0, nA) are A tiles, [nA, nA + nB) are B tiles; the last CTA to finish
// (threadfence + done-counter) computes the exact counters and plan statistics.
__global__ void __launch_bounds__(kK1Threads, 4)
k1_pass(const float* __restrict__ A, int64_t M, int64_t K, int64_t lda, uint32_t* __restrict__ abits,
        int64_t a_tiles_x, int64_t nA, const float* __restrict__ B, int64_t ldb, uint8_t* __restrict__ codes,
        int64_t nreg, uint32_t* __restrict__ bgrp, int64_t b_tiles_x, int64_t nB, int64_t kw, K1Scratch z,
        int has_a, int has_b, unsigned long long* __restrict__ stats) {
  const int64_t bid = blockIdx.x;
  if (bid < nA)
    k1_a_tile(A, M, K, lda, abits, kw, z, bid % a_tiles_x, bid / a_tiles_x);
  else
    k1_b_tile(B, K, ldb, codes, nreg, bgrp, kw, z, (bid - nA) % b_tiles_x, (bid - nA) / b_tiles_x);
  __shared__ unsigned int last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();  // cumulative over the CTA's writes ordered by the barrier above
    last = atomicAdd(z.done, 1u) == (unsigned int)(nA + nB - 1);
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  if (threadIdx.x == 0) *z.done = 0u;  // ready for the next launch (no other CTA is left)
  k1_finalize_block(z.acol, z.bpop, z.bnz, K, M, nreg, has_a, has_b, z.slice_nz, stats);
  if (z.choose && has_a && has_b) k1_choose_path(z, M, kw, stats);
  if (z.row_cnt && nB > 0) k1_block_exclusive_scan(z.row_cnt, z.n_tb * kw, 3, z.row_off);
  if (nA > 0) {  // exclusive prefix of the 32-row tile sums for k1_csr's row_ptr
    __shared__ int64_t carry;
    __shared__ int64_t wsum[kK1Threads / 32];
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    const int64_t ntile = (M + kK1Rows - 1) / kK1Rows;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int64_t base = 0; base < ntile; base += kK1Threads) {
      const int64_t t = base + threadIdx.x;
      const int64_t v = t < ntile ? (int64_t)z.tile_sum[t] : 0;
      int64_t x = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int64_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      if (lane == 31) wsum[warp] = x;
      __syncthreads();
      int64_t before = carry;
      for (int w = 0; w < warp; ++w) before += wsum[w];
      if (t < ntile) z.tile_prefix[t] = before + x - v;
      __syncthreads();
      if (threadIdx.x == kK1Threads - 1) carry = before + x;
      __syncthreads();
    }
    if (threadIdx.x == 0) z.tile_prefix[ntile] = carry;
  }
}

// --------------------------------------------------------------- CSR index lists
// Per-row ascending index lists (CSR) from the bitmap, no second pass over A.  A CTA owns
// 8 rows (one per warp).  row_ptr comes from the 32-row tile prefix the K1 pass's last CTA
// scanned, plus at most 31 row counts: no separate scan launch.  Each warp then expands its
// row: popc per bitmap word, warp prefix sum, each lane writes its word's set bits.  Index
// type: uint16 when K <= 65536, else uint32.
constexpr int kCsrRows = 8;

template <typename Idx>
__global__ void __launch_bounds__(256) k1_csr(const uint32_t* __restrict__ abits, const uint32_t* __restrict__ arow,
                                              const int64_t* __restrict__ tile_prefix, int64_t M, int64_t kw,
                                              int64_t* __restrict__ row_ptr, Idx* __restrict__ cols) {
  __shared__ int64_t s_off[kCsrRows + 1];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t r0 = (int64_t)blockIdx.x * kCsrRows;
  if (warp == 0) {
    const int64_t t0 = (r0 / 32) * 32;  // first row of r0's 32-row tile
    // counts of rows [t0, r0) (lanes 0..r0-t0-1) and of this CTA's rows (lanes 24..31 -> rows r0..r0+7)
    const int64_t i_pre = t0 + lane;
    uint32_t pre = (i_pre < r0) ? arow[i_pre] : 0u;
#pragma unroll
    for (int o = 16; o; o >>= 1) pre += __shfl_xor_sync(0xffffffffu, pre, o);
    const int64_t i_own = r0 + (lane & 7);
    const uint32_t own = (lane < 8 && i_own < M) ? arow[i_own] : 0u;
    uint32_t x = own;
#pragma unroll
    for (int o = 1; o < 8; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if ((lane & 7) >= o) x += y;
    }
    const int64_t base = tile_prefix[r0 / 32] + (int64_t)pre;
    if (lane < 8) s_off[lane] = base + (int64_t)(x - own);
    if (lane == 7) s_off[8] = base + (int64_t)x;
  }
  __syncthreads();
  const int64_t row = r0 + warp;
  if (threadIdx.x < kCsrRows && r0 + threadIdx.x < M) row_ptr[r0 + threadIdx.x] = s_off[threadIdx.x];
  if (threadIdx.x == 0 && r0 + kCsrRows >= M) row_ptr[M] = s_off[M - r0];
  if (row >= M) return;
  // per 1024-column chunk: lanes expand their words' set bits into the warp's smem buffer
  // at their prefix offsets, then the warp streams the chunk's list out contiguously
  // (coalesced stores instead of 32 scattered 2-byte streams)
  __shared__ Idx s_buf[kCsrRows][1024];
  Idx* buf = s_buf[warp];
  int64_t out = s_off[warp];
  const uint32_t* bits = abits + row * kw;
  for (int64_t w0 = 0; w0 < kw; w0 += 32) {
    const int64_t w = w0 + lane;
    uint32_t word = w < kw ? bits[w] : 0u;
    const uint32_t n = __popc(word);
    uint32_t x = n;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    uint32_t pos = x - n;
    while (word) {
      const int b = __ffs(word) - 1;
      word &= word - 1;
      buf[pos++] = (Idx)(w * 32 + b);
    }
    const uint32_t total = __shfl_sync(0xffffffffu, x, 31);
    __syncwarp();
    for (uint32_t i = lane; i < total; i += 32) cols[out + i] = buf[i];
    __syncwarp();
    out += total;
  }
}

// ---------------------------------------------------------------- counters + stats
// Exact WorkCounters of the coming multiply and plan_stats:
//   lane_fma_ops  = Σ_k acol[k] * 8 * bpop[k]
//   invocations   = Σ_k acol[k] * bnz[k]
//   zero regions  = Σ_k acol[k] * (nreg - bnz[k])
//   rows_skipped  = M*K - Σ_k acol[k]
//   stats         = Σ_k bpop[k], Σ_k (nreg - bnz[k])
// out: u64[9] = {inv, lanes, skipped, zreg, nnzA, pop_total, zero_codes, path, span}
//   span: K2-SIMT mask granularity, from the cost model of DESIGN.md (K2 variants):
//   16-column slices cost ~41 issue slots per non-zero (k, slice), 8-column groups ~23 per
//   non-zero (k, group); pick the cheaper (slice_nz[0] = # non-zero (k, slice) pairs).
__device__ void k1_finalize_block(const uint32_t* __restrict__ acol, const uint32_t* __restrict__ bpop,
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
    out[8] = out[7];  // the K2-SIMT span alone (out[7] may become 32 = K2-TC, k1_choose_path)
  }
}

// ------------------------------------------------------ B steps for K2-TC (dense tiles)
// For each 192-column TC tile tb, the live k (B[k, tile] has a non-zero; tlive) are
// numbered in ascending order, positions p = 0 .. nlive-1, and grouped 8 per MMA step.  Step
// s of tile tb is a 12 KB image at tcb + (tb * maxsteps + s) * 3072 floats: B[k_p][n] for
// its 8 positions split into tf32 hi (first 6 KB) and lo = v - hi (second 6 KB), each in the
// K-major SWIZZLE_NONE core-matrix layout the UMMA descriptor reads with LBO = 128 B and
// SBO = 256 B: element (n, j) at (n % 8) * 16 + (n / 8) * 256 + (j / 4) * 128 + (j % 4) * 4.
// tck[tb][p] = k_p (-1 past nlive, whose B entries are zero); tcn[tb] = nlive.  Every CTA
// of a tile re-derives the tile's chunk prefix from the kw mask words (no scan launch) and
// packs kPtSteps steps; steps straddle chunk boundaries freely (positions, not chunks,
// define a step), so padding is at most 7 k per tile.
constexpr int kPackThreads = 256;  // k1_pack_rows
constexpr int kPtSteps = 4;
constexpr int kPtThreads = 256;

struct PackTcArgs {
  const float* B;
  int64_t ldb;
  const uint32_t* tlive;
  int64_t kw, maxsteps;
  float* tcb;
  int32_t* tck;
  int32_t* tcn;
};

// CTA (bx = step block, tb = tile) of the K2-TC pack; dynamic smem (2 kw + 1) words.
__device__ __forceinline__ void k1_pack_tc_cta(const PackTcArgs& g, int64_t bx, int64_t tb) {
  const float* __restrict__ B = g.B;
  const int64_t ldb = g.ldb, kw = g.kw, maxsteps = g.maxsteps;
  const uint32_t* __restrict__ tlive = g.tlive;
  float* __restrict__ tcb = g.tcb;
  int32_t* __restrict__ tck = g.tck;
  int32_t* __restrict__ tcn = g.tcn;
  extern __shared__ __align__(16) uint32_t pt_smem[];  // masks [kw] | prefix [kw + 1]
  __shared__ int32_t s_k[kPtSteps * 8];
  __shared__ int32_t wsum[kPtThreads / 32];
  uint32_t* s_m = pt_smem;
  int32_t* s_pre = reinterpret_cast<int32_t*>(pt_smem + kw);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t n0 = tb * kTcTileN;
  // chunk masks and their exclusive popcount prefix (block scan, carried over kw / 256 rounds)
  int32_t carry = 0;
  for (int64_t base = 0; base < kw; base += kPtThreads) {
    const int64_t c = base + tid;
    const uint32_t m = c < kw ? tlive[tb * kw + c] : 0u;
    if (c < kw) s_m[c] = m;
    const int32_t v = __popc(m);
    int32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) wsum[warp] = x;
    __syncthreads();
    int32_t before = carry;
    for (int w = 0; w < warp; ++w) before += wsum[w];
    if (c < kw) s_pre[c] = before + x - v;
    int32_t total_round = 0;
    for (int w = 0; w < kPtThreads / 32; ++w) total_round += wsum[w];
    carry += total_round;
    __syncthreads();
  }
  if (tid == 0) s_pre[kw] = carry;
  __syncthreads();
  const int32_t total = carry;
  const int64_t nsteps = (total + 7) / 8;
  if (bx == 0 && tid == 0) tcn[tb] = total;
  const int64_t s0 = bx * kPtSteps;
  if (s0 >= nsteps) return;
  if (tid < kPtSteps * 8) {
    const int64_t p = s0 * 8 + tid;
    int32_t k = -1;
    if (p < total) {
      int64_t lo = 0, hi = kw - 1;  // last chunk c with s_pre[c] <= p
      while (lo < hi) {
        const int64_t mid = (lo + hi + 1) >> 1;
        if (s_pre[mid] <= p) lo = mid;
        else hi = mid - 1;
      }
      uint32_t m = s_m[lo];
      for (int64_t d = p - s_pre[lo]; d; --d) m &= m - 1;
      k = (int32_t)(lo * 32 + __ffs(m) - 1);
    }
    s_k[tid] = k;
    if (p < maxsteps * 8) tck[tb * maxsteps * 8 + p] = k;
  }
  __syncthreads();
  // job = (step, k-quad q, column n): 4 B values -> one float4 hi + one float4 lo
  for (int j = tid; j < kPtSteps * 2 * kTcTileN; j += kPtThreads) {
    const int sl = j / (2 * kTcTileN), q = (j / kTcTileN) & 1, n = j % kTcTileN;
    const int64_t s = s0 + sl;
    if (s >= nsteps) break;
    const bool col_ok = n0 + n < ldb;
    float v[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int32_t k = s_k[sl * 8 + 4 * q + i];
      v[i] = (k >= 0 && col_ok) ? __ldg(B + (int64_t)k * ldb + n0 + n) : 0.0f;
    }
    uint32_t h[4], l[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      h[i] = __float_as_uint(v[i]) & 0xFFFFE000u;
      l[i] = __float_as_uint(v[i] - __uint_as_float(h[i]));
    }
    float* img = tcb + (tb * maxsteps + s) * (kTcTileN * 16);
    const int off = (n & 7) * 4 + (n >> 3) * 64 + q * 32;  // in floats
    *reinterpret_cast<uint4*>(img + off) = make_uint4(h[0], h[1], h[2], h[3]);
    *reinterpret_cast<uint4*>(img + kTcTileN * 8 + off) = make_uint4(l[0], l[1], l[2], l[3]);
  }
}

__global__ void __launch_bounds__(kPtThreads) k1_pack_tc(PackTcArgs g) { k1_pack_tc_cta(g, blockIdx.x, blockIdx.y); }

// ----------------------------------------------------------- B rows for K2-SIMT
// For each 256-column tile tb and 32-k chunk c, a contiguous record at row_off[tb*kw + c]
// (64-byte units): 3 header rows = the 32 group k-masks of the tile's 8-column groups
// (uint32 each, bit kk <-> k = 32c + kk) and the 16 slices' first record rows, then for
// slice j = 0..15 (16 columns = groups
// 2j, 2j+1) and every k of the chunk with a non-zero block in the slice, ascending, the
// raw 16 floats B[k][16j .. 16j+15].  K2-SIMT moves each record with one bulk copy.
struct PackRowsArgs {
  const float* B;
  int64_t ldb;
  const uint32_t* bgrp;
  int64_t kw;
  const int64_t* row_off;
  uint4* rows;
};

// CTA (c = 32-k chunk, tb = 256-column tile) of the K2-SIMT pack.
__device__ __forceinline__ void k1_pack_rows_cta(const PackRowsArgs& g, int64_t c, int64_t tb) {
  const float* __restrict__ B = g.B;
  const int64_t ldb = g.ldb, kw = g.kw;
  const uint32_t* __restrict__ bgrp = g.bgrp;
  const int64_t* __restrict__ row_off = g.row_off;
  uint4* __restrict__ rows = g.rows;
  __shared__ uint32_t s_g[32];
  __shared__ uint32_t s_base[17];
  const int tid = threadIdx.x, lane = tid & 31;
  const int64_t n0 = tb * 256, k0 = c * 32;
  if (tid < 32) {
    const int64_t g = (n0 >> 3) + lane;
    const uint32_t m = (n0 + 8 * lane < ldb) ? bgrp[g * kw + c] : 0u;
    s_g[lane] = m;
    const uint32_t um = m | __shfl_xor_sync(0xffffffffu, m, 1);  // slice union (even lanes)
    uint32_t n = (lane & 1) == 0 ? (uint32_t)__popc(um) : 0u;
    uint32_t x = n;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if ((lane & 1) == 0) s_base[lane >> 1] = x - n;
    if (lane == 31) s_base[16] = x;
  }
  __syncthreads();
  uint4* out = rows + row_off[tb * kw + c] * 4;
  if (tid < 8) out[tid] = make_uint4(s_g[4 * tid], s_g[4 * tid + 1], s_g[4 * tid + 2], s_g[4 * tid + 3]);
  if (tid >= 8 && tid < 12) {  // header row 2: first record row of each slice
    const int q = 4 * (tid - 8);
    out[tid] = make_uint4(3 + s_base[q], 3 + s_base[q + 1], 3 + s_base[q + 2], 3 + s_base[q + 3]);
  }
  const uint32_t total = s_base[16];
  for (uint32_t p = tid; p < total * 4; p += kPackThreads) {
    const uint32_t t = p >> 2, q = p & 3;
    int j = 0;
    while (j < 15 && s_base[j + 1] <= t) ++j;
    uint32_t m = s_g[2 * j] | s_g[2 * j + 1];
    for (uint32_t d = t - s_base[j]; d; --d) m &= m - 1;
    const int kk = __ffs(m) - 1;
    const float4 v = ldg_stream(B + (k0 + kk) * ldb + n0 + 16 * j + 4 * q);
    out[12 + p] = make_uint4(__float_as_uint(v.x), __float_as_uint(v.y), __float_as_uint(v.z), __float_as_uint(v.w));
  }
}

__global__ void __launch_bounds__(kPackThreads) k1_pack_rows(PackRowsArgs g) {
  k1_pack_rows_cta(g, blockIdx.x, blockIdx.y);
}

// AUTO: both packs in one launch (CTAs [0, n_rows) = K2-SIMT rows, the rest = K2-TC steps),
// each CTA gated by the path K1's last CTA chose — one launch instead of two, and the
// gated-out half exits at entry.
__global__ void __launch_bounds__(kPtThreads)
k1_pack_auto(PackRowsArgs gr, int64_t rows_x, int64_t n_rows, PackTcArgs gt, int64_t tc_x,
             const unsigned long long* __restrict__ sel) {
  const int64_t bid = blockIdx.x;
  const bool tc = *sel == 32ull;
  if (bid < n_rows) {
    if (!tc) k1_pack_rows_cta(gr, bid % rows_x, bid / rows_x);
  } else if (tc) {
    k1_pack_tc_cta(gt, (bid - n_rows) % tc_x, (bid - n_rows) / tc_x);
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
