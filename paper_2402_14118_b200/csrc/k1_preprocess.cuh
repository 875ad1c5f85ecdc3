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
//                                   kernel_table.cpp:19) == the BPlan codes; rebuilt from bgrp
//                                   by k1_codes_export on request (not on the hot path)
//   bgrp    uint32 [ngrp][kw]       B group k-bitmaps: bit (k%32) of word k/32 of group g set
//                                   iff B[k, 8g:8g+8] has a non-zero (transposed block masks)
//   bpop    uint32 [K]              Σ popcount(codes[k][:])   (lane ops per A non-zero / 8)
//   bnz     uint32 [K]              # codes != 0 in row k     (kernel invocations per A nz)
#pragma once
#include <cstdint>
#include <type_traits>
#include <cuda_runtime.h>

#include "tc_ptx.cuh"

namespace mmmcu {

constexpr int kK1Threads = 256;  // 8 compute warps; each lane owns 4 columns of a 1024-column tile
constexpr int kK1Block = kK1Threads + 32;  // + the TMA producer warp (k1_pass)
constexpr int kK1Cols = 4 * kK1Threads;  // 1024 columns per CTA tile
constexpr int kK1Rows = 32;              // rows per CTA tile (one 32-bit k-word for B)
#ifndef TD_TN
#define TD_TN 192
#endif
constexpr int kTcTileN = TD_TN;          // K2-TC C tile width (columns)

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
//   za = arow[M] | acol[K] | flags | row ranges;  zb = btot (6 x u64) | group ranges | bpop[K] | bnz[K] | ...
struct K1Scratch {
  uint32_t* arow;
  uint32_t* acol;
  uint32_t* tile_sum;     // [ceil(M/32)] non-zeros per 32-row tile (zeroed)
  uint32_t* nonfinite_a;  // set iff A holds an Inf / NaN / subnormal (zeroed): AUTO keeps K2-SIMT
  int64_t* tile_prefix;   // [ceil(M/32) + 1] exclusive prefix of tile_sum (written by the last CTA)
  // fp16-split operand scales and range guard (K2-TC, AUTO): per A row and per 8-column B
  // group, the bits of max|x| and the complement of the SMALLEST LOCAL MAXIMUM (A: of the
  // row's 128-column chunks, B: of the group's 32-k tiles that hold a non-zero), packed in one
  // zero-initialised 64-bit word (a complement turns the min into a max)
  unsigned long long* rrng;  // [M]: (max << 32) | ~(smallest 128-column chunk max), k1_red_range
  unsigned long long* grng;  // [ldb / 8]: the same per 8-column group over its 32-k tiles
  int64_t ngrp;           // ldb / 8
  uint32_t* wide_a;       // set when some A row's range is too wide for the fp16 split (zeroed);
                          // btot[4] is the same flag for the B groups
  uint32_t* bpop;
  uint32_t* bnz;
  unsigned long long* btot;  // B totals: {Σ non-zero (k, slice), Σ bpop, Σ bnz, Inf/NaN/subnormal seen,
                             //            some group too wide for the fp16 split} (zeroed)
  unsigned int* done;
  unsigned int* next_tile;  // K1 tile counter (dynamic scheduling; reset by the last CTA)
  // K2-TC operands (nullptr when the TC path is not prepared)
  float* at;              // A^T per 128-row tile: at[(rt * kpad + k) * 128 + (i % 128)], zero padded
  int64_t kpad;           // K rounded up to 32
  int64_t m_at;           // M rounded up to 256 (K2-TC pair tiles)
  uint32_t* tlive;        // [n_tc][kw] live-k mask per kTcTileN-column TC tile: bit kk of word c
                          // set iff B[32c + kk, tile columns] has a non-zero (zeroed, atomicOr)
  int64_t* tc_pre;        // [n_tc + 1] exclusive prefix of the tiles' fp16 step counts (k1_fin, AUTO);
                          // tc_pre[n_tc] = -1 when k1_fin did not count the tiles (k1_pack_auto then
                          // deals fixed step blocks).  nullptr outside AUTO
  int32_t* tcn;           // [n_tc] live k per TC tile (k1_fin writes it with tc_pre)
  int64_t n_tb;           // 256-column tiles of B (K2-SIMT records)
  int64_t n_tc;           // kTcTileN-column tiles of B (K2-TC)
  int choose;             // AUTO: pick K2-SIMT vs K2-TC from the cost model (both operand sets built)
  int num_sms;            // the device's SM count (cost-model parallelism)
  int64_t K;              // the contraction length (cost model)
  // the other halves of the double-buffered scratch, zeroed by this pass for the next plan
  uint4* zero_a;
  int64_t zero_a_n;
  uint4* zero_b;
  int64_t zero_b_n;
  // K2-SIMT operand: raw non-zero B block rows per (256-column tile, chunk)
  uint32_t* row_cnt;      // [n_tb][kw] non-zero (k, 16-column slice) rows (zeroed)
  int64_t* row_off;       // [n_tb * kw + 1] exclusive prefix of (row_cnt + 3 header rows), 64-byte units
};


__device__ __forceinline__ bool k1_range_wide(unsigned long long rng);

// AUTO path choice (stats[7] := 32 for K2-TC, else the K2-SIMT span stays): estimated
// SM-cycles of each path from the plan, constants measured on B200 (K2 choice):
//   K2-SIMT = records * 1158 + row tiles * (span 16: 26 * slice_nz | span 8: 17.5 * pop)
//             records = row tiles * 256-column tiles * 32-k chunks
//   K2-TC   = row tiles * Σ_tiles (24200 + 940 * stages), stages = ceil(live k / 32) (fp16
//             split on CTA pairs: 6 MMAs of 16 k per stage; 940 SM-cycles per 128-row stage
//             measured on the dense 4096^3 cells)
//   + the K1 pack of the path's B operand, measured on configs[3] (2.4 GB of B): K2-SIMT rows
//     19 SM-cycles per non-zero (k, slice), K2-TC step images 85 per live (k, tile) (the
//     SIMT pack cost 0.37 ms there, 3.5x the old bytes-at-HBM-rate estimate, which made AUTO
//     pick K2-SIMT, 2.17 ms, over K2-TC, 1.98 ms);
//   each divided by min(#SMs, its CTA count).

// Block-wide exclusive scan of (cnt[t] + add) -> out[0..n] (out[n] = total); one CTA.
// Each thread owns a contiguous segment and loads it with independent loads (one memory
// latency for the whole scan, not one per 256 elements), then one block scan of the sums.
template <typename T, typename F>
__device__ void k1_block_scan_fn(int64_t n, F load, int64_t* __restrict__ out) {
  __shared__ int64_t wsum[32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t seg = (n + blockDim.x - 1) / blockDim.x;
  const int64_t b0 = threadIdx.x * seg, b1 = min(b0 + seg, n);
  int64_t local = 0;
  for (int64_t i = b0; i < b1; ++i) local += (int64_t)load(i);
  int64_t x = local;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int64_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) wsum[warp] = x;
  __syncthreads();
  int64_t before = 0;
  for (int w2 = 0; w2 < warp; ++w2) before += wsum[w2];
  int64_t run = before + x - local;
  for (int64_t i = b0; i < b1; ++i) {
    out[i] = run;
    run += (int64_t)load(i);
  }
  if (threadIdx.x == blockDim.x - 1) out[n] = run;
  __syncthreads();
}

__device__ void k1_block_exclusive_scan(const uint32_t* __restrict__ cnt, int64_t n, uint32_t add,
                                        int64_t* __restrict__ out) {
  k1_block_scan_fn<uint32_t>(n, [&](int64_t i) { return (int64_t)cnt[i] + add; }, out);
}

// The K2-SIMT record offsets on their own (a forced K2-SIMT multiply on an AUTO plan whose
// last CTA chose K2-TC and skipped them).
__global__ void __launch_bounds__(kK1Threads) k1_row_off(const uint32_t* __restrict__ cnt, int64_t n,
                                                         int64_t* __restrict__ out) {
  k1_block_exclusive_scan(cnt, n, 3, out);
}

#ifdef K1_PROF
__device__ unsigned long long* k1_prof = nullptr;  // debug builds: per-CTA globaltimer stamps
__device__ unsigned long long k1_fin_prof[8];      // debug builds: the last CTA's finalize phases
__device__ __forceinline__ unsigned long long k1_now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#endif
#ifdef K1_PROF
#define K1_FIN_STAMP(i) \
  if (threadIdx.x == 0) k1_fin_prof[i] = k1_now()
#else
#define K1_FIN_STAMP(i)
#endif

__host__ __device__ constexpr int k1_fin_smem() { return 4096 * 4; }  // k1_fin's live-k counters
// k1_fin: 32 warps — 16 for the range guard, 12 for the live-k counts, 4 for the tile prefix
constexpr int kFinWarps = 32, kFinRangeWarps = 16, kFinLiveWarps = 12;

// Exclusive scan of n values over a warp group (gsize threads starting at warp w0, named
// barrier bar), each thread a contiguous segment; out[n] = total.
template <typename F>
__device__ void k1_group_scan(int64_t n, F load, int64_t* __restrict__ out, int gtid, int gsize, int bar,
                              int64_t* s_wsum) {
  const int lane = gtid & 31, gw = gtid >> 5, nw = gsize >> 5;
  const int64_t seg = (n + gsize - 1) / gsize;
  const int64_t b0 = gtid * seg, b1 = min(b0 + seg, n);
  int64_t local = 0;
  for (int64_t i = b0; i < b1; ++i) local += (int64_t)load(i);
  int64_t x = local;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int64_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) s_wsum[gw] = x;
  asm volatile("bar.sync %0, %1;" ::"r"(bar), "r"(gsize) : "memory");
  int64_t before = 0;
  for (int w2 = 0; w2 < gw; ++w2) before += s_wsum[w2];
  int64_t run = before + x - local;
  for (int64_t i = b0; i < b1; ++i) {
    out[i] = run;
    run += (int64_t)load(i);
  }
  if (gtid == gsize - 1) out[n] = run;
  (void)nw;
}

// The finalize of a K1 pass (k1_fin, 1024 threads), on the critical path of the call chain,
// so its independent parts run side by side in warp groups with many loads in flight (one
// or two global round trips each instead of a chain): warps 0-15 the fp16 range guard,
// 16-27 the live k per TC tile (AUTO cost model), 28-31 the CSR's 32-row tile prefix; then thread 0 the plan totals and the AUTO
// path choice; then (K2-SIMT possible only) the record-offset scan with all threads.
__device__ void k1_finalize(const K1Scratch& z, int64_t M, int64_t K, int64_t nreg, int64_t kw, int has_a, int has_b,
                            int64_t nA, int64_t nB, unsigned long long* __restrict__ stats, uint32_t* s_tcnt) {
  __shared__ uint32_t s_wide[2];
  __shared__ unsigned long long s_st, s_live;
  __shared__ int64_t s_wsum[kFinWarps];
  __shared__ int64_t s_wsum_tc[kFinLiveWarps];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const bool choose = z.choose && has_a && has_b;
  const int64_t nw = z.n_tc * kw;
  const bool fits = choose && z.n_tc <= k1_fin_smem() / 4 && nw < 0x7fffffff;
  if (tid < 2) s_wide[tid] = 0u;
  for (int64_t t = tid; fits && t < z.n_tc; t += blockDim.x) s_tcnt[t] = 0u;
  __syncthreads();
  K1_FIN_STAMP(1);
  if (warp < kFinRangeWarps) {  // ---- range guard
    constexpr int kT = 32 * kFinRangeWarps;
    auto scan = [&](const unsigned long long* __restrict__ w, int64_t n) {
      bool wide = false;
      for (int64_t i0 = tid; i0 < n; i0 += 4 * kT) {
        unsigned long long v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int64_t i = i0 + u * kT;
          v[u] = i < n ? w[i] : 0ull;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) wide |= k1_range_wide(v[u]);
      }
      return wide;
    };
    const bool wa = nA > 0 && z.rrng ? scan(z.rrng, M) : false;
    const bool wb = nB > 0 && z.grng ? scan(z.grng, z.ngrp) : false;
    if (__any_sync(0xffffffffu, wa) && lane == 0) atomicOr(&s_wide[0], 1u);
    if (__any_sync(0xffffffffu, wb) && lane == 0) atomicOr(&s_wide[1], 1u);
  } else if (warp < kFinRangeWarps + kFinLiveWarps) {  // ---- live k per TC tile (popcount of its kw words)
    constexpr int kT = 32 * kFinLiveWarps;
    const int gt = tid - 32 * kFinRangeWarps, gw = gt >> 5;
    unsigned long long st = 0, live = 0;
    if (fits) {
      for (int64_t i0 = gt; i0 < nw; i0 += 8 * kT) {
        uint32_t v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int64_t i = i0 + u * kT;
          v[u] = i < nw ? z.tlive[i] : 0u;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int64_t i = i0 + u * kT;
          if (v[u]) atomicAdd(&s_tcnt[(uint32_t)i / (uint32_t)kw], (uint32_t)__popc(v[u]));
        }
      }
      asm volatile("bar.sync 3, %0;" ::"r"(kT) : "memory");
      for (int64_t tb = gt; tb < z.n_tc; tb += kT) {
        live += s_tcnt[tb];
        st += (s_tcnt[tb] + 31) / 32;  // fp16-split stages of 32 live k
      }
    } else if (choose) {
      for (int64_t tb = gw; tb < z.n_tc; tb += kFinLiveWarps) {  // a warp per tile
        uint32_t n = 0;
        for (int64_t w = lane; w < kw; w += 32) n += __popc(z.tlive[tb * kw + w]);
#pragma unroll
        for (int o = 16; o; o >>= 1) n += __shfl_xor_sync(0xffffffffu, n, o);
        if (lane == 0) {
          live += n;
          st += (n + 31) / 32;
        }
      }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      st += __shfl_xor_sync(0xffffffffu, st, o);
      live += __shfl_xor_sync(0xffffffffu, live, o);
    }
    if (gt == 0) {
      s_st = 0;
      s_live = 0;
    }
    asm volatile("bar.sync 3, %0;" ::"r"(kT) : "memory");
    if (lane == 0) {
      atomicAdd(&s_st, st);
      atomicAdd(&s_live, live);
    }
    // the tiles' live counts and the exclusive prefix of their fp16 step counts: k1_pack_auto
    // cuts the concatenated steps of all tiles into equal shares, one per CTA
    if (z.tc_pre && z.choose) {
      if (fits) {
        for (int64_t tb = gt; tb < z.n_tc; tb += kT) z.tcn[tb] = (int32_t)s_tcnt[tb];
        k1_group_scan(z.n_tc, [&](int64_t i) { return (s_tcnt[i] + 15u) / 16u; }, z.tc_pre, gt, kT, 3, s_wsum_tc);
      } else if (gt == 0) {
        z.tc_pre[z.n_tc] = -1;
      }
    }
  } else {  // ---- the CSR's 32-row tile prefix
    if (nA > 0) {
      const int64_t ntile = (M + kK1Rows - 1) / kK1Rows;
      const uint32_t* ts = z.tile_sum;
      constexpr int kT = 32 * (kFinWarps - kFinRangeWarps - kFinLiveWarps);
      k1_group_scan(ntile, [&](int64_t i) { return ts[i]; }, z.tile_prefix, tid - (kFinWarps * 32 - kT), kT, 4,
                    s_wsum);
    }
  }
  __syncthreads();
  K1_FIN_STAMP(2);
  if (tid == 0) {
    // plan totals: pop_total, zero codes and the K2-SIMT span from the B tiles' totals
    // btot = {Σ non-zero (k, slice), Σ bpop, Σ bnz} (span: 16-column slices cost ~41 issue
    // slots per non-zero (k, slice), 8-column groups ~23 per non-zero (k, group))
    const unsigned long long pop = has_b ? z.btot[1] : 0ull, bnz = has_b ? z.btot[2] : 0ull;
    stats[5] = pop;
    stats[6] = has_b ? (unsigned long long)(K * nreg) - bnz : 0ull;
    stats[7] = (has_b && 41ull * z.btot[0] > 23ull * pop) ? 8ull : 16ull;
    stats[8] = stats[7];  // the K2-SIMT span alone (stats[7] may become 32 = K2-TC)
    if (s_wide[0]) *z.wide_a = 1u;
    if (s_wide[1]) z.btot[4] = 1ull;
    if (choose) {
      // AUTO path choice (k1_finalize; stats[7] := 32 for K2-TC): estimated SM-cycles of each path, see
      // the cost-model comment at the top of this file
      const double rt = (double)((M + 127) / 128);
      const double span = (double)stats[7];
      const double slice_nz = (double)z.btot[0], pp = (double)pop;
      const double simt = rt * (double)z.n_tb * (double)kw * 1158.0 +
                          rt * (span == 16.0 ? 26.0 * slice_nz : 17.5 * pp) + 19.0 * slice_nz;
      const double tc = rt * (24200.0 * (double)z.n_tc + 940.0 * (double)s_st) + 85.0 * (double)s_live;
      const double sms = (double)z.num_sms;
      const double par_simt = fmin(sms, rt * (double)z.n_tb), par_tc = fmin(sms, rt * (double)z.n_tc);
      const bool nonfinite = *z.nonfinite_a != 0u || z.btot[3] != 0ull;
      const bool wide = *z.wide_a != 0u || z.btot[4] != 0ull;
      if (!nonfinite && !wide && tc / par_tc < simt / par_simt) stats[7] = 32ull;
    }
  }
  __syncthreads();
  K1_FIN_STAMP(3);
  // the K2-SIMT record offsets only when K2-SIMT can run (its pack is gated out otherwise)
  if (z.row_cnt && nB > 0 && !(z.choose && (stats[7] == 32ull || stats[7] == 48ull)))
    k1_block_exclusive_scan(z.row_cnt, z.n_tb * kw, 3, z.row_off);
  K1_FIN_STAMP(4);
}

// ------------------------------------------------------------------ fused K1 pass
// One persistent launch (2 CTAs per SM): tiles [0, nA) are A tiles, [nA, nA + nB) B tiles,
// CTA b takes tiles b, b + gridDim.x, ...  Rows reach the SM by TMA bulk copies (one per
// row segment of <= 4 KB) into a ring of 8-row stages (k1_pass<ST, CTAS>), so HBM sees the copies of
// the next stages while the warps run the mask / shuffle / A^T work of the current one:
// thread 0 refills a stage as soon as the 8 warps have read it into registers.  The last
// CTA to finish (threadfence + done-counter) computes the exact counters, plan statistics
// and the AUTO path choice.

// Rows per ring stage: an 8-row group (the tile functions' unit) spans 8 / kK1SR stages, so a
// stage is released, and refilled, after half a group (finer-grained refills keep more of the
// ring in flight while the warps compute: 4 x 16 KB measured faster than 2 x 32 KB).
#ifndef K1_SR
#define K1_SR 4
#endif
constexpr int kK1SR = K1_SR;
static_assert(8 % kK1SR == 0, "stage rows must divide the 8-row group");

template <int ST>
struct K1RingT {
  float4 buf[ST][kK1SR][kK1Threads];  // kK1SR rows x 1024 columns per stage
  uint64_t full[ST];
  uint64_t empty[ST];
  int64_t tile[ST];               // the tile this stage's group belongs to (-1: no more)
};

__device__ __forceinline__ void k1_bulk(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   (uint32_t)__cvta_generic_to_shared(dst)),
               "l"(src), "r"(bytes), "r"((uint32_t)__cvta_generic_to_shared(bar))
               : "memory");
}
__device__ __forceinline__ void k1_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "K1W_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra K1W_%=;\n\t}" ::"r"((uint32_t)__cvta_generic_to_shared(bar)),
      "r"(parity)
      : "memory");
}

struct K1Args {
  const float* A;
  int64_t M, K, lda;
  uint32_t* abits;
  int64_t a_tx, nA;
  const float* B;
  int64_t ldb;
  int64_t nreg;
  uint32_t* bgrp;
  int64_t b_tx, nB, kw;
};

// Row groups in consumption order: the tiles of this CTA, each tile's 8-row groups.
// Tiles are handed out dynamically (atomic counter): the producer takes the next tile when
// it starts issuing its groups and tags every stage with the tile, so the compute warps
// follow the same sequence; a CTA that runs fast takes more tiles (no static tail).
#ifndef K1_STATIC_EIGHTHS
// eighths of the tiles dealt statically, the rest by an atomic counter.  Alone, 0 / 4 / 7 measured
// 42.9 / 42.4 / 44.1 us; 0 (all dynamic) is the default because a pass that shares the GPU
// with another stream's K2-TC has only some of its CTAs resident, and statically dealt tiles
// would wait for the others (sweep step on 2 streams: 21.8 -> 21.1 ms)
#define K1_STATIC_EIGHTHS 0
#endif
struct K1Cursor {
  const K1Args* g;
  const K1Scratch* z;
  int64_t t, rb, rend, c0;  // current tile, its next group's first row, row end, first column
  const float* base;
  int64_t ld, cols;         // row stride, readable columns of the operand
  int64_t n_static = 0;     // this CTA's statically assigned tiles taken so far
  // ~7/8 of the tiles are dealt statically (CTA b: b, b + grid, ...), the rest handed out
  // through an atomic counter to whichever CTA is free first: balance without a
  // contended counter on every tile
  __device__ int64_t grab() {
    const int64_t total = g->nA + g->nB;
    const int64_t per = (total * K1_STATIC_EIGHTHS / 8) / gridDim.x;  // static tiles per CTA
    if (n_static < per) return blockIdx.x + (n_static++) * (int64_t)gridDim.x;
    return per * (int64_t)gridDim.x + (int64_t)atomicAdd(z->next_tile, 1u);
  }
  __device__ void next_tile() {
    t = grab();
    tile_setup();
  }
  __device__ void tile_setup() {
    const K1Args& a = *g;
    while (t < a.nA + a.nB) {
      if (t < a.nA) {
        const int64_t tx = t % a.a_tx, ty = t / a.a_tx;
        rb = ty * kK1Rows;
        const int64_t rows_end = z->at ? z->m_at : a.M;  // A^T tiles run to the 128-row boundary
        rend = min(rb + kK1Rows, rows_end);
        c0 = tx * kK1Cols;
        base = a.A;
        ld = a.lda;
        cols = (a.K + 3) & ~int64_t(3);
        // copies stop at row M (rows past it are zeros, not read)
        if (rb < rend) return;
      } else {
        const int64_t tt = t - a.nA, tx = tt % a.b_tx, kwi = tt / a.b_tx;
        rb = kwi * 32;
        rend = min(rb + 32, a.K);
        c0 = tx * kK1Cols;
        base = a.B;
        ld = a.ldb;
        cols = a.ldb;
        if (rb < rend) return;
      }
      t = grab();
    }
  }
  __device__ bool done() const { return t >= g->nA + g->nB; }
  // issue this group's row copies into stage slot s, then advance
  template <class R>
  __device__ void issue(R& r, int s) {
    const K1Args& a = *g;
    const int64_t lim = t < a.nA ? a.M : rend;  // A rows past M are zeros: not read
    const int64_t rows_valid = lim - rb >= kK1SR ? kK1SR : (lim - rb > 0 ? lim - rb : 0);
    const uint32_t bytes = (uint32_t)((cols - c0 >= kK1Cols ? kK1Cols : cols - c0) * 4);
    r.tile[s] = t;
    mbar_expect(&r.full[s], (uint32_t)rows_valid * bytes);
    for (int u = 0; u < rows_valid; ++u) k1_bulk(&r.buf[s][u][0], base + (rb + u) * ld + c0, bytes, &r.full[s]);
    rb += kK1SR;
    if (rb >= rend && (rb & 7) == 0) next_tile();  // whole 8-row groups (a group's stages share a tile)
  }
  // no more tiles: one stage tagged -1 tells the compute warps to stop
  template <class R>
  __device__ void finish(R& r, int s) {
    r.tile[s] = -1;
    mbar_expect(&r.full[s], 0u);
  }
  __device__ static void mbar_expect(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(bar)),
                 "r"(bytes)
                 : "memory");
  }
};

// Loader for the tile functions: the next 8-row group from the ring (thread 0 also refills).
template <int ST>
struct K1RingLoaderT {
  K1RingT<ST>& r;
  K1Cursor& cur;
  uint32_t J;  // groups consumed
  // the tile of the next group (-1: done); waits for the stage to land
  __device__ int64_t peek() {
    const int s = J % ST;
    k1_wait(&r.full[s], (J / ST) & 1u);
    return r.tile[s];
  }
  // x[u][j] = row u, column colofs[j] of the next 8-row group (0 for !ok[j] or u >= nvalid)
  // FULL: all 8 rows and all columns of the group are valid (no per-element selects)
  template <bool FULL = false>
  __device__ void rows(float (&x)[8][4], const int (&colofs)[4], const bool (&ok)[4], int nvalid) {
#pragma unroll
    for (int h = 0; h < 8 / kK1SR; ++h) {  // the group's stages, in order
      const int s = J % ST;
      k1_wait(&r.full[s], (J / ST) & 1u);
      const float* st = reinterpret_cast<const float*>(&r.buf[s][0][0]);
#pragma unroll
      for (int v = 0; v < kK1SR; ++v) {
        const int u = h * kK1SR + v;
#pragma unroll
        for (int j = 0; j < 4; ++j)
          x[u][j] = (FULL || (ok[j] && u < nvalid)) ? st[v * kK1Cols + colofs[j]] : 0.0f;
      }
      // the TMA refill of this slot (async proxy) must not overtake these generic-proxy reads
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if ((threadIdx.x & 31) == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(
                                                    (uint32_t)__cvta_generic_to_shared(&r.empty[s]))
                                                : "memory");
      ++J;
    }
  }
  // v[u] = row u, columns col4 .. col4+3 of the next 8-row group (one LDS.128 per row: a warp
  // reads 512 contiguous bytes); zeros for !ok or u >= nvalid
  template <bool FULL = false>
  __device__ void rows4(uint4 (&v)[8], int col4, bool ok, int nvalid) {
#pragma unroll
    for (int h = 0; h < 8 / kK1SR; ++h) {
      const int s = J % ST;
      k1_wait(&r.full[s], (J / ST) & 1u);
      const uint4* st = reinterpret_cast<const uint4*>(&r.buf[s][0][0]);
#pragma unroll
      for (int q = 0; q < kK1SR; ++q) {
        const int u = h * kK1SR + q;
        v[u] = (FULL || (ok && u < nvalid)) ? st[q * (kK1Cols / 4) + (col4 >> 2)] : make_uint4(0u, 0u, 0u, 0u);
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if ((threadIdx.x & 31) == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(
                                                    (uint32_t)__cvta_generic_to_shared(&r.empty[s]))
                                                : "memory");
      ++J;
    }
  }
};

// Ballot formulation over the smem ring (k1_pass): warp w owns the 32-column chunks
// {2w, 2w+1, 2w+16, 2w+17} of the 1024-column tile (a 64-column region is one warp's chunk
// pair) and lane l column l of each chunk, so one __ballot_sync per (row, chunk) IS the
// 32-bit mask word: bitmap words, region codes, group / slice masks and popcounts all come
// from warp-uniform ballots instead of per-lane shuffle chains.
__device__ __forceinline__ int k1_chunk(int w, int j) { return 2 * w + (j & 1) + 16 * (j >> 1); }

// Values K2-TC cannot reproduce within the tolerance: Inf / NaN (0 * Inf terms) and
// subnormals (tf32 operands are flushed).  The tile loops track max / min of the |x| bit
// patterns; K1 flags them and AUTO keeps K2-SIMT.

// Fold a tile's local maxima (bits of |x|: largest mx, smallest mn) into a row's / group's
// range word rng = (max << 32) | ~(smallest local max) with two non-returning 32-bit atomic
// maxima (RED.MAX: the complement turns the min into a max), so no tile waits on a round
// trip; whether the final range is too wide for the fp16 split is decided once all tiles are
// in (k1_finalize, the last CTA).
__device__ __forceinline__ void k1_red_range(unsigned long long* rng, uint32_t mx, uint32_t mn) {
  uint32_t* w = reinterpret_cast<uint32_t*>(rng);  // little-endian: w[1] = high word
  atomicMax(w + 1, mx);
  atomicMax(w, ~mn);
}
// A final range word too wide for the fp16 split: max exponent outside [-86, 114], or local
// maxima more than 2^17 apart (0: no non-zero seen)
__device__ __forceinline__ bool k1_range_wide(unsigned long long rng) {
  const uint32_t cmax = (uint32_t)(rng >> 32), cmin = ~(uint32_t)rng;
  if (cmax == 0u) return false;
  const int emax = (int)(cmax >> 23) - 127, emin = (int)(cmin >> 23) - 127;
  return emax < -86 || emax > 114 || emax - emin > 17;
}

// A tiles: warp w owns the contiguous 128 columns 128w .. 128w+127 (chunks 4w .. 4w+3), so
// one warp-wide max per row is the max of a contiguous 128-column chunk of the row
__device__ __forceinline__ int k1_chunk_a(int w, int j) { return 4 * w + j; }

template <typename Loader>
__device__ __forceinline__ void k1_a_tile_b(Loader& ld, int64_t M, int64_t K, uint32_t* __restrict__ abits, int64_t kw,
                                            const K1Scratch& z, int64_t tx, int64_t ty) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t c0 = tx * kK1Cols, r0 = ty * kK1Rows;
  int colofs[4];
  bool ok[4];
  int64_t col[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    colofs[j] = 32 * k1_chunk_a(w, j) + lane;
    col[j] = c0 + colofs[j];
    ok[j] = col[j] < K;
  }
  // |x| bit patterns: max (>= 0x7F800000 = Inf / NaN) and min of |x| - 1 (unsigned: zeros wrap
  // to 0xFFFFFFFF; < 0x7FFFFF = a subnormal) for the operand flags; per row the max of each
  // warp's contiguous 128-column chunk (one warp max per row), folded over the 8 warps at the
  // end of the tile into one atomic pair per row (row max, smallest non-zero chunk max)
  uint32_t amax_b = 0u, amin_b = 0xFFFFFFFFu, warp_total = 0u;
  __shared__ uint32_t s_ab[kK1Rows][32];  // the tile's bitmap words (row, chunk)
  __shared__ uint32_t s_cm[kK1Rows][8];   // per row, the max of each warp's 128-column chunk
  __shared__ uint32_t s_cnt[kK1Rows][8];  // per row, the non-zeros of each warp's chunk
  const int64_t rend = min(r0 + kK1Rows, M);
  const int64_t rend_at = z.at ? min(r0 + kK1Rows, z.m_at) : rend;
  // one 8-row group: the A^T stores, then per row the ballot words, counts and ranges.  FULL:
  // all 8 rows and all 1024 columns valid (the common case; no per-element bounds tests)
  auto group = [&](auto full_tag, int64_t rb, int nvalid) {
    constexpr bool FULL = decltype(full_tag)::value;
    float x[8][4];
    ld.template rows<FULL>(x, colofs, ok, nvalid);
#ifdef K1_NOCOMP_A
    return;
#endif
#ifdef K1_NOAT
    if (false) {
#else
    if (z.at) {
#endif
      // A^T tile row k = col holds rows rb..rb+7 at offset rb % 128: two 16-byte stores
      const int64_t rt = rb >> 7;
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (FULL || col[j] < z.kpad) {
          // one 32-byte store (STG.256: a whole sector per request; two 16-byte stores per
          // sector made the A^T writes L2-request bound)
          float* d = z.at + (rt * z.kpad + col[j]) * 128 + (rb & 127);
          asm volatile("st.global.v8.f32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(d), "f"(x[0][j]),
                       "f"(x[1][j]), "f"(x[2][j]), "f"(x[3][j]), "f"(x[4][j]), "f"(x[5][j]), "f"(x[6][j]),
                       "f"(x[7][j])
                       : "memory");
        }
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      if (!FULL && u >= nvalid) break;
      const int64_t i = rb + u;
      uint32_t cnt = 0, rmx = 0u, rmn = 0xFFFFFFFFu;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const bool nz = x[u][j] != 0.0f;
        const uint32_t ab = __float_as_uint(x[u][j]) & 0x7FFFFFFFu;
        rmx = max(rmx, ab);
        rmn = min(rmn, ab - 1u);
        const uint32_t m = __ballot_sync(0xffffffffu, nz);
        cnt += __popc(m);
        if (lane == j) s_ab[i - r0][k1_chunk_a(w, j)] = m;  // staged: written row-contiguous below
      }
#ifndef K1_NO_RANGE
      if (z.rrng) {  // max of the row's 128-column chunk (this warp's columns)
        const uint32_t cm = __reduce_max_sync(0xffffffffu, rmx);
        if (lane == 0) s_cm[i - r0][w] = cm;
      }
#endif
      amax_b = max(amax_b, rmx);
      amin_b = min(amin_b, rmn);
      if (lane == 0) s_cnt[i - r0][w] = cnt;
      warp_total += cnt;
    }
  };
  const bool cols_full = c0 + kK1Cols <= K;
  for (int64_t rb = r0; rb < rend_at; rb += 8) {
    const int nvalid = rend - rb >= 8 ? 8 : (rend - rb > 0 ? (int)(rend - rb) : 0);
    if (cols_full && nvalid == 8) group(std::true_type{}, rb, 8);
    else group(std::false_type{}, rb, nvalid);
  }
  if (lane == 0 && warp_total) atomicAdd(&z.tile_sum[ty], warp_total);
  {
    const uint32_t mb = __reduce_max_sync(0xffffffffu, amax_b), mn = __reduce_min_sync(0xffffffffu, amin_b);
    if (lane == 0 && (mb >= 0x7F800000u || mn < 0x007FFFFFu)) atomicOr(z.nonfinite_a, 1u);
  }
  // (per-column non-zero counts, for the WorkCounters only, come from the bitmap on request:
  // k1_bitcols)
  // the tile's bitmap words, row by row (32 words = 128 contiguous bytes per row)
  asm volatile("bar.sync 2, %0;" ::"r"(kK1Threads) : "memory");
  const int64_t wd = (c0 >> 5) + lane;
  for (int rr = w; rr < kK1Rows; rr += kK1Threads / 32) {
    if (r0 + rr < rend && wd < kw) abits[(r0 + rr) * kw + wd] = s_ab[rr][lane];
  }
  if (threadIdx.x < kK1Rows && r0 + threadIdx.x < rend) {  // one count atomic per row and tile
    uint32_t n = 0;
#pragma unroll
    for (int q = 0; q < 8; ++q) n += s_cnt[threadIdx.x][q];
    if (n) atomicAdd(&z.arow[r0 + threadIdx.x], n);
  }
#ifndef K1_NO_RANGE
  if (z.rrng && threadIdx.x < kK1Rows && r0 + threadIdx.x < rend) {  // one RED pair per row and tile
    const int rr = threadIdx.x;
    uint32_t mx = 0u, mn = 0xFFFFFFFFu;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      // chunks past K hold no column: their max stays 0 and is no local max
      const uint32_t v = (c0 + 128 * q < K) ? s_cm[rr][q] : 0u;
      mx = max(mx, v);
      if (v) mn = min(mn, v);
    }
    if (mx) k1_red_range(&z.rrng[r0 + rr], mx, mn);
  }
#endif
  asm volatile("bar.sync 2, %0;" ::"r"(kK1Threads) : "memory");
}

// B tile: warp w owns the contiguous 128 columns 128w .. 128w+127 of the 1024-column tile and
// lane l the 4 columns 4l .. 4l+3 (half of an 8-column group): per row one LDS.128, the
// lane's half-group k-mask bit (hw, no ballot), and the range of its |x| bit patterns with
// 3-input integer min / max (VIMNMX3 / VIADDMNMX) — ~15 instructions per row and 128 columns
// (the one-column-per-lane ballot formulation took ~36 and left the pass issue-bound on
// B-dominated streams).  Everything else — group k-masks (gword = the two half masks OR-ed;
// lane g < 16 keeps group g), region / slice / plan totals, the TC tiles' live-k words —
// follows from the 32-bit masks at the end of the tile.  The codes themselves are not stored:
// k1_codes_export rebuilds them from bgrp when a caller asks (export path).
template <typename Loader>
__device__ __forceinline__ void k1_b_tile_b(Loader& ld, int64_t K, int64_t ldb, int64_t nreg,
                                            uint32_t* __restrict__ bgrp, int64_t kw, const K1Scratch& z, int64_t tx,
                                            int64_t kwi) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t c0 = tx * kK1Cols, k0 = kwi * 32;
  const int col4 = 128 * w + 4 * lane;       // this lane's 4 columns within the tile
  const bool ok4 = c0 + col4 < ldb;          // (ldb is a multiple of 64: all 4 or none)
  // lane g < 16 owns 8-column group g of the warp (lanes 2g, 2g+1 hold its halves); lanes 0..7
  // are the warp's first 64-column region, lanes 8..15 its second
  const int64_t gcol = c0 + 128 * w + 8 * lane;
  const bool gown = lane < 16 && gcol < ldb;
  uint32_t hw = 0;                                // k-mask of this lane's half group
  uint32_t cmx = 0u, cmn = 0xFFFFFFFFu;           // max |x| bits, min (|x| bits - 1) of the lane's columns
  const int64_t kend = min(k0 + 32, K);
  const bool cols_full = c0 + kK1Cols <= ldb;
#pragma unroll
  for (int kb8 = 0; kb8 < 4; ++kb8) {
    const int64_t kb = k0 + 8 * kb8;
    if (kb >= kend) break;
    uint4 v[8];
    if (cols_full && kend - kb >= 8) ld.template rows4<true>(v, col4, ok4, 8);
    else ld.rows4(v, col4, ok4, kend - kb >= 8 ? 8 : (int)(kend - kb));
#ifdef K1_NOCOMP_B
    continue;
#endif
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const uint32_t a = v[u].x & 0x7FFFFFFFu, b = v[u].y & 0x7FFFFFFFu, c = v[u].z & 0x7FFFFFFFu,
                     d = v[u].w & 0x7FFFFFFFu;
      const uint32_t m4 = max(max(a, b), max(c, d));
      cmx = max(cmx, m4);
      cmn = min(min(cmn, min(a - 1u, b - 1u)), min(c - 1u, d - 1u));
      if (m4) hw |= 1u << (8 * kb8 + u);  // exact zero test: |x| bits != 0
    }
  }
  const uint32_t gw2 = hw | __shfl_xor_sync(0xffffffffu, hw, 1);  // the group's mask (both halves)
  uint32_t gword = __shfl_sync(0xffffffffu, gw2, (2 * lane) & 31);
  if (!gown) gword = 0;
  if (gown) bgrp[(gcol >> 3) * kw + kwi] = gword;
  // plan totals of the warp: Σ_k # non-zero groups = Σ_g popc(gword_g); Σ_k # non-zero
  // regions = popc of each region's OR-ed masks (lanes 0-7 / 8-15).  The per-k factors
  // (bpop, bnz) are derived from bgrp only when counters are requested (k1_counters).
  uint32_t pop_w = __popc(gword);
  uint32_t ror = gword;
  ror |= __shfl_xor_sync(0xffffffffu, ror, 1);
  ror |= __shfl_xor_sync(0xffffffffu, ror, 2);
  ror |= __shfl_xor_sync(0xffffffffu, ror, 4);
  uint32_t nz_w = (lane == 0 || lane == 8) ? (uint32_t)__popc(ror) : 0u;
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    pop_w += __shfl_xor_sync(0xffffffffu, pop_w, o);
    nz_w += __shfl_xor_sync(0xffffffffu, nz_w, o);
  }
  {
    // this tile's max of each 8-column group (even lane: halves 2g, 2g+1 = lanes l, l+1)
    const uint32_t mx = max(cmx, __shfl_xor_sync(0xffffffffu, cmx, 1));
    const int64_t g = (c0 + col4) >> 3;
    if (z.grng && (lane & 1) == 0 && mx && 8 * g < ldb) k1_red_range(&z.grng[g], mx, mx);
    const uint32_t mb = __reduce_max_sync(0xffffffffu, cmx), mn = __reduce_min_sync(0xffffffffu, cmn);
    if (lane == 0 && (mb >= 0x7F800000u || mn < 0x007FFFFFu)) atomicOr(&z.btot[3], 1ull);
  }
  if (lane == 0 && pop_w) atomicAdd(&z.btot[1], (unsigned long long)pop_w);
  if (lane == 0 && nz_w) atomicAdd(&z.btot[2], (unsigned long long)nz_w);
  // (k, 16-column slice) pairs with a non-zero: even group lanes own slice (2s, 2s+1)
  const uint32_t sib = __shfl_down_sync(0xffffffffu, gword, 1);
  uint32_t srows = (gown && (lane & 1) == 0) ? (uint32_t)__popc(gword | sib) : 0u;
  if (z.row_cnt && srows) atomicAdd(&z.row_cnt[(gcol >> 8) * kw + kwi], srows);
#pragma unroll
  for (int o = 16; o; o >>= 1) srows += __shfl_xor_sync(0xffffffffu, srows, o);
  if (lane == 0 && srows) atomicAdd(&z.btot[0], (unsigned long long)srows);
  // the TC tile's live-k word (non-returning RED.OR; the live counts per tile are taken from
  // the words by the last CTA, k1_finalize, and by the TC pack)
  if (z.tlive && gword) atomicOr(&z.tlive[(gcol / kTcTileN) * kw + kwi], gword);
}

// Region codes (kernel_table.cpp:19: bit 7-j <-> 8-column group j, MSB first) from the group
// k-masks — export path (BPlan codes), one thread per (k, region).
__global__ void k1_codes_export(const uint32_t* __restrict__ bgrp, int64_t K, int64_t nreg, int64_t kw,
                                uint8_t* __restrict__ codes) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= K * nreg) return;
  const int64_t k = t / nreg, r = t % nreg;
  uint32_t code = 0;
#pragma unroll
  for (int g = 0; g < 8; ++g) code |= ((bgrp[(8 * r + g) * kw + (k >> 5)] >> (k & 31)) & 1u) << (7 - g);
  codes[t] = (uint8_t)code;
}

// ST ring stages of 32 KB per CTA, CTAS CTAs per SM: 2 x 3 for operands of a few thousand
// tiles (the sweep), 6 x 1 for large ones (cfg4's 2.25 GiB B: K1 1.8 -> 1.3 ms), chosen at
// launch by the tile count
template <int ST, int CTAS>
__global__ void __launch_bounds__(kK1Block, CTAS)
k1_pass(K1Args g, K1Scratch z) {
  tc::pdl_wait();  // launched with programmatic serialization after the previous call's last kernel
  {  // the next plan's scratch halves (nothing reads them any more: the previous kernels are done)
    const int64_t i0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, st = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = i0; i < z.zero_a_n; i += st) z.zero_a[i] = make_uint4(0u, 0u, 0u, 0u);
    for (int64_t i = i0; i < z.zero_b_n; i += st) z.zero_b[i] = make_uint4(0u, 0u, 0u, 0u);
  }
#ifdef K1_PROF
  const unsigned long long t_start = k1_now();
#endif
  extern __shared__ __align__(128) uint8_t k1_raw[];
  K1RingT<ST>& r = *reinterpret_cast<K1RingT<ST>*>(k1_raw + ((128 - ((uint32_t)__cvta_generic_to_shared(k1_raw) & 127)) & 127));
  const int64_t M = g.M, K = g.K, nA = g.nA, kw = g.kw, nreg = g.nreg;
  K1Cursor cur{&g, &z, (int64_t)blockIdx.x, 0, 0, 0, nullptr, 0, 0};
  if (threadIdx.x == 0) {
    for (int s = 0; s < ST; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(&r.full[s])),
                   "r"(1u)
                   : "memory");
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(&r.empty[s])),
                   "r"((uint32_t)(kK1Threads / 32))
                   : "memory");
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x >= kK1Threads) {
    // TMA producer warp: refill a stage as soon as the 8 compute warps have read it
    if (threadIdx.x == kK1Threads) {
      cur.next_tile();
      uint32_t J = 0;
      for (; !cur.done(); ++J) {
        const int s = J % ST;
        k1_wait(&r.empty[s], ((J / ST) & 1u) ^ 1u);
        cur.issue(r, s);
      }
      const int s = J % ST;
      k1_wait(&r.empty[s], ((J / ST) & 1u) ^ 1u);
      cur.finish(r, s);
    }
  } else {
    K1RingLoaderT<ST> ld{r, cur, 0u};
    for (;;) {
      const int64_t t = ld.peek();
      if (t < 0) break;
      if (t < nA)
        k1_a_tile_b(ld, M, K, g.abits, kw, z, t % g.a_tx, t / g.a_tx);
      else
        k1_b_tile_b(ld, K, g.ldb, nreg, g.bgrp, kw, z, (t - nA) % g.b_tx, (t - nA) / g.b_tx);
    }
  }
  __syncthreads();
  // every CTA's tiles are done: the finalize kernel (k1_fin) may be scheduled; it waits in
  // griddepcontrol.wait for this grid to complete
  tc::pdl_trigger();
#ifdef K1_PROF
  if (threadIdx.x == 0 && k1_prof) {
    k1_prof[4 * blockIdx.x] = t_start;
    k1_prof[4 * blockIdx.x + 1] = k1_now();
  }
#endif
}

// The finalize of a K1 pass: one CTA of 1024 threads launched with programmatic
// serialization right after k1_pass (a separate kernel: folded into the pass's last CTA it
// cost the pass's tile loops register spills).  s_tcnt: dynamic shared memory (k1_fin_smem).
struct K1FinArgs {
  int64_t M, K, nreg, kw, nA, nB;
  int has_a, has_b;
};
__global__ void __launch_bounds__(32 * kFinWarps) k1_fin(const __grid_constant__ K1Scratch z, K1FinArgs f,
                                                   unsigned long long* __restrict__ stats) {
  extern __shared__ __align__(16) uint32_t fin_smem[];
  tc::pdl_trigger();  // the pack / CSR CTAs may become resident now (they wait for this grid)
  tc::pdl_wait();     // the K1 pass is complete and its writes are visible
  K1_FIN_STAMP(0);
  if (threadIdx.x == 0) {
    *z.next_tile = 0u;    // ready for the next pass
    z.next_tile[1] = 0u;  // the item counter of the k1_pack_auto launch behind this kernel
  }
  k1_finalize(z, f.M, f.K, f.nreg, f.kw, f.has_a, f.has_b, f.nA, f.nB, stats, fin_smem);
}

// --------------------------------------------------------------- CSR index lists
// Per-row ascending index lists (CSR: row_ptr int64 [M+1] + columns) from K1's bitmap, no
// second pass over A: warp ballot words -> popc -> warp prefix sums -> positions.  A CTA owns
// kCsrRows = 8 rows, warp w row r0 + w, walked in 1024-column chunks with a running offset
// (so no word is read twice).  row_ptr comes from the 32-row tile prefix the K1 pass's last
// CTA scanned plus at most 31 row counts.  Each lane expands its word's set bits into the
// warp's shared staging run (lane order = ascending column), then the chunk's list is copied
// out coalesced.  In AUTO these items ride in the pack launch (k1_pack_auto), next to the
// memory-bound pack items, instead of a launch of their own.
// Index type: uint16 when K <= 65536, else uint32.
constexpr int kCsrRows = 8;

struct CsrArgs {
  const uint32_t* abits;
  const uint32_t* arow;
  const int64_t* tile_prefix;
  int64_t M, kw;
  int64_t* row_ptr;
  void* cols;       // uint16_t or uint32_t
  int idx_bytes;    // 2 or 4
};

// stage: dynamic shared memory of (blockDim / 32) x 1024 indices (k1_csr_smem); 256 threads
__device__ __forceinline__ void k1_csr_cta(const CsrArgs& g, int64_t cta, void* stage) {
  __shared__ int64_t s_off[kCsrRows + 1];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t r0 = cta * kCsrRows, M = g.M, kw = g.kw;
  if (warp == 0) {
    const int64_t t0 = (r0 / 32) * 32;  // first row of r0's 32-row tile
    // counts of rows [t0, r0) (lanes 0..r0-t0-1) and of this CTA's rows (lanes 0..kCsrRows-1)
    const int64_t i_pre = t0 + lane;
    uint32_t pre = (i_pre < r0) ? g.arow[i_pre] : 0u;
#pragma unroll
    for (int o = 16; o; o >>= 1) pre += __shfl_xor_sync(0xffffffffu, pre, o);
    const int64_t i_own = r0 + lane;
    const uint32_t own = (lane < kCsrRows && i_own < M) ? g.arow[i_own] : 0u;
    uint32_t x = own;
#pragma unroll
    for (int o = 1; o < kCsrRows; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    const int64_t base = g.tile_prefix[r0 / 32] + (int64_t)pre;
    if (lane < kCsrRows) s_off[lane] = base + (int64_t)(x - own);
    if (lane == kCsrRows - 1) s_off[kCsrRows] = base + (int64_t)x;
  }
  __syncthreads();
  if (threadIdx.x < kCsrRows && r0 + threadIdx.x < M) g.row_ptr[r0 + threadIdx.x] = s_off[threadIdx.x];
  if (threadIdx.x == 0 && r0 + kCsrRows >= M) g.row_ptr[M] = s_off[M - r0];
  const int64_t row = r0 + warp;
  if (warp < kCsrRows && row < M) {
    const uint32_t* bits = g.abits + row * kw;
    int64_t out = s_off[warp];
    uint32_t nxt = lane < kw ? bits[lane] : 0u;  // the next chunk's word, loaded one chunk ahead
    for (int64_t c0 = 0; c0 < kw; c0 += 32) {
      const int64_t w = c0 + lane;
      uint32_t word = nxt;
      nxt = w + 32 < kw ? bits[w + 32] : 0u;
      const uint32_t n = __popc(word);
      uint32_t x = n;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      // expand the set bits into this warp's shared staging run, then one coalesced copy of
      // the chunk's list (scattered 2-byte global stores cost the L2 ~20x their bytes)
      const uint32_t col0 = (uint32_t)(w * 32), total = __shfl_sync(0xffffffffu, x, 31);
      uint32_t pos = x - n;
      if (g.idx_bytes == 2) {
        uint16_t* buf = reinterpret_cast<uint16_t*>(stage) + warp * 1024;
        for (; word; word &= word - 1u) buf[pos++] = (uint16_t)(col0 + (uint32_t)__ffs(word) - 1u);
        __syncwarp();
        uint16_t* dst = static_cast<uint16_t*>(g.cols) + out;
        // 16-byte stores of 8 indices once dst is 16-byte aligned (2-byte stores left the L2
        // with partial-sector writes)
        const uint32_t head = min(total, (uint32_t)((8u - (uint32_t)((out) & 7)) & 7u));
        if (lane < head) dst[lane] = buf[lane];
        for (uint32_t i = head + 8 * lane; i + 8 <= total; i += 256) {
          uint32_t w[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) w[q] = (uint32_t)buf[i + 2 * q] | ((uint32_t)buf[i + 2 * q + 1] << 16);
          *reinterpret_cast<uint4*>(dst + i) = make_uint4(w[0], w[1], w[2], w[3]);
        }
        const uint32_t tail0 = head + ((total - head) & ~7u);
        if (tail0 + lane < total && total > head) dst[tail0 + lane] = buf[tail0 + lane];
      } else {
        uint32_t* buf = reinterpret_cast<uint32_t*>(stage) + warp * 1024;
        for (; word; word &= word - 1u) buf[pos++] = col0 + (uint32_t)__ffs(word) - 1u;
        __syncwarp();
        uint32_t* dst = static_cast<uint32_t*>(g.cols) + out;
        for (uint32_t i = lane; i < total; i += 32) dst[i] = buf[i];
      }
      out += total;
      __syncwarp();  // the staging run is reused by the next chunk
    }
  }
  __syncthreads();  // s_off is reused by this CTA's next item (k1_pack_auto)
}

// Standalone launch (forced K2 variants, A-only preprocessing).
__host__ __device__ constexpr int k1_csr_smem(int idx_bytes) { return 8 * 1024 * idx_bytes; }

__global__ void __launch_bounds__(256) k1_csr(CsrArgs g) {
  extern __shared__ __align__(16) uint8_t csr_stage[];
  tc::pdl_wait();  // launched with programmatic serialization after k1_pass
  k1_csr_cta(g, blockIdx.x, csr_stage);
}

// ---------------------------------------------------------------- counters + stats
// Exact WorkCounters of the coming multiply:
//   lane_fma_ops  = Σ_k acol[k] * 8 * bpop[k]
//   invocations   = Σ_k acol[k] * bnz[k]
//   zero regions  = Σ_k acol[k] * (nreg - bnz[k])
//   rows_skipped  = M*K - Σ_k acol[k]
// out[0..4] = {inv, lanes, skipped, zreg, nnzA}.  Only a caller that asks for the counters
// pays for this pass (mmmcu_get_counters / multiply with counters): it is not needed to
// multiply.  The plan totals out[5] = Σ bpop (pop_total), out[6] = Σ (nreg - bnz)
// (zero codes) and the path choice out[7] / span out[8] come from K1's last CTA
// (k1_finalize) out of per-warp atomics of the B tiles.
// bpop[k] (# non-zero 8-column groups of row k), bnz[k] (# non-zero 64-column regions) and
// acol[k] (# non-zeros of A's column k; the K1 pass no longer accumulates them) are column
// counts of the group k-masks / of A's bitmap:
// Column counts of a row-major bit matrix bits[R][W] (bit b of word w <-> column 32w + b):
// out[c] += # rows with bit c set; with ORN = 8 the rows are OR-ed in aligned groups of 8 first
// (out[c] += # groups with bit c set in any of their rows).  Serves acol (A's bitmap, rows = A
// rows), bpop (B's group k-masks, rows = 8-column groups) and bnz (the same masks OR-ed per
// 64-column region).  CTA = 32 word columns x 256 rows: lane = word column (coalesced 128-byte
// row segments), warp w rows 32w .. 32w+31; 32 per-bit counters per thread, summed over the
// CTA's warps in shared memory, then one global atomic per column (out is zeroed by the
// caller).  (One thread per column walking all rows, 32 lanes on the same word, took ~0.5 ms
// per 4096^2 operand: WorkCounters on every multiply tripled the sweep step.)
constexpr int kBcRows = 256;
template <int ORN>
__global__ void __launch_bounds__(256) k1_bitcols(const uint32_t* __restrict__ bits, int64_t R, int64_t W, int64_t ncols,
                                                  uint32_t* __restrict__ out) {
  __shared__ uint32_t acc[32][33];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 32 * 33; i += 256) (&acc[0][0])[i] = 0u;
  __syncthreads();
  const int64_t wc = (int64_t)blockIdx.x * 32 + lane;
  const int64_t r0 = (int64_t)blockIdx.y * kBcRows + warp * 32;
  uint32_t cnt[32];
#pragma unroll
  for (int b = 0; b < 32; ++b) cnt[b] = 0u;
  if (wc < W) {
#pragma unroll 1
    for (int g = 0; g < 32 / ORN; ++g) {
      uint32_t word = 0u;
#pragma unroll
      for (int q = 0; q < ORN; ++q) {
        const int64_t r = r0 + g * ORN + q;
        if (r < R) word |= __ldg(bits + r * W + wc);
      }
#pragma unroll
      for (int b = 0; b < 32; ++b) cnt[b] += (word >> b) & 1u;
    }
#pragma unroll
    for (int b = 0; b < 32; ++b)
      if (cnt[b]) atomicAdd(&acc[lane][b], cnt[b]);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 32 * 32; i += 256) {
    const int l = i >> 5, b = i & 31;
    const int64_t c = ((int64_t)blockIdx.x * 32 + l) * 32 + b;
    const uint32_t v = acc[l][b];
    if (v && c < ncols) atomicAdd(out + c, v);
  }
}

__global__ void __launch_bounds__(1024) k1_counters(const uint32_t* __restrict__ acol, const uint32_t* __restrict__ bpop,
                                                    const uint32_t* __restrict__ bnz, int64_t K, int64_t M, int64_t nreg,
                                                    int has_a, int has_b, unsigned long long* __restrict__ out) {
  unsigned long long s[4] = {0, 0, 0, 0};
#pragma unroll 4
  for (int64_t k = threadIdx.x; k < K; k += blockDim.x) {
    const unsigned long long a = has_a ? acol[k] : 0ull;
    const unsigned long long p = has_b ? bpop[k] : 0ull;
    const unsigned long long n = has_b ? bnz[k] : 0ull;
    const unsigned long long z = has_b ? (unsigned long long)nreg - n : 0ull;
    s[0] += a * n;
    s[1] += a * 8ull * p;
    s[2] += a * z;
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
#ifndef K1_PT_STEPS
#define K1_PT_STEPS 8
#endif
constexpr int kPtSteps = K1_PT_STEPS;  // step images per K2-TC pack CTA
constexpr int kPtThreads = 256;

struct PackTcArgs {
  const float* B;
  int64_t ldb;
  const uint32_t* tlive;
  int64_t kw, maxsteps;
  float* tcb;
  int32_t* tck;
  int32_t* tcn;
  int f16;                            // fp16 split: 16 live k per step, B group g scaled by 2^sB[g]
  const unsigned long long* grng;     // per 8-column group: max|B| bits << 32 | ... (K1 pass), fp16 only
};

// Steps [s_lo, s_hi) of tile tb of the K2-TC pack (s_hi is clipped to the tile's step count;
// s_hi < 0: the fixed step block s_lo .. s_lo + kPtSteps); dynamic smem (2 kw + 1) words.
__device__ __forceinline__ void k1_pack_tc_range(const PackTcArgs& g, int64_t tb, int64_t s_lo, int64_t s_hi) {
  const float* __restrict__ B = g.B;
  const int64_t ldb = g.ldb, kw = g.kw, maxsteps = g.maxsteps;
  const uint32_t* __restrict__ tlive = g.tlive;
  float* __restrict__ tcb = g.tcb;
  int32_t* __restrict__ tck = g.tck;
  int32_t* __restrict__ tcn = g.tcn;
  extern __shared__ __align__(16) uint32_t pt_smem[];  // masks [kw] | prefix [kw + 1]
  __shared__ int32_t s_k[kPtSteps * 16];
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
  const int SK = g.f16 ? 16 : 8;  // live k per step
  const int64_t nsteps_all = (total + SK - 1) / SK;
  if (s_lo == 0 && tid == 0) tcn[tb] = total;
  const int64_t nsteps = s_hi < 0 ? min(nsteps_all, s_lo + kPtSteps) : min(nsteps_all, s_hi);  // end of this range
  for (int64_t s0 = s_lo; s0 < nsteps; s0 += kPtSteps) {
  __syncthreads();  // s_k of the previous block is no longer read
  if (tid < kPtSteps * SK && s0 * SK + tid < nsteps * SK) {
    const int64_t p = s0 * SK + tid;
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
  if (g.f16) {
    // job = (step, k-octet q, 4-column group c4 of the 48 in the tile): 8 rows x 4 columns of B
    // by 8 independent 16-byte loads (a warp reads 512 contiguous bytes per row), scaled by the
    // columns' 8-column group's 2^sB, split into fp16 hi / lo: 4 columns x 8 k = one 16-byte
    // hi and one 16-byte lo store per column.  K2-TC runs fp16 tiles on CTA pairs, each CTA
    // holding one column half h (96 columns) of B: a tile's images are stored per half,
    // [h][step], a half step = hi image (3 KB) | lo image (3 KB), element (c, j) of column
    // c = n - 96h at byte (c % 8) * 16 + (c / 8) * 256 + (j / 8) * 128 + (j % 8) * 2 of its image
    constexpr int kC4 = kTcTileN / 4, kHalf = kTcTileN / 2;
    constexpr int kJobs = kPtSteps * 2 * kC4, kPer = (kJobs + kPtThreads - 1) / kPtThreads;
    // per job 8 independent 16-byte loads in flight (4 CTAs per SM: ~128 KB per SM)
#pragma unroll 1
    for (int u = 0; u < kPer; ++u) {
      const int j = tid + u * kPtThreads;
      const int sl = j / (2 * kC4), q = (j / kC4) & 1, n = 4 * (j % kC4);
      const int64_t s = s0 + sl;
      if (j >= kJobs || s >= nsteps) break;
      float4 v[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int32_t k = n0 + n < ldb ? s_k[sl * 16 + 8 * q + i] : -1;
        v[i] = k >= 0 ? ldg_stream(B + (int64_t)k * ldb + n0 + n) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
      const bool col_ok = n0 + n < ldb;
      const float sb = col_ok ? tc::exp2_int(tc::f16_scale_exp((uint32_t)(__ldg(g.grng + ((n0 + n) >> 3)) >> 32))) : 1.0f;
      const int hf = n / kHalf, c = n % kHalf;
      float* img = tcb + ((tb * 2 + hf) * maxsteps + s) * (kHalf * 16);
      const int off = (c & 7) * 4 + (c >> 3) * 64 + q * 32;  // in floats; columns c .. c+3 follow at +4
      uint32_t h[4][4], l[4][4];
#pragma unroll
      for (int cc = 0; cc < 4; ++cc) {
        float x[8];
#pragma unroll
        for (int i = 0; i < 8; ++i)
          x[i] = (cc == 0 ? v[i].x : cc == 1 ? v[i].y : cc == 2 ? v[i].z : v[i].w) * sb;
#pragma unroll
        for (int i = 0; i < 4; ++i) tc::split_f16x2(x[2 * i], x[2 * i + 1], h[cc][i], l[cc][i]);
      }
      // columns c, c+1 (and c+2, c+3) are adjacent 16-byte chunks: two 32-byte stores per image
#pragma unroll
      for (int pr = 0; pr < 2; ++pr) {
        asm volatile("st.global.v8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(img + off + 8 * pr),
                     "r"(h[2 * pr][0]), "r"(h[2 * pr][1]), "r"(h[2 * pr][2]), "r"(h[2 * pr][3]),
                     "r"(h[2 * pr + 1][0]), "r"(h[2 * pr + 1][1]), "r"(h[2 * pr + 1][2]), "r"(h[2 * pr + 1][3])
                     : "memory");
        asm volatile("st.global.v8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(img + kHalf * 8 + off + 8 * pr),
                     "r"(l[2 * pr][0]), "r"(l[2 * pr][1]), "r"(l[2 * pr][2]), "r"(l[2 * pr][3]),
                     "r"(l[2 * pr + 1][0]), "r"(l[2 * pr + 1][1]), "r"(l[2 * pr + 1][2]), "r"(l[2 * pr + 1][3])
                     : "memory");
      }
    }
    continue;
  }
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
    for (int i = 0; i < 4; ++i) {  // tc::split_tf32
      h[i] = __float_as_uint(v[i]) & 0xFFFFE000u;
      l[i] = __float_as_uint(v[i] - __uint_as_float(h[i]));
    }
    float* img = tcb + (tb * maxsteps + s) * (kTcTileN * 16);
    const int off = (n & 7) * 4 + (n >> 3) * 64 + q * 32;  // in floats
    *reinterpret_cast<uint4*>(img + off) = make_uint4(h[0], h[1], h[2], h[3]);
    *reinterpret_cast<uint4*>(img + kTcTileN * 8 + off) = make_uint4(l[0], l[1], l[2], l[3]);
  }
  }  // step blocks of the range
}

// CTA (bx = step block, tb = tile) of the K2-TC pack
__device__ __forceinline__ void k1_pack_tc_cta(const PackTcArgs& g, int64_t bx, int64_t tb) {
  k1_pack_tc_range(g, tb, bx * kPtSteps, -1);
}

__global__ void __launch_bounds__(kPtThreads, 4) k1_pack_tc(PackTcArgs g) { k1_pack_tc_cta(g, blockIdx.x, blockIdx.y); }

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

// AUTO: the K2-TC step images, the K2-SIMT record rows (only the one K1's last CTA chose) and
// A's CSR index lists in ONE persistent launch: each CTA walks the work items w = blockIdx.x,
// + gridDim.x, ... of [chosen pack items | CSR items], so the gated-out pack costs nothing
// (one CTA per item made ~5.5 k CTAs per 4096^2 cell, most of them exiting at entry).
__global__ void __launch_bounds__(kPtThreads, 4)
k1_pack_auto(PackRowsArgs gr, int64_t rows_x, int64_t n_rows, PackTcArgs gt, int64_t tc_x, int64_t n_tcb,
             const unsigned long long* __restrict__ sel, CsrArgs gc, int64_t n_csr,
             const int64_t* __restrict__ tc_pre, int64_t n_tiles, unsigned int* __restrict__ item_ctr) {
  tc::pdl_wait();  // launched with programmatic serialization after k1_pass
  extern __shared__ __align__(16) uint32_t pt_smem[];  // TC pack scan words / CSR staging
  const unsigned long long v = *sel;  // 8 / 16 K2-SIMT (rows), 32 K2-TC (step images), 48 K2-CSR (neither)
  int64_t n_pack = v == 32ull ? n_tcb : (v == 8ull || v == 16ull) ? n_rows : 0;
  // K2-TC with the tiles' step prefix from k1_fin: the concatenated steps of all tiles are cut
  // into gridDim.x equal shares (fixed blocks of kPtSteps steps left the CTAs holding two
  // blocks as the critical path: 704 blocks on 592 CTAs for a dense 4096^2 B, and every block
  // of a sparse-k tile past its live steps still paid the prefix scan)
  const int64_t s_all = (v == 32ull && tc_pre) ? tc_pre[n_tiles] : -1;
  const int64_t n_shares = s_all >= 0 ? (int64_t)gridDim.x : 0;
  if (s_all >= 0) n_pack = 0;
  // Items are taken from an atomic counter (reset by k1_fin), not dealt by CTA index: when this
  // launch shares the GPU with another stream's K2-TC only some of its CTAs are resident, and
  // they walk the whole list.  Items: [step shares | fixed pack blocks | CSR row groups].
  __shared__ unsigned int s_item;
#ifdef K1_PACK_STATIC
  unsigned int s_round = 0;
#endif
  for (;;) {
#ifdef K1_PACK_STATIC  // (timing variant: items dealt by CTA index)
    if (threadIdx.x == 0) s_item = s_round++ * gridDim.x + blockIdx.x;
#else
    if (threadIdx.x == 0) s_item = atomicAdd(item_ctr, 1u);
#endif
    __syncthreads();
    const int64_t w = (int64_t)s_item;
    __syncthreads();
    if (w >= n_shares + n_pack + n_csr) break;
    if (w < n_shares) {
      const int64_t lo = s_all * w / n_shares, hi = s_all * (w + 1) / n_shares;
      if (lo < hi) {
        int64_t a = 0, b = n_tiles - 1;  // last tile tb with tc_pre[tb] <= lo
        while (a < b) {
          const int64_t mid = (a + b + 1) >> 1;
          if (tc_pre[mid] <= lo) a = mid;
          else b = mid - 1;
        }
        for (int64_t tb = a; tb < n_tiles && tc_pre[tb] < hi; ++tb) {
          const int64_t t0 = tc_pre[tb], t1 = tc_pre[tb + 1];
          const int64_t b0 = (lo > t0 ? lo : t0) - t0, b1 = (hi < t1 ? hi : t1) - t0;
          if (b0 < b1) {
            k1_pack_tc_range(gt, tb, b0, b1);
            __syncthreads();  // shared memory is reused by the next piece
          }
        }
      }
    } else if (w < n_shares + n_pack) {
      const int64_t x = w - n_shares;
      if (v == 32ull) k1_pack_tc_cta(gt, x % tc_x, x / tc_x);
      else k1_pack_rows_cta(gr, x % rows_x, x / rows_x);
    } else {
      k1_csr_cta(gc, w - n_shares - n_pack, pt_smem);
    }
    __syncthreads();  // shared memory is reused by the next item
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
