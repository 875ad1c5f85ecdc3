// K2-SIMT — masked fp32 GEMM on the CUDA cores (sm_100a), exact ascending-k fmaf chains.
//
// Replaces SPEC multiply_mmm / multiply_parallel (PAPER Fig. 10,
// PAPER.md:426-436).  The paper's runtime code lookup — one indirect call per
// (non-zero a_ik, 64-wide region), dispatching a straight-line routine that FMAs only the
// non-zero 8-wide groups (kernel_table.cpp:12-28) — becomes mask intersection here:
//
//   CTA   = 128 rows x 256 columns of C; 16 warps; one 16-column slice per warp.
//   lane  = 4 rows (4l .. 4l+3 of the tile) x 16 columns: 64 fp32 accumulators that start
//           from C (c += a*b semantics) and end in C.
//   k     = walked in chunks of 64.  For every chunk each warp reads the B block masks of
//           its slice (K1's transposed group bitmaps) and iterates ONLY the k whose B block
//           is non-zero (warp-uniform loop: no divergence, the B-side skip of Fig. 10's
//           `fps[code]`).  A's element mask is applied per lane by predication (the A-side
//           skip of Fig. 4): a lane whose a_ik == 0 issues no FMA for that row.
//   smem  = double-buffered A^T chunk [64 k][128 rows] (swizzled, 32 KB) + B chunk
//           [64 k][256 cols] (64 KB) of which only non-zero 8/16-column blocks are fetched
//           (cp.async, 16 B granules).  B values reach the FMAs as warp broadcasts.
//
// Every C element receives fmaf(a_ik, b_kj, c) for its surviving k in ascending order,
// exactly the oracle's chain (orc_multiply_mmm), so results are bit-identical.  This v1
// kernel is only launched with SPAN=8 (each group walks its own mask); the TMA-fed v2 below
// is the normal exact path.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace mmmcu {

constexpr int kK2Threads = 512;
constexpr int kK2TM = 128;  // rows per CTA
constexpr int kK2TN = 256;  // columns per CTA (16 warps x 16)
constexpr int kK2KC = 64;   // k per chunk
constexpr int kK2SmemA = kK2KC * kK2TM * 4;
constexpr int kK2SmemB = kK2KC * kK2TN * 4;
constexpr int kK2Smem = 2 * (kK2SmemA + kK2SmemB);  // 192 KB

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const uint32_t s = (uint32_t)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// A^T chunk index: 4-row groups XOR-swizzled by (k/4)%8 so that the transposing stores
// are at most 2-way bank conflicted and each lane's 4-row LDS.128 stays contiguous.
__device__ __forceinline__ int at_index(int k, int row) { return k * kK2TM + (row ^ (((k >> 2) & 7) << 2)); }

// 64-bit k-mask of a 16-column slice for chunk words (w0, w0+1) from the group bitmaps.
__device__ __forceinline__ uint64_t slice_mask(const uint32_t* __restrict__ bgrp, int64_t kw, int64_t g0,
                                               int64_t w0, int groups) {
  uint64_t m = 0;
  for (int g = 0; g < groups; ++g) {
    const uint32_t* p = bgrp + (g0 + g) * kw;
    const uint32_t lo = w0 < kw ? p[w0] : 0u;
    const uint32_t hi = w0 + 1 < kw ? p[w0 + 1] : 0u;
    m |= (uint64_t)lo | ((uint64_t)hi << 32);
  }
  return m;
}

// SPAN = width (columns) of the block mask a warp iterates: 16 (one mask for the slice,
// the natural choice for B block widths >= 16) or 8 (two masks, one per 8-wide group:
// exact group-level skipping for 8-wide blocks).
template <int SPAN>
__global__ void __launch_bounds__(kK2Threads, 1)
k2_simt_bcast(const float* __restrict__ A, int64_t lda, const float* __restrict__ B, int64_t ldb,
              float* __restrict__ C, int64_t ldc, int64_t M, int64_t K, int64_t Np,
              const uint32_t* __restrict__ bgrp, int64_t kw, const unsigned long long* __restrict__ sel) {
  static_assert(SPAN == 8 || SPAN == 16, "SPAN must be 8 or 16");
  if (sel && *sel != (unsigned long long)SPAN) return;  // device-side variant choice (k1_finalize)
  constexpr int NS = 16 / SPAN;  // spans per warp
  extern __shared__ __align__(16) float smem[];
  // stage st: A^T at smem + st*KC*TM, B at smem + 2*KC*TM + st*KC*TN (no pointer arrays:
  // dynamically indexed local arrays would live in local memory)
  auto sA = [&](int st) { return smem + st * (kK2KC * kK2TM); };
  auto sB = [&](int st) { return smem + 2 * kK2KC * kK2TM + st * (kK2KC * kK2TN); };

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t m0 = (int64_t)blockIdx.y * kK2TM;
  const int64_t n0 = (int64_t)blockIdx.x * kK2TN;
  const int64_t ncol = n0 + 16 * warp;           // this warp's 16-column slice
  const bool slice_ok = ncol < Np;               // Np is a multiple of 64
  const int64_t g0 = ncol >> 3;                  // first 8-column group of the slice

  // ---- accumulators start from C (c += a*b)
  float2 acc[NS][4][SPAN / 2];
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const int64_t row = m0 + 4 * lane + r;
#pragma unroll
    for (int s = 0; s < NS; ++s)
#pragma unroll
      for (int j = 0; j < SPAN / 2; ++j) {
        float2 v = make_float2(0.f, 0.f);
        if (slice_ok && row < M) v = *reinterpret_cast<const float2*>(C + row * ldc + ncol + s * SPAN + 2 * j);
        acc[s][r][j] = v;
      }
  }

  const int64_t nchunks = (K + kK2KC - 1) / kK2KC;

  // ---- staging helpers
  // A: 128 rows x 64 k = 2048 float4; thread t loads f = t + 512 j: row f/16, kq f%16.
  float4 areg[4];
  auto load_a = [&](int64_t c) {
    const int64_t k0 = c * kK2KC;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int f = tid + kK2Threads * j;
      const int row = f >> 4, kq = f & 15;
      const int64_t gr = m0 + row, gk = k0 + 4 * kq;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (gr < M && gk < K) {
        v = __ldg(reinterpret_cast<const float4*>(A + gr * lda + gk));
        // K need not be a multiple of 4: zero the columns past K (reads stay inside lda)
        if (gk + 4 > K) {
          if (gk + 1 >= K) v.y = 0.f;
          if (gk + 2 >= K) v.z = 0.f;
          if (gk + 3 >= K) v.w = 0.f;
        }
      }
      areg[j] = v;
    }
  };
  auto store_a = [&](float* dst) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int f = tid + kK2Threads * j;
      const int row = f >> 4, kq = f & 15;
      dst[at_index(4 * kq + 0, row)] = areg[j].x;
      dst[at_index(4 * kq + 1, row)] = areg[j].y;
      dst[at_index(4 * kq + 2, row)] = areg[j].z;
      dst[at_index(4 * kq + 3, row)] = areg[j].w;
    }
  };
  // B: only the non-zero (k, slice) rows of this warp's slice: 4 lanes x 16 B per k row.
  auto load_b = [&](int64_t c, float* dst, uint64_t mask) {
    if (!slice_ok) return;
    const int64_t k0 = c * kK2KC;
    const int grp = lane >> 2, piece = lane & 3;
    uint64_t m = mask;
    while (m) {  // warp-uniform: 8 k rows per pass, 4 lanes (4 x 16 B) per row
      uint64_t t = m;
      for (int i = 0; i < grp; ++i) t &= t - 1;  // drop this group's predecessors
      if (t) {
        const int kk = __ffsll((long long)t) - 1;
        cp_async16(dst + kk * kK2TN + 16 * warp + 4 * piece, B + (k0 + kk) * ldb + ncol + 4 * piece);
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) m &= m - 1;  // (m & (m-1)) of 0 stays 0
    }
  };

  // Slice masks are loaded two chunks ahead (registers) so that the B fetch of chunk c+1,
  // issued at the top of iteration c, never waits on a fresh global load.
  uint64_t mask_cur[NS], mask_nxt[NS], mask_nn[NS];
  auto masks_for = [&](int64_t c, uint64_t* out) {
#pragma unroll
    for (int s = 0; s < NS; ++s)
      out[s] = (slice_ok && c < nchunks) ? slice_mask(bgrp, kw, g0 + s * (SPAN / 8), 2 * c, SPAN / 8) : 0ull;
  };
  auto bmask = [&](const uint64_t* m) { return NS == 1 ? m[0] : (m[0] | m[NS - 1]); };

  // ---- prologue: chunk 0 staged, chunk 1 masks in flight
  masks_for(0, mask_cur);
  masks_for(1, mask_nxt);
  load_a(0);
  store_a(sA(0));
  load_b(0, sB(0), bmask(mask_cur));
  cp_async_commit();
  cp_async_wait_all();
  __syncthreads();

  for (int64_t c = 0; c < nchunks; ++c) {
    const int st = (int)(c & 1);
    const bool more = c + 1 < nchunks;
    if (more) {
      load_a(c + 1);
      load_b(c + 1, sB(st ^ 1), bmask(mask_nxt));
      cp_async_commit();
    }
    masks_for(c + 2, mask_nn);
    // ---- compute chunk c: warp-uniform walk over the slice's non-zero B rows
    const float* at = sA(st);
    const float* bs = sB(st) + 16 * warp;
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      uint64_t m = mask_cur[s];
      while (m) {
        const int kk = __ffsll((long long)m) - 1;
        m &= m - 1;
        const float4 av = *reinterpret_cast<const float4*>(at + at_index(kk, 4 * lane));
        float2 b[SPAN / 2];
#pragma unroll
        for (int q = 0; q < SPAN / 4; ++q) {
          const float4 bv = *reinterpret_cast<const float4*>(bs + kk * kK2TN + s * SPAN + 4 * q);
          b[2 * q] = make_float2(bv.x, bv.y);
          b[2 * q + 1] = make_float2(bv.z, bv.w);
        }
        const float a4[4] = {av.x, av.y, av.z, av.w};
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          if (a4[r] != 0.0f) {
            const float2 a2 = make_float2(a4[r], a4[r]);
#pragma unroll
            for (int j = 0; j < SPAN / 2; ++j) acc[s][r][j] = __ffma2_rn(a2, b[j], acc[s][r][j]);
          }
        }
      }
    }
    if (more) store_a(sA(st ^ 1));
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      mask_cur[s] = mask_nxt[s];
      mask_nxt[s] = mask_nn[s];
    }
    cp_async_wait_all();
    __syncthreads();
  }

  // ---- epilogue: write the accumulators back
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const int64_t row = m0 + 4 * lane + r;
    if (!slice_ok || row >= M) continue;
#pragma unroll
    for (int s = 0; s < NS; ++s)
#pragma unroll
      for (int j = 0; j < SPAN / 2; ++j)
        *reinterpret_cast<float2*>(C + row * ldc + ncol + s * SPAN + 2 * j) = acc[s][r][j];
  }
}

// ------------------------------------------------------------------------------------
// multiply_simple (PAPER Fig. 2): dense C += A*B, ascending-k fmaf per
// element (bit-identical to orc_multiply_simple).  64x64 tiles, 256 threads, 4x4 per thread.
__global__ void __launch_bounds__(256)
k2_dense(const float* __restrict__ A, int64_t lda, const float* __restrict__ B, int64_t ldb, float* __restrict__ C,
         int64_t ldc, int64_t M, int64_t K, int64_t N) {
  __shared__ float sa[16][64 + 4];
  __shared__ float sb[16][64];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int64_t m0 = (int64_t)blockIdx.y * 64, n0 = (int64_t)blockIdx.x * 64;
  float acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t r = m0 + ty * 4 + i, cc = n0 + tx * 4 + j;
      acc[i][j] = (r < M && cc < N) ? C[r * ldc + cc] : 0.f;
    }
  for (int64_t k0 = 0; k0 < K; k0 += 16) {
    for (int t = threadIdx.x; t < 16 * 64; t += 256) {
      const int kk = t & 15, rr = t >> 4;
      const int64_t gr = m0 + rr, gk = k0 + kk;
      sa[kk][rr] = (gr < M && gk < K) ? A[gr * lda + gk] : 0.f;
      const int cc = t & 63, kb = t >> 6;
      const int64_t gkb = k0 + kb, gc = n0 + cc;
      sb[kb][cc] = (gkb < K && gc < N) ? B[gkb * ldb + gc] : 0.f;
    }
    __syncthreads();
    const int kmax = (int)(K - k0 < 16 ? K - k0 : 16);
    for (int kk = 0; kk < kmax; ++kk) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = sa[kk][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = sb[kk][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t r = m0 + ty * 4 + i, cc = n0 + tx * 4 + j;
      if (r < M && cc < N) C[r * ldc + cc] = acc[i][j];
    }
}


// ====================================================================================
// K2-SIMT v2 — the same exact computation, fed by bulk async copies of K1's MMA-ready
// operands (A^T per 128-row tile, raw non-zero B block rows per (256-column tile, chunk)).
//
//   CTA   = 128 rows x 256 columns of C, 16 compute warps (one 16-column slice each).  A 17th
//           producer warp would put 5 warps on one SMSP and cap registers at 96, which
//           serialises the B loads; instead the LAST warp to finish a chunk refills its
//           stage (shared counter, acq_rel).  4 smem stages of {A^T chunk [32 k][128 rows],
//           B record: 3 header rows (32 group k-masks, 16 slice offsets) + the chunk's
//           non-zero slice rows}.
//   lane  = rows 4l .. 4l+3 of the tile x the warp's 16 columns (64 fp32 accumulators,
//           initialised from C).  Per non-zero B row k of its slice the warp issues one
//           conflict-free LDS.128 of the 4 A values, 4 broadcast LDS.128 of B[k][slice] and
//           32 FFMA2 predicated on a != 0 — the ascending-k fmaf chain of the oracle.
//   SPAN  = 16: one walk per slice over the union mask, each group's FMAs predicated on its
//           own code bit; 8: one walk per 8-column group over its own mask.  Both touch set
//           groups only (kernel_table.cpp:17-20), so Inf / NaN in A and -0.0 in C behave as
//           in the reference.
// ====================================================================================
constexpr int kS2Warps = 16;
constexpr int kS2Threads = kS2Warps * 32;  // no producer warp: 4 warps/SMSP keep 128 registers
constexpr int kS2Stages = 4;
constexpr int kS2KC = 32;
constexpr int kS2MaxRows = 3 + 16 * kS2KC;  // header + every (k, slice) of a chunk

struct alignas(128) S2Stage {
  float at[kS2KC][128];          // 16 KB
  float4 rows[kS2MaxRows][4];    // 33 KB: header (3 rows) + B block rows
};
struct S2Shared {
  S2Stage st[kS2Stages];
  uint64_t full[kS2Stages];
  uint32_t pend[kS2Stages];  // warps done with the stage's current chunk
  // followed by the tile's chunk offsets (int64, kw + 1), dynamic
};
constexpr int kS2SmemBase = (int)sizeof(S2Shared) + 128;

__device__ __forceinline__ void s2_bulk(void* smem_dst, const void* gsrc, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   (uint32_t)__cvta_generic_to_shared(smem_dst)),
               "l"(gsrc), "r"(bytes), "r"((uint32_t)__cvta_generic_to_shared(bar))
               : "memory");
}
__device__ __forceinline__ void s2_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void s2_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void s2_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"((uint32_t)__cvta_generic_to_shared(bar)) : "memory");
}
__device__ __forceinline__ void pdl_wait_simt() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void s2_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "S2W_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra S2W_%=;\n\t}" ::"r"((uint32_t)__cvta_generic_to_shared(bar)),
      "r"(parity)
      : "memory");
}

template <int SPAN>
__device__ __forceinline__ void k2_simt2_body(const float* __restrict__ AT, int64_t kpad,
                                              const float4* __restrict__ brows, const int64_t* __restrict__ row_off,
                                              int64_t kw, float* __restrict__ C, int64_t ldc, int64_t M, int64_t Np,
                                              int64_t rt, int64_t tb) {
  static_assert(SPAN == 8 || SPAN == 16, "SPAN must be 8 or 16");
  extern __shared__ __align__(128) uint8_t s2_raw[];
  S2Shared& sh = *reinterpret_cast<S2Shared*>(s2_raw + ((128 - ((uint32_t)__cvta_generic_to_shared(s2_raw) & 127)) & 127));
  int64_t* offs = reinterpret_cast<int64_t*>(&sh + 1);

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t m0 = rt * 128, n0 = tb * 256;

  for (int64_t c = tid; c <= kw; c += kS2Threads) offs[c] = row_off[tb * kw + c];
  if (tid == 0) {
    for (int s = 0; s < kS2Stages; ++s) {
      s2_init(&sh.full[s], 1);
      sh.pend[s] = 0;
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  // chunk x lives in stage x % S: chunks 0..S-1 now, chunk x + S by the last warp done with x
  auto issue = [&](int64_t x) {
    const int s = (int)(x % kS2Stages);
    const uint32_t nrows = (uint32_t)(offs[x + 1] - offs[x]);
    s2_expect_tx(&sh.full[s], 16384u + nrows * 64u);
    s2_bulk(&sh.st[s].at[0][0], AT + (rt * kpad + x * kS2KC) * 128, 16384u, &sh.full[s]);
    s2_bulk(&sh.st[s].rows[0][0], brows + offs[x] * 4, nrows * 64u, &sh.full[s]);
  };
  if (tid == 0)
    for (int64_t x = 0; x < kw && x < kS2Stages; ++x) issue(x);

  // -------------------------------------------------------------------- compute
  const int j = warp;                       // slice
  const int64_t ncol = n0 + 16 * j;
  const bool slice_ok = ncol < Np;
  constexpr int NS = 16 / SPAN;
  float2 acc[NS][4][SPAN / 2];
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const int64_t row = m0 + 4 * lane + r;
#pragma unroll
    for (int s = 0; s < NS; ++s)
#pragma unroll
      for (int q = 0; q < SPAN / 2; ++q)
        acc[s][r][q] = (slice_ok && row < M) ? *reinterpret_cast<const float2*>(C + row * ldc + ncol + s * SPAN + 2 * q)
                                             : make_float2(0.f, 0.f);
  }

  for (int64_t c = 0; c < kw; ++c) {
    const int st = (int)(c % kS2Stages);
    s2_wait(&sh.full[st], (uint32_t)((c / kS2Stages) & 1));
    const S2Stage& S = sh.st[st];
    const uint32_t* hdr = reinterpret_cast<const uint32_t*>(&S.rows[0][0]);
    const uint32_t g0 = hdr[2 * j], g1 = hdr[2 * j + 1];
    const uint32_t um = g0 | g1;
    uint32_t base = hdr[32 + j];  // first record row of this slice (header row 2)
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      uint32_t m = NS == 1 ? um : (s == 0 ? g0 : g1);
      // two non-zero B rows per iteration: both rows' loads are issued before the FMAs
      // (ILP across k); FMAs stay in ascending k, so the per-element fmaf chain is unchanged.
      // SPAN 16 walks the slice's union mask, so each 8-column group is FMA'd only when ITS
      // code bit is set (kernel_table.cpp:17-20 touches set groups only): no fma(a, +0, c)
      // terms, which would turn Inf / NaN a into NaN and -0.0 c into +0.0.
      auto fma_row = [&](const float4& av, const float4 (&bq)[SPAN / 4], bool live0, bool live1) {
        float2 b[SPAN / 2];
#pragma unroll
        for (int q = 0; q < SPAN / 4; ++q) {
          b[2 * q] = make_float2(bq[q].x, bq[q].y);
          b[2 * q + 1] = make_float2(bq[q].z, bq[q].w);
        }
        const float a4[4] = {av.x, av.y, av.z, av.w};
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          const float2 a2 = make_float2(a4[r], a4[r]);
          const bool anz = a4[r] != 0.0f;
#pragma unroll
          for (int q = 0; q < SPAN / 2; ++q) {
            const bool live = q < 4 ? live0 : live1;  // group of columns 2q, 2q+1
            if (anz && live) acc[s][r][q] = __ffma2_rn(a2, b[q], acc[s][r][q]);
          }
        }
      };
      while (m) {
        const int k1 = __ffs(m) - 1;
        m &= m - 1;
        const bool two = m != 0;
        const int k2 = two ? __ffs(m) - 1 : k1;
        if (two) m &= m - 1;
        const uint32_t r1 = base + (NS == 1 ? 0u : (uint32_t)__popc(um & ((1u << k1) - 1u)));
        const uint32_t r2 = NS == 1 ? r1 + (two ? 1u : 0u) : base + (uint32_t)__popc(um & ((1u << k2) - 1u));
        if (NS == 1) base += two ? 2u : 1u;
        const float4 av1 = *reinterpret_cast<const float4*>(&S.at[k1][4 * lane]);
        const float4 av2 = *reinterpret_cast<const float4*>(&S.at[k2][4 * lane]);
        float4 b1[SPAN / 4], b2[SPAN / 4];
#pragma unroll
        for (int q = 0; q < SPAN / 4; ++q) {
          b1[q] = S.rows[r1][s * (SPAN / 4) + q];
          b2[q] = S.rows[r2][s * (SPAN / 4) + q];
        }
        if (NS == 1) {
          fma_row(av1, b1, (g0 >> k1) & 1u, (g1 >> k1) & 1u);
          if (two) fma_row(av2, b2, (g0 >> k2) & 1u, (g1 >> k2) & 1u);
        } else {  // SPAN 8: m is the group's own mask
          fma_row(av1, b1, true, true);
          if (two) fma_row(av2, b2, true, true);
        }
      }
    }
    __syncwarp();
    if (lane == 0) {
      uint32_t old;
      asm volatile("atom.acq_rel.cta.shared::cta.add.u32 %0, [%1], 1;"
                   : "=r"(old)
                   : "r"((uint32_t)__cvta_generic_to_shared(&sh.pend[st]))
                   : "memory");
      if (old == kS2Warps - 1) {  // every warp is done with stage st: refill it
        sh.pend[st] = 0;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        if (c + kS2Stages < kw) issue(c + kS2Stages);
      }
    }
  }

#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const int64_t row = m0 + 4 * lane + r;
    if (!slice_ok || row >= M) continue;
#pragma unroll
    for (int s = 0; s < NS; ++s)
#pragma unroll
      for (int q = 0; q < SPAN / 2; ++q)
        *reinterpret_cast<float2*>(C + row * ldc + ncol + s * SPAN + 2 * q) = acc[s][r][q];
  }
}

template <int SPAN>
__global__ void __launch_bounds__(kS2Threads, 1)
k2_simt2(const float* __restrict__ AT, int64_t kpad, const float4* __restrict__ brows, const int64_t* __restrict__ row_off,
         int64_t kw, float* __restrict__ C, int64_t ldc, int64_t M, int64_t Np, const unsigned long long* __restrict__ sel) {
  if (sel && *sel != (unsigned long long)SPAN) return;  // device-side span choice (k1_finalize_block)
  k2_simt2_body<SPAN>(AT, kpad, brows, row_off, kw, C, ldc, M, Np, blockIdx.y, blockIdx.x);
}

// One launch for both spans (and AUTO): *sel = 8 / 16 runs that span, anything else (32 =
// K2-TC chosen) exits at entry.  Persistent (grid <= one CTA per SM, tiles t = blockIdx.x,
// + gridDim.x, ...): when K2-TC was chosen the gated-out launch costs one wave of exiting
// CTAs instead of four (5 us per call with a tile-per-CTA grid).
__global__ void __launch_bounds__(kS2Threads, 1)
k2_simt2_any(const float* __restrict__ AT, int64_t kpad, const float4* __restrict__ brows,
             const int64_t* __restrict__ row_off, int64_t kw, float* __restrict__ C, int64_t ldc, int64_t M, int64_t Np,
             const unsigned long long* __restrict__ sel, int64_t n_tb, int64_t n_rt) {
  pdl_wait_simt();  // launched with programmatic serialization after the K1 pack
  const unsigned long long v = *sel;
  if (v != 8ull && v != 16ull) return;
  for (int64_t t = blockIdx.x; t < n_tb * n_rt; t += gridDim.x) {
    if (v == 8ull)
      k2_simt2_body<8>(AT, kpad, brows, row_off, kw, C, ldc, M, Np, t / n_tb, t % n_tb);
    else
      k2_simt2_body<16>(AT, kpad, brows, row_off, kw, C, ldc, M, Np, t / n_tb, t % n_tb);
    __syncthreads();  // the next tile re-initialises the stage barriers and offsets
  }
}

}  // namespace mmmcu
