// K2-TC — dense-tile masked GEMM on the 5th-generation tensor cores (tcgen05, kind::tf32,
// 3xTF32 split), for cells whose masks leave the 128 x 192 C tiles dense enough to pay
// (BASELINE north_star: "tensor cores only for tiles that the masks leave dense enough ...
// and only if the result stays inside tolerance").
//
// Work unit: one CTA = one 128-row x 192-column C tile.  The k loop runs only over the
// tile's LIVE k (B[k, tile] has a non-zero, from K1's tlive masks), 8 per MMA step, so B's
// block sparsity removes whole k-steps; A's element zeros are multiplied (the tile is dense
// enough by the choice of this path).  Per step:
//   B: one 24 KB bulk copy of two K1-packed 8-k step images (tf32 hi / lo, UMMA K-major);
//   A: the 4 transform warps load the step's 8 live rows of the K1 A^T tile
//      (at[(rt*kpad + k)*128 + i], coalesced, 2 stages ahead), split them into tf32 hi / lo
//      and store them to TMEM (lane = row, column = k) — per-k TMA copies of 512 B cost
//      more TMA issue slots than the MMAs leave (measured: 0.92 vs 0.62 ms, 4096^3);
//   one thread issues, per 8 k, D += A_lo*B_hi + A_hi*B_lo + A_hi*B_hi (M=128, N=192, K=8).
//
// Accuracy: the tensor core's fp32 accumulation truncates at every MMA, an error that grows
// with the number of MMAs into one accumulator (measured worst 6.7e-6 * Σ|a||b| with 512
// steps into one D at 4096^3, against the 1e-5 tolerance; 0.9e-6 with 64-step segments,
// 0.7e-6 with 32).  So the k loop is cut into 256-k segments accumulated in two
// alternating TMEM accumulators D0 / D1: while the MMAs fill one, the 8 accumulator warps
// add the other into fp32 registers (round-to-nearest adds), so the tensor pipe never waits
// for a drain.  At the end C = C0 + P, staged through shared memory and coalesced.
//
// Warp roles (448 threads; 14 warps cap registers at 128): 0-3 A transform, 4-11
// accumulators (segment drain + C update), 12 TMA producer, 13 MMA issuer.  TMEM (512
// columns): D0 [0,192), D1 [192,384), 4 A slots [384,512) of 32 columns (2 x (hi 8 | lo 8)).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "tc_ptx.cuh"

namespace mmmcu {

#ifndef TD_SEG
#define TD_SEG 16
#endif
constexpr int kTdStages = 8;    // B smem stages of kTdSub MMA sub-steps (16 k) each
constexpr int kTdSub = 2;       // MMA sub-steps (8 k, 3 MMAs) per stage
constexpr int kTdASlots = 4;    // A TMEM slots (32 columns: per sub-step hi 8 | lo 8)
constexpr int kTdThreads = 448; // warps 0-3 transform, 4-11 accumulators, 12 producer, 13 MMA
constexpr int kTdSeg = TD_SEG;  // stages (256 k) per TMEM accumulation segment
constexpr int kTdTM = 128;
constexpr int kTdTN = 192;
constexpr int kTdStepFloats = kTdTN * 8 * 2;  // one 8-k step image (K1): hi | lo, 12 KB
constexpr int kTdPStride = kTdTN + 4;         // staged P row stride (floats): conflict-free 16-byte accesses

struct TdShared {
  float b[kTdStages][kTdSub * kTdStepFloats];  // 8 x 24 KB; after the last MMA: C-update staging
  uint64_t full[kTdStages];                    // B stage landed (TMA bytes)
  uint64_t empty[kTdStages];                   // B stage consumed (tcgen05.commit)
  uint64_t aready[kTdASlots];                  // A slot written (4 transform warps)
  uint64_t aempty[kTdASlots];                  // A slot consumed (tcgen05.commit)
  uint64_t seg_full[2];                        // segment's last MMAs done (tcgen05.commit)
  uint64_t seg_empty[2];                       // D drained (8 accumulator warps)
  uint32_t tmem_base;
};
constexpr int kTdSmem = (int)sizeof(TdShared) + 1024;

__device__ __forceinline__ void td_bulk(void* smem_dst, const void* gsrc, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   tc::smem_u32(smem_dst)),
               "l"(gsrc), "r"(bytes), "r"(tc::smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void td_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(tc::smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void td_named_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

__global__ void __launch_bounds__(kTdThreads, 1)
k2_tc(const float* __restrict__ AT, int64_t kpad, const float* __restrict__ tcb, const int32_t* __restrict__ tck,
      const int32_t* __restrict__ tcn, int64_t maxsteps, float* __restrict__ C, int64_t ldc, int64_t M, int64_t N,
      const unsigned long long* __restrict__ sel) {
  if (sel && *sel != 32ull) return;  // device-side path choice (k1_finalize): 32 = TC
  extern __shared__ __align__(1024) uint8_t td_raw[];
  TdShared& sh = *reinterpret_cast<TdShared*>(td_raw + ((1024 - (tc::smem_u32(td_raw) & 1023)) & 1023));
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t rt = blockIdx.x, tb = blockIdx.y;
  const int64_t m0 = rt * kTdTM, n0 = tb * kTdTN;
  const int32_t total = tcn[tb];
  const int nsteps = (total + 7) >> 3;                 // 8-k sub-steps
  const int nstage = (nsteps + kTdSub - 1) / kTdSub;   // 16-k stages
  const int nseg = (nstage + kTdSeg - 1) / kTdSeg;

  if (tid == 0) {
    for (int s = 0; s < kTdStages; ++s) {
      tc::mbar_init(&sh.full[s], 1);
      tc::mbar_init(&sh.empty[s], 1);
    }
    for (int s = 0; s < kTdASlots; ++s) {
      tc::mbar_init(&sh.aready[s], 4);
      tc::mbar_init(&sh.aempty[s], 1);
    }
    for (int d = 0; d < 2; ++d) {
      tc::mbar_init(&sh.seg_full[d], 1);
      tc::mbar_init(&sh.seg_empty[d], 8);
    }
    tc::fence_mbar_init();
  }
  if (warp == 0) tc::tmem_alloc(&sh.tmem_base, 512);
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tbase = sh.tmem_base;
  constexpr uint32_t kAcol = 2 * kTdTN;  // TMEM columns of the A slots

  if (warp == 12) {
    // ------------------------------------------------------- TMA producer (B stages)
    if (lane == 0) {
      for (int j = 0; j < nstage; ++j) {
        const int st = j % kTdStages;
        const uint32_t bytes = (uint32_t)min(kTdSub, nsteps - kTdSub * j) * kTdStepFloats * 4u;
        tc::mbar_wait(&sh.empty[st], (uint32_t)(((j / kTdStages) & 1) ^ 1));
        td_expect_tx(&sh.full[st], bytes);
        td_bulk(sh.b[st], tcb + ((int64_t)tb * maxsteps + kTdSub * j) * kTdStepFloats, bytes, &sh.full[st]);
      }
    }
    __syncwarp();
  } else if (warp == 13) {
    // ------------------------------------------------------------------ MMA issuer
    // The whole warp runs the loop (warp-uniform operands stay in uniform registers); one
    // elected lane issues.  Per stage: 2 barrier waits (~60 cycles each even when already
    // complete) and 3 commits against 6 MMAs (576 cycles): 8-k stages left the tensor pipe
    // waiting on this chain.
    const uint32_t idesc = tc::idesc_tf32_m128(kTdTN);
    for (int j = 0; j < nstage; ++j) {
      const int st = j % kTdStages, sa = j % kTdASlots;
      const int g = j / kTdSeg, d = g & 1;
      if (j % kTdSeg == 0 && g >= 2) tc::mbar_wait(&sh.seg_empty[d], (uint32_t)(((g - 2) >> 1) & 1));
      tc::mbar_wait(&sh.full[st], (uint32_t)((j / kTdStages) & 1));
      tc::mbar_wait(&sh.aready[sa], (uint32_t)((j / kTdASlots) & 1));
      tc::fence_after_sync();
      const uint32_t baddr = tc::smem_u32(sh.b[st]);
      const uint32_t dcol = tbase + d * kTdTN;
      const bool two = kTdSub * j + 1 < nsteps;
      if (tc::elect_one()) {
#pragma unroll
        for (int u = 0; u < kTdSub; ++u) {
          if (u == 0 || two) {
            const uint32_t bu = baddr + u * kTdStepFloats * 4;
            const uint64_t bhi = tc::smem_desc(bu, 128, 256), blo = tc::smem_desc(bu + kTdTN * 32, 128, 256);
            const uint32_t ahi = tbase + kAcol + 32 * sa + 16 * u, alo = ahi + 8;
            tc::mma_tf32_ts(dcol, alo, bhi, idesc, (j % kTdSeg != 0 || u > 0) ? 1u : 0u);
            tc::mma_tf32_ts(dcol, ahi, blo, idesc, 1u);
            tc::mma_tf32_ts(dcol, ahi, bhi, idesc, 1u);
          }
        }
        tc::mma_commit(&sh.empty[st]);
        tc::mma_commit(&sh.aempty[sa]);
        if (j % kTdSeg == kTdSeg - 1 || j == nstage - 1) tc::mma_commit(&sh.seg_full[d]);
      }
      __syncwarp();
    }
  } else if (warp < 4) {
    // ---------------------------------------------------------------- A transform
    // Thread r owns tile row r (== TMEM lane r).  A is read straight from the K1 A^T tile
    // (a warp reads 128 contiguous bytes per k) one batch of 2 stages ahead, with the
    // live-k list two batches ahead; split into tf32 hi / lo; tcgen05.st into the slot's
    // TMEM columns once the MMAs of stage j - kTdASlots have released them.
    constexpr int kB = 2, KB = 8 * kTdSub * kB;  // stages per batch, k per batch
    const int r = tid;
    const uint32_t lane_off = (uint32_t)(warp * 32) << 16;
    const float* acol = AT + rt * kpad * 128 + r;
    const int4* kx4 = reinterpret_cast<const int4*>(tck + tb * maxsteps * 8);
    const int npos = nsteps * 8, nb = (nstage + kB - 1) / kB;
    auto load_k = [&](int b, int (&k)[KB]) {
#pragma unroll
      for (int q = 0; q < KB / 4; ++q) {
        const int4 v = (b * KB + 4 * q < npos) ? __ldg(kx4 + b * (KB / 4) + q) : make_int4(-1, -1, -1, -1);
        k[4 * q] = v.x;
        k[4 * q + 1] = v.y;
        k[4 * q + 2] = v.z;
        k[4 * q + 3] = v.w;
      }
    };
    auto load_a = [&](const int (&k)[KB], float (&a)[KB]) {
#pragma unroll
      for (int i = 0; i < KB; ++i) a[i] = k[i] >= 0 ? __ldg(acol + (int64_t)k[i] * 128) : 0.0f;
    };
    int kn[KB];
    float ac[KB], an[KB];
    load_k(0, kn);
    load_a(kn, ac);
    load_k(1, kn);
#pragma unroll 1
    for (int b = 0; b < nb; ++b) {
      load_a(kn, an);  // batch b + 1 (all -1 past the end: no loads)
      load_k(b + 2, kn);
#pragma unroll
      for (int i = 0; i < kB; ++i) {
        const int j = kB * b + i;
        if (j < nstage) {
          const int sa = j % kTdASlots;
          tc::mbar_wait(&sh.aempty[sa], (uint32_t)(((j / kTdASlots) & 1) ^ 1));
          tc::fence_after_sync();
#pragma unroll
          for (int u = 0; u < kTdSub; ++u) {
            uint32_t hi[8], lo[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) tc::split_tf32(ac[16 * i + 8 * u + e], hi[e], lo[e]);
            tc::tmem_st8(tbase + lane_off + kAcol + 32 * sa + 16 * u, hi);
            tc::tmem_st8(tbase + lane_off + kAcol + 32 * sa + 16 * u + 8, lo);
          }
          tc::tmem_st_wait();
          tc::fence_before_sync();
          __syncwarp();
          if (lane == 0) tc::mbar_arrive(&sh.aready[sa]);
        }
      }
#pragma unroll
      for (int e = 0; e < KB; ++e) ac[e] = an[e];
    }
  } else {
    // ------------------------------------------------------ accumulator warps 4..11
    // Warp w: tile row 32*(w%4) + lane (its TMEM lane), columns 96*((w-4)/4) .. +95, held
    // as fp32 registers.  Each segment's D is added in (round-to-nearest), then released.
    const int q4 = warp & 3, half = (warp - 4) >> 2;
    const int r = 32 * q4 + lane;
    const uint32_t taddr = tbase + ((uint32_t)(q4 * 32) << 16) + 96 * half;
    float acc[96];
#pragma unroll
    for (int j = 0; j < 96; ++j) acc[j] = 0.0f;
    for (int g = 0; g < nseg; ++g) {
      const int d = g & 1;
      tc::mbar_wait_sleep(&sh.seg_full[d], (uint32_t)((g >> 1) & 1));
      tc::fence_after_sync();
#pragma unroll
      for (int c = 0; c < 6; ++c) {
        uint32_t v[16];
        tc::tmem_ld16(taddr + d * kTdTN + 16 * c, v);
        tc::tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < 16; ++j) acc[16 * c + j] += __uint_as_float(v[j]);
      }
      tc::fence_before_sync();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&sh.seg_empty[d]);
    }
    if (nseg > 0) {
      // C = C0 + P through the (now idle) B stages: rows staged with a 196-float stride
      // (conflict-free 16-byte stores), then updated row by row, lanes along the row
      float* stage = &sh.b[0][0];
      float4* prow = reinterpret_cast<float4*>(stage + r * kTdPStride + 96 * half);
#pragma unroll
      for (int q = 0; q < 24; ++q) prow[q] = make_float4(acc[4 * q], acc[4 * q + 1], acc[4 * q + 2], acc[4 * q + 3]);
      td_named_sync(1, 256);
      for (int rr = warp - 4; rr < kTdTM; rr += 8) {
        const int64_t row = m0 + rr;
        if (row >= M) break;
        float* crow = C + row * ldc + n0;
        const float* pr = stage + rr * kTdPStride;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int col = 4 * lane + 128 * h;
          if (col < kTdTN) {
            const int64_t gcol = n0 + col;
            if (gcol + 3 < N) {
              float4 cv = *reinterpret_cast<const float4*>(crow + col);
              const float4 pv = *reinterpret_cast<const float4*>(pr + col);
              cv.x += pv.x;
              cv.y += pv.y;
              cv.z += pv.z;
              cv.w += pv.w;
              *reinterpret_cast<float4*>(crow + col) = cv;
            } else {
              for (int e = 0; e < 4; ++e)
                if (gcol + e < N) crow[col + e] += pr[col + e];
            }
          }
        }
      }
    }
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) {
    tc::fence_after_sync();
    tc::tmem_dealloc(tbase, 512);
  }
}

}  // namespace mmmcu
