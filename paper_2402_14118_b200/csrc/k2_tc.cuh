// K2-TC — dense-tile masked GEMM on the 5th-generation tensor cores (tcgen05, kind::tf32,
// 3xTF32 split), for cells whose masks leave the 128 x 192 C tiles dense enough to pay
// (BASELINE north_star: "tensor cores only for tiles that the masks leave dense enough ...
// and only if the result stays inside tolerance").
//
// Work unit: a 128-row x 192-column C tile (persistent CTAs, see below).  The k loop runs only over the
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
// 0.7e-6 with 32).  So the k loop is cut into 512-k segments accumulated in two
// alternating TMEM accumulators D0 / D1: while the MMAs fill one, the 4 accumulator warps
// add the other into the tile's fp32 partial P in shared memory (round-to-nearest adds),
// so the tensor pipe never waits for a drain.  At the end C = C0 + P, coalesced.
//
// Warp roles (320 threads): 0-3 A transform, 4-7 accumulators (segment drain + C update),
// 8 TMA producer, 9 MMA issuer.  TMEM (512
// columns): D0 [0,192), D1 [192,384), 4 A slots [384,512) of 32 columns (2 x (hi 8 | lo 8)),
// one per stage.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "tc_ptx.cuh"

namespace mmmcu {

#ifdef TD_PROF
__device__ unsigned long long* td_prof = nullptr;  // debug builds only: per-CTA cycle counters
#define TD_CLK(v) const long long v = clock64()
#define TD_ADD(i, x) (prof[i] += (x))
#else
#define TD_CLK(v)
#define TD_ADD(i, x)
#endif

#ifndef TD_KB
#define TD_KB 2
#endif
#ifndef TD_SEG
#define TD_SEG 32
#endif
#ifndef TD_STAGES
#define TD_STAGES 4
#endif
constexpr int kTdStages = TD_STAGES;  // stages of kTdSub MMA sub-steps (16 k): B smem + A TMEM slot
constexpr int kTdSub = 2;       // MMA sub-steps (8 k, 3 MMAs) per stage
constexpr int kTdThreads = 320; // warps 0-3 transform, 4-7 accumulators, 8 producer, 9 MMA
constexpr int kTdSeg = TD_SEG;  // stages (512 k) per TMEM accumulation segment (worst 1.0e-6)
constexpr int kTdTM = 128;
#ifndef TD_TN
#define TD_TN 192
#endif
constexpr int kTdTN = TD_TN;
constexpr int kTdStepFloats = kTdTN * 8 * 2;  // one 8-k step image (K1): hi | lo, 12 KB
constexpr int kTdPStride = kTdTN + 4;         // staged P row stride (floats): conflict-free 16-byte accesses

struct TdShared {
  float b[kTdStages][kTdSub * kTdStepFloats];  // B step images
  float a[kTdStages][8 * kTdSub][kTdTM];       // the stage's live A^T rows (8 KB each)
  float p[kTdTM][kTdPStride];                  // the tile's fp32 partial P (98 KB)
  uint64_t tma[kTdStages];     // the stage's B image and A rows landed (TMA bytes)
  uint64_t full[kTdStages];    // stage ready: A split into its TMEM slot (4 transform warps)
  uint64_t empty[kTdStages];   // stage consumed: one tcgen05.commit frees B / A smem and the A slot
  uint64_t seg_full[2];                        // segment's last MMAs done (tcgen05.commit)
  uint64_t seg_empty[2];                       // D drained (4 accumulator warps)
  uint32_t tmem_base;
};
constexpr int kTdSmem = (int)sizeof(TdShared) + 128;

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
// A tile whose B columns leave >= 3/4 of k live gets its A rows by TMA (runs of consecutive
// live k: ~1 copy per stage); sparser tiles would need up to 16 copies of 512 B per stage,
// more TMA time than the MMAs leave, so their A rows come through the transform warps' loads.
__device__ __forceinline__ bool td_dense(int32_t live, int64_t kpad) { return 4 * (int64_t)live >= 3 * kpad; }

__device__ __forceinline__ void td_named_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// Persistent: CTA b takes tiles t = b, b + gridDim.x, ...; tile t = (row tile t % m_tiles,
// column tile t / m_tiles), so the CTAs running together share B column tiles (L2 reuse).
// Every role walks the same tile sequence with running stage / slot / segment counters, so
// the producer and the transform warps run into the next tile while the accumulator warps
// update C for the previous one.
__global__ void __launch_bounds__(kTdThreads, 1)
k2_tc(const float* __restrict__ AT, int64_t kpad, const float* __restrict__ tcb, const int32_t* __restrict__ tck,
      const int32_t* __restrict__ tcn, int64_t maxsteps, float* __restrict__ C, int64_t ldc, int64_t M, int64_t N,
      int64_t m_tiles, int64_t n_tiles, const unsigned long long* __restrict__ sel) {
  if (sel && *sel != 32ull) return;  // device-side path choice (k1_finalize): 32 = TC
  extern __shared__ __align__(128) uint8_t td_raw[];
  TdShared& sh = *reinterpret_cast<TdShared*>(td_raw + ((128 - (tc::smem_u32(td_raw) & 127)) & 127));
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t ntiles = m_tiles * n_tiles;

  if (tid == 0) {
    for (int s = 0; s < kTdStages; ++s) {
      tc::mbar_init(&sh.tma[s], 1);
      tc::mbar_init(&sh.full[s], 4);
      tc::mbar_init(&sh.empty[s], 1);
    }
    for (int d = 0; d < 2; ++d) {
      tc::mbar_init(&sh.seg_full[d], 1);
      tc::mbar_init(&sh.seg_empty[d], 4);
    }
    tc::fence_mbar_init();
  }
  if (warp == 0) tc::tmem_alloc(&sh.tmem_base, 512);
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tbase = sh.tmem_base;
  constexpr uint32_t kAcol = 2 * kTdTN;  // TMEM columns of the A slots

  if (warp == 8) {
    // ---------------------------------------------------- TMA producer (B and A per stage)
    // Per stage: one bulk copy of the two B step images, and the stage's 16 live A^T rows
    // of the tile — one bulk copy per run of consecutive live k (a dense tile: 1 copy of
    // 8 KB).  Lane e < 16 holds live k number e of the stage (prefetched a stage ahead).
    uint32_t J = 0;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
      const int64_t rt = t % m_tiles, tb = t / m_tiles;
      const int32_t total = tcn[tb];
      const int nsteps = (total + 7) >> 3;
      const int nstage = (nsteps + kTdSub - 1) / kTdSub;
      const bool a_tma = td_dense(total, kpad);  // else the transform warps load A (LDG)
      const int32_t* kx = tck + tb * maxsteps * 8;
      const float* atile = AT + rt * kpad * 128;
      const int npos = nsteps * 8;
      // lane l holds live k number 32p + l for the stage pair p (prefetched a pair ahead:
      // the tck latency stays off the per-stage issue path)
      int kpair = lane < npos ? __ldg(kx + lane) : -1;
      int knext = 0;
      for (int j = 0; j < nstage; ++j, ++J) {
        const int st = J % kTdStages;
        if ((j & 1) == 0) {
          const int pn = (j + 2) * 16 + lane;
          knext = pn < npos ? __ldg(kx + pn) : -1;
        }
        int kcur = __shfl_sync(0xffffffffu, kpair, 16 * (j & 1) + (lane & 15));
        if (lane >= 16) kcur = -1;
        const int prev = __shfl_up_sync(0xffffffffu, kcur, 1);
        const bool valid = a_tma && lane < 16 && kcur >= 0;
        const bool cont = valid && lane > 0 && prev + 1 == kcur;
        const uint32_t vmask = __ballot_sync(0xffffffffu, valid);
        const uint32_t cmask = __ballot_sync(0xffffffffu, cont);
        const uint32_t bytes = (uint32_t)min(kTdSub, nsteps - kTdSub * j) * kTdStepFloats * 4u;
        if (lane == 0) {
          tc::mbar_wait(&sh.empty[st], ((J / kTdStages) & 1u) ^ 1u);
          td_expect_tx(&sh.tma[st], bytes + 512u * (uint32_t)__popc(vmask));
          td_bulk(sh.b[st], tcb + (tb * maxsteps + kTdSub * j) * kTdStepFloats, bytes, &sh.tma[st]);
        }
        __syncwarp();
        if (valid && !cont) {  // run start: rows kcur .. kcur + len - 1 -> slots lane .. lane + len - 1
          const uint32_t len = (uint32_t)__ffs(~(cmask >> (lane + 1)));
          td_bulk(sh.a[st][lane], atile + (int64_t)kcur * 128, 512u * len, &sh.tma[st]);
        }
        if (j & 1) kpair = knext;
      }
    }
  } else if (warp == 9) {
    // ------------------------------------------------------------------ MMA issuer
    // The whole warp runs the loop (warp-uniform operands stay in uniform registers); one
    // elected lane issues.  Each tcgen05.commit costs the tensor pipe ~50 cycles (measured:
    // 112.6 vs 96.1 cycles per N=192 MMA with a commit every 3), so a stage carries 6 MMAs
    // and ONE commit that frees both its B smem and its A TMEM slot.
    const uint32_t idesc = tc::idesc_tf32_m128(kTdTN);
    uint32_t J = 0, G = 0;
#ifdef TD_PROF
    long long prof[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    const long long p0 = clock64();
#endif
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
      const int64_t tb = t / m_tiles;
      const int nsteps = (tcn[tb] + 7) >> 3;
      const int nstage = (nsteps + kTdSub - 1) / kTdSub;
      for (int j = 0; j < nstage; ++j, ++J) {
        const int st = J % kTdStages;
        const uint32_t d = G & 1u;
        TD_CLK(c0);
        if (j % kTdSeg == 0 && G >= 2) tc::mbar_wait(&sh.seg_empty[d], ((G - 2) >> 1) & 1u);
        TD_CLK(c1);
        tc::mbar_wait(&sh.tma[st], (J / kTdStages) & 1u);
        tc::mbar_wait(&sh.full[st], (J / kTdStages) & 1u);
        TD_CLK(c2);
        TD_ADD(0, c1 - c0);
        TD_ADD(1, c2 - c1);
        tc::fence_after_sync();
        const uint32_t baddr = tc::smem_u32(sh.b[st]);
        const uint32_t dcol = tbase + d * kTdTN;
        const bool two = kTdSub * j + 1 < nsteps;
        const bool seg_end = j % kTdSeg == kTdSeg - 1 || j == nstage - 1;
        if (tc::elect_one()) {
#pragma unroll
          for (int u = 0; u < kTdSub; ++u) {
            if (u == 0 || two) {
              const uint32_t bu = baddr + u * kTdStepFloats * 4;
              const uint64_t bhi = tc::smem_desc(bu, 128, 256), blo = tc::smem_desc(bu + kTdTN * 32, 128, 256);
              const uint32_t ahi = tbase + kAcol + 32 * st + 16 * u, alo = ahi + 8;
              tc::mma_tf32_ts(dcol, alo, bhi, idesc, (j % kTdSeg != 0 || u > 0) ? 1u : 0u);
              tc::mma_tf32_ts(dcol, ahi, blo, idesc, 1u);
              tc::mma_tf32_ts(dcol, ahi, bhi, idesc, 1u);
            }
          }
          tc::mma_commit(&sh.empty[st]);
          if (seg_end) tc::mma_commit(&sh.seg_full[d]);
        }
        __syncwarp();
        if (seg_end) ++G;
        TD_CLK(c3);
        TD_ADD(2, c3 - c2);
      }
    }
#ifdef TD_PROF
    if (lane == 0 && td_prof) {
      unsigned long long* q = td_prof + 16 * blockIdx.x;
      for (int i = 0; i < 3; ++i) q[i] = prof[i];
      q[3] = clock64() - p0;
    }
#endif
  } else if (warp < 4) {
    // ---------------------------------------------------------------- A transform
    // Thread r owns tile row r (== TMEM lane r).  Per stage it splits the stage's 16 live A
    // values of its row into tf32 hi / lo and stores them with one tcgen05.st of 32 columns
    // into the stage's TMEM slot, then arrives on full.  The values come from smem (dense
    // tiles: the producer's TMA runs, `tma` barrier) or from the K1 A^T tile directly
    // (sparse tiles: coalesced loads one batch of 2 stages ahead, live-k list two batches
    // ahead, after the slot's previous MMAs released it: `empty` barrier).
    const int r = tid;
    const uint32_t lane_off = (uint32_t)(warp * 32) << 16;
    uint32_t J = 0;
    auto store_slot = [&](int st, const float (&vals)[8 * kTdSub]) {
      uint32_t v[32];  // slot columns: per sub-step u, hi at 16u .. 16u+7, lo at 16u+8 ..
#pragma unroll
      for (int u = 0; u < kTdSub; ++u)
#pragma unroll
        for (int e = 0; e < 8; ++e) tc::split_tf32(vals[8 * u + e], v[16 * u + e], v[16 * u + 8 + e]);
      tc::fence_after_sync();
      tc::tmem_st32(tbase + lane_off + kAcol + 32 * st, v);
      tc::tmem_st_wait();
      tc::fence_before_sync();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&sh.full[st]);
    };
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
      const int64_t rt = t % m_tiles, tb = t / m_tiles;
      const int32_t total = tcn[tb];
      const int nsteps = (total + 7) >> 3;
      const int nstage = (nsteps + kTdSub - 1) / kTdSub;
      if (td_dense(total, kpad)) {
        for (int j = 0; j < nstage; ++j, ++J) {
          const int st = J % kTdStages;
          const int nvalid = min(8 * kTdSub, total - 8 * kTdSub * j);
          tc::mbar_wait(&sh.tma[st], (J / kTdStages) & 1u);  // implies the slot's MMAs are done
          float vals[8 * kTdSub];
#pragma unroll
          for (int q = 0; q < 8 * kTdSub; ++q) vals[q] = q < nvalid ? sh.a[st][q][r] : 0.0f;
          store_slot(st, vals);
        }
      } else {
        constexpr int kB = TD_KB, KB = 8 * kTdSub * kB;  // stages per batch, k per batch
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
              const uint32_t Jj = J + j;
              const int st = Jj % kTdStages;
              tc::mbar_wait(&sh.empty[st], ((Jj / kTdStages) & 1u) ^ 1u);
              float vals[8 * kTdSub];
#pragma unroll
              for (int q = 0; q < 8 * kTdSub; ++q) vals[q] = ac[8 * kTdSub * i + q];
              store_slot(st, vals);
            }
          }
#pragma unroll
          for (int e = 0; e < KB; ++e) ac[e] = an[e];
        }
        J += nstage;
      }
    }
  } else {
    // ------------------------------------------------------- accumulator warps 4..7
    // Thread = tile row r = 32*(w%4) + lane (its TMEM lane).  The tile's fp32 partial P lives
    // in shared memory (row stride 196 floats: conflict-free 16-byte accesses): each
    // segment's D is added into the row (round-to-nearest; P = D for the first segment),
    // 16 columns per tcgen05.ld, then D is released.  After the tile's last segment,
    // C = C0 + P goes out with lanes along the rows (coalesced), while the MMAs already run
    // the next tile.  Keeping P out of registers leaves the transform warps the register
    // file (a spilling transform ran sparse tiles 2x slower).
    const int q4 = warp & 3;
    const int r = 32 * q4 + lane;
    const uint32_t taddr = tbase + ((uint32_t)(q4 * 32) << 16);
    float4* prow = reinterpret_cast<float4*>(&sh.p[r][0]);
    uint32_t G = 0;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
      const int64_t rt = t % m_tiles, tb = t / m_tiles;
      const int nsteps = (tcn[tb] + 7) >> 3;
      const int nstage = (nsteps + kTdSub - 1) / kTdSub;
      const int nseg = (nstage + kTdSeg - 1) / kTdSeg;
      if (nseg == 0) continue;
      for (int g = 0; g < nseg; ++g, ++G) {
        const uint32_t d = G & 1u;
        tc::mbar_wait_sleep(&sh.seg_full[d], (G >> 1) & 1u);
        tc::fence_after_sync();
#pragma unroll 1
        for (int c = 0; c < kTdTN / 16; ++c) {
          uint32_t v[16];
          tc::tmem_ld16(taddr + d * kTdTN + 16 * c, v);
          tc::tmem_ld_wait();
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            float4 x = make_float4(__uint_as_float(v[4 * q]), __uint_as_float(v[4 * q + 1]),
                                   __uint_as_float(v[4 * q + 2]), __uint_as_float(v[4 * q + 3]));
            if (g > 0) {
              const float4 y = prow[4 * c + q];
              x.x = y.x + x.x;
              x.y = y.y + x.y;
              x.z = y.z + x.z;
              x.w = y.w + x.w;
            }
            prow[4 * c + q] = x;
          }
        }
        tc::fence_before_sync();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(&sh.seg_empty[d]);
      }
      const int64_t m0 = rt * kTdTM, n0 = tb * kTdTN;
      td_named_sync(1, 128);  // every row of P is final
      // warp q4 updates rows q4, q4+4, ...; per 8 rows all loads go out before the adds
      const int64_t gc0 = n0 + 4 * lane, gc1 = gc0 + 128;
      const bool full0 = gc0 + 3 < N, full1 = lane < 16 && gc1 + 3 < N;
#pragma unroll 1
      for (int i0 = 0; i0 < 32; i0 += 8) {
        float4 cv[8][2];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int64_t row = m0 + q4 + 4 * (i0 + i);
          const float* crow = C + row * ldc;
          if (row < M && full0) cv[i][0] = *reinterpret_cast<const float4*>(crow + gc0);
          if (row < M && full1) cv[i][1] = *reinterpret_cast<const float4*>(crow + gc1);
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int rr = q4 + 4 * (i0 + i);
          const int64_t row = m0 + rr;
          if (row >= M) break;
          float* crow = C + row * ldc;
          const float* pr = sh.p[rr];
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int col = 4 * lane + 128 * h;
            if (col >= kTdTN) continue;
            const int64_t gcol = n0 + col;
            if (h == 0 ? full0 : full1) {
              float4 c4 = cv[i][h];
              const float4 pv = *reinterpret_cast<const float4*>(pr + col);
              c4.x += pv.x;
              c4.y += pv.y;
              c4.z += pv.z;
              c4.w += pv.w;
              *reinterpret_cast<float4*>(crow + gcol) = c4;
            } else {
#pragma unroll
              for (int e = 0; e < 4; ++e)
                if (gcol + e < N) crow[gcol + e] += pr[col + e];
            }
          }
        }
      }
      td_named_sync(1, 128);  // P may be overwritten by the next tile's first drain
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
