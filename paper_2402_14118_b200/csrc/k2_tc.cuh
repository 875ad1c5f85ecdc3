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

#ifndef TD_STAGES
#define TD_STAGES 4
#endif
#ifndef TD_STAGES16
#define TD_STAGES16 4
#endif
#ifndef TD_TN
#define TD_TN 192
#endif
constexpr int kTdTN = TD_TN;
constexpr int kTdStepFloats = kTdTN * 8 * 2;  // one K1 step image (8 k tf32 or 16 k fp16): hi | lo, 12 KB
// Operand precision of K2-TC: tf32 split (kind::tf32, 8 k per MMA) or fp16 split
// (kind::f16, 16 k per MMA at the same cycles per MMA: half the tensor time per k; operands
// scaled by powers of two so that fp16's 5-bit exponent holds them, see tc::f16_scale_exp).
template <bool F16>
struct TdCfg {
  static constexpr bool kPair = F16;                             // fp16: CTA pairs (cta_group::2, M=256)
  static constexpr int kStages = F16 ? TD_STAGES16 : TD_STAGES;  // B smem + A TMEM slot per stage
  static constexpr int kSub = 2;                                 // MMA sub-steps (3 MMAs each) per stage
  static constexpr int kStepK = F16 ? 16 : 8;                    // k per MMA sub-step (one K1 step image)
  static constexpr int kStageK = kStepK * kSub;                  // live k per stage: 16 / 32
  static constexpr int kSeg = 512 / kStageK;                     // stages per 512-k accumulation segment
  // B smem per stage: kSub step images, of which a pair CTA holds its N/2 columns
  static constexpr int kBStageFloats = kSub * kTdStepFloats / (kPair ? 2 : 1);
};
constexpr int kTdSub = 2;
constexpr int kTdThreads = 320; // warps 0-3 transform, 4-7 accumulators, 8 producer, 9 MMA
constexpr int kTdTM = 128;
constexpr int kTdPStride = kTdTN + 4;         // staged P row stride (floats): conflict-free 16-byte accesses

template <bool F16>
struct TdShared {
  using Cfg = TdCfg<F16>;
  float b[Cfg::kStages][Cfg::kBStageFloats];         // B step images (pair: this CTA's half)
  float a[Cfg::kStages][Cfg::kStageK][kTdTM];         // the stage's live A^T rows (8 / 16 KB)
  float p[kTdTM][kTdPStride];                         // the tile's fp32 partial P (98 KB)
  uint64_t tma[Cfg::kStages];     // the stage's B image and A rows landed (TMA bytes)
  uint64_t full[Cfg::kStages];    // stage ready: A split into its TMEM slot (4 transform warps)
  uint64_t empty[Cfg::kStages];   // stage consumed: one tcgen05.commit frees B / A smem and the A slot
  uint64_t seg_full[2];           // segment's last MMAs done (tcgen05.commit)
  uint64_t seg_empty[2];          // D drained (4 accumulator warps)
  uint32_t tmem_base;
};
template <bool F16>
constexpr int td_smem() { return (int)sizeof(TdShared<F16>) + 128; }

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
// update C for the previous one.  F16: amax / bmax hold the bits of max|A| / max|B| (K1),
// from which the power-of-two operand scales and the epilogue's unscale follow.
template <bool F16>
__global__ void __launch_bounds__(kTdThreads, 1)
k2_tc(const float* __restrict__ AT, int64_t kpad, const float* __restrict__ tcb, const int32_t* __restrict__ tck,
      const int32_t* __restrict__ tcn, int64_t maxsteps, float* __restrict__ C, int64_t ldc, int64_t M, int64_t N,
      int64_t m_tiles, int64_t n_tiles, const unsigned long long* __restrict__ sel,
      const uint32_t* __restrict__ amax, const unsigned long long* __restrict__ bmax) {
  using Cfg = TdCfg<F16>;
  constexpr int kStages = Cfg::kStages, kSub = Cfg::kSub, kStepK = Cfg::kStepK, kStageK = Cfg::kStageK,
                kSeg = Cfg::kSeg;
  constexpr bool kPair = Cfg::kPair;
  constexpr int kNArrive = kPair ? 8 : 4;  // transform / accumulator warps signalling the MMA issuer
  // (sel is read by both CTAs of a pair: both exit, or neither)
  if (sel && *sel != 32ull) return;  // device-side path choice (k1_finalize): 32 = TC
  extern __shared__ __align__(128) uint8_t td_raw[];
  TdShared<F16>& sh = *reinterpret_cast<TdShared<F16>*>(td_raw + ((128 - (tc::smem_u32(td_raw) & 127)) & 127));
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // pair: rank r of the cluster owns row tile 2p + r of pair tile p; the leader (r = 0) issues
  const uint32_t rank = kPair ? tc::cluster_rank() : 0u;
  const bool leader = rank == 0u;
  const int64_t unit0 = kPair ? blockIdx.x / 2 : blockIdx.x, nunits = kPair ? gridDim.x / 2 : gridDim.x;
  const int64_t m_units = kPair ? (m_tiles + 1) / 2 : m_tiles;  // (pair) row tiles per column tile
  const int64_t ntiles = m_units * n_tiles;
  auto row_tile = [&](int64_t t) { return kPair ? 2 * (t % m_units) + rank : t % m_units; };
  // a signal for the MMA issuer: local arrive, or (pair follower) remote arrive on the leader
  auto signal_issuer = [&](uint64_t* bar) {
    if (!kPair || leader) tc::mbar_arrive(bar);
    else tc::mbar_arrive_remote(bar, 0u);
  };

  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) {
      tc::mbar_init(&sh.tma[s], 1);
      tc::mbar_init(&sh.full[s], kNArrive);
      tc::mbar_init(&sh.empty[s], 1);
    }
    for (int d = 0; d < 2; ++d) {
      tc::mbar_init(&sh.seg_full[d], 1);
      tc::mbar_init(&sh.seg_empty[d], kNArrive);
    }
    tc::fence_mbar_init();
  }
  if (warp == 0) {
    if (kPair) tc::tmem_alloc2(&sh.tmem_base, 512);
    else tc::tmem_alloc(&sh.tmem_base, 512);
  }
  tc::fence_before_sync();
  if (kPair) tc::cluster_sync_all();  // the peer's barriers are initialised before any remote arrive
  else __syncthreads();
  tc::fence_after_sync();
  const uint32_t tbase = sh.tmem_base;
  constexpr uint32_t kAcol = 2 * kTdTN;  // TMEM columns of the A slots
  auto nsteps_of = [&](int32_t total) { return (total + kStepK - 1) / kStepK; };

  if (warp == 8) {
    // ---------------------------------------------------- producer (B and A per stage)
    // Per stage: one bulk copy of the stage's B step images, and the stage's live A^T rows of
    // the tile.  Dense tiles: one bulk copy per run of consecutive live k (1 copy of 8 / 16
    // KB).  Sparse tiles (short runs: per-run TMA copies would cost more TMA time than the
    // MMAs leave): the warp copies each live row with one 16-byte cp.async per lane
    // (LDGSTS, 512 B per instruction), tracked by the same barrier (cp.async.mbarrier.arrive,
    // issued before the expect_tx arrive so the phase cannot complete early).  Lane
    // e < kStageK holds live k number e of the stage (prefetched a stage ahead).
    uint32_t J = 0;
    for (int64_t t = unit0; t < ntiles; t += nunits) {
      const int64_t rt = row_tile(t), tb = t / m_units;
      const int32_t total = tcn[tb];
      const int nsteps = nsteps_of(total);
      const int nstage = (nsteps + kSub - 1) / kSub;
      const bool a_tma = td_dense(total, kpad);  // else A rows by cp.async
      // pair: the tile's step images are stored per column half (K1 pack), this CTA's half
      // of a stage is one contiguous copy
      const float* bsrc = kPair ? tcb + (tb * 2 + rank) * maxsteps * (kTdStepFloats / 2)
                                : tcb + tb * maxsteps * kTdStepFloats;
      constexpr int kStepCopy = kPair ? kTdStepFloats / 2 : kTdStepFloats;  // floats per step in this CTA
      const int32_t* kx = tck + tb * maxsteps * 8;
      const float* atile = AT + rt * kpad * 128;
      const int npos = nsteps * kStepK;
      int kc = (lane < kStageK && lane < npos) ? __ldg(kx + lane) : -1;
      for (int j = 0; j < nstage; ++j, ++J) {
        const int st = J % kStages;
        const int pn = (j + 1) * kStageK + lane;
        const int kn = (lane < kStageK && pn < npos) ? __ldg(kx + pn) : -1;
        const int prev = __shfl_up_sync(0xffffffffu, kc, 1);
        const bool valid = a_tma && kc >= 0;
        const bool cont = valid && lane > 0 && prev + 1 == kc;
        const uint32_t vmask = __ballot_sync(0xffffffffu, valid);
        const uint32_t cmask = __ballot_sync(0xffffffffu, cont);
        const uint32_t bytes = (uint32_t)min(kSub, nsteps - kSub * j) * kStepCopy * 4u;
        if (lane == 0) tc::mbar_wait(&sh.empty[st], ((J / kStages) & 1u) ^ 1u);
        __syncwarp();
        if (!a_tma) {
#pragma unroll 4
          for (int q = 0; q < kStageK; ++q) {
            const int kq = __shfl_sync(0xffffffffu, kc, q);
            if (kq >= 0)
              asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(tc::smem_u32(&sh.a[st][q][4 * lane])),
                           "l"(atile + (int64_t)kq * 128 + 4 * lane)
                           : "memory");
          }
          asm volatile("cp.async.mbarrier.arrive.shared::cta.b64 [%0];" ::"r"(tc::smem_u32(&sh.tma[st])) : "memory");
          __syncwarp();
        }
        if (lane == 0) {
          td_expect_tx(&sh.tma[st], bytes + 512u * (uint32_t)__popc(vmask));
          td_bulk(sh.b[st], bsrc + (int64_t)kSub * j * kStepCopy, bytes, &sh.tma[st]);
        }
        __syncwarp();
        if (valid && !cont) {  // run start: rows kc .. kc + len - 1 -> slots lane .. lane + len - 1
          const uint32_t len = lane == 31 ? 1u : (uint32_t)__ffs(~(cmask >> (lane + 1)));
          td_bulk(sh.a[st][lane], atile + (int64_t)kc * 128, 512u * len, &sh.tma[st]);
        }
        kc = kn;
      }
    }
  } else if (warp == 9) {
    if (!leader) goto td_done;  // pair follower: the leader issues the pair's MMAs
    // ------------------------------------------------------------------ MMA issuer
    // The whole warp runs the loop (warp-uniform operands stay in uniform registers); one
    // elected lane issues.  Each tcgen05.commit costs the tensor pipe ~50 cycles (measured:
    // 112.6 vs 96.1 cycles per N=192 MMA with a commit every 3), so a stage carries 6 MMAs
    // and ONE commit that frees both its B smem and its A TMEM slot.
    const uint32_t idesc = F16 ? tc::idesc_f16_m256(kTdTN) : tc::idesc_tf32_m128(kTdTN);
    uint32_t J = 0, G = 0;
#ifdef TD_PROF
    long long prof[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    const long long p0 = clock64();
#endif
    for (int64_t t = unit0; t < ntiles; t += nunits) {
      const int64_t tb = t / m_units;
      const int nsteps = nsteps_of(tcn[tb]);
      const int nstage = (nsteps + kSub - 1) / kSub;
      for (int j = 0; j < nstage; ++j, ++J) {
        const int st = J % kStages;
        const uint32_t d = G & 1u;
        TD_CLK(c0);
        if (j % kSeg == 0 && G >= 2) tc::mbar_wait(&sh.seg_empty[d], ((G - 2) >> 1) & 1u);
        TD_CLK(c1);
        tc::mbar_wait(&sh.tma[st], (J / kStages) & 1u);
        tc::mbar_wait(&sh.full[st], (J / kStages) & 1u);
        TD_CLK(c2);
        TD_ADD(0, c1 - c0);
        TD_ADD(1, c2 - c1);
        tc::fence_after_sync();
        const uint32_t baddr = tc::smem_u32(sh.b[st]);
        const uint32_t dcol = tbase + d * kTdTN;
        const bool seg_end = j % kSeg == kSeg - 1 || j == nstage - 1;
        if (tc::elect_one()) {
#pragma unroll
          for (int u = 0; u < kSub; ++u) {
            if (u == 0 || kSub * j + u < nsteps) {
              // per step: hi image then lo image (pair: of this CTA's N/2 columns)
              constexpr int kImg = kPair ? kTdTN * 16 : kTdTN * 32;  // bytes of one hi (or lo) image
              const uint32_t bu = baddr + u * 2 * kImg;
              const uint64_t bhi = tc::smem_desc(bu, 128, 256), blo = tc::smem_desc(bu + kImg, 128, 256);
              const uint32_t ahi = tbase + kAcol + 32 * st + 16 * u, alo = ahi + 8;
              const uint32_t acc0 = (j % kSeg != 0 || u > 0) ? 1u : 0u;
              if (F16) {
                tc::mma_f16_ts_pair(dcol, alo, bhi, idesc, acc0);
                tc::mma_f16_ts_pair(dcol, ahi, blo, idesc, 1u);
                tc::mma_f16_ts_pair(dcol, ahi, bhi, idesc, 1u);
              } else {
                tc::mma_tf32_ts(dcol, alo, bhi, idesc, acc0);
                tc::mma_tf32_ts(dcol, ahi, blo, idesc, 1u);
                tc::mma_tf32_ts(dcol, ahi, bhi, idesc, 1u);
              }
            }
          }
          if (kPair) {
            tc::mma_commit_pair(&sh.empty[st]);
            if (seg_end) tc::mma_commit_pair(&sh.seg_full[d]);
          } else {
            tc::mma_commit(&sh.empty[st]);
            if (seg_end) tc::mma_commit(&sh.seg_full[d]);
          }
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
    // Thread r owns tile row r (== TMEM lane r).  Per stage it waits for the stage's A^T rows
    // in shared memory (`tma`: the producer's bulk copies or cp.async rows; it also implies
    // the slot's previous MMAs are done), splits its row's live A values into hi / lo
    // (tf32: 16 values, one column each; fp16: 32 values scaled by 2^sA, two per column),
    // stores them with one tcgen05.st of 32 columns into the stage's TMEM slot and signals
    // the MMA issuer (`full`).
    const int r = tid;
    const uint32_t lane_off = (uint32_t)(warp * 32) << 16;
    const float sa = F16 ? tc::exp2_int(tc::f16_scale_exp(*amax)) : 1.0f;
    uint32_t J = 0;
    auto store_slot = [&](int st, const float (&vals)[kStageK]) {
      uint32_t v[32];  // slot columns: per sub-step u, hi at 16u .. 16u+7, lo at 16u+8 ..
#pragma unroll
      for (int u = 0; u < kSub; ++u) {
        if (F16) {
#pragma unroll
          for (int e = 0; e < 8; ++e)
            tc::split_f16x2(vals[16 * u + 2 * e] * sa, vals[16 * u + 2 * e + 1] * sa, v[16 * u + e], v[16 * u + 8 + e]);
        } else {
#pragma unroll
          for (int e = 0; e < 8; ++e) tc::split_tf32(vals[8 * u + e], v[16 * u + e], v[16 * u + 8 + e]);
        }
      }
      tc::fence_after_sync();
      tc::tmem_st32(tbase + lane_off + kAcol + 32 * st, v);
      tc::tmem_st_wait();
      tc::fence_before_sync();
      __syncwarp();
      if (lane == 0) signal_issuer(&sh.full[st]);
    };
    for (int64_t t = unit0; t < ntiles; t += nunits) {
      const int64_t tb = t / m_units;
      const int32_t total = tcn[tb];
      const int nsteps = nsteps_of(total);
      const int nstage = (nsteps + kSub - 1) / kSub;
      for (int j = 0; j < nstage; ++j, ++J) {
        const int st = J % kStages;
        const int nvalid = min(kStageK, total - kStageK * j);
        tc::mbar_wait(&sh.tma[st], (J / kStages) & 1u);  // implies the slot's MMAs are done
        float vals[kStageK];
#pragma unroll
        for (int q = 0; q < kStageK; ++q) vals[q] = q < nvalid ? sh.a[st][q][r] : 0.0f;
        store_slot(st, vals);
      }
    }
  } else {
    // ------------------------------------------------------- accumulator warps 4..7
    // Thread = tile row r = 32*(w%4) + lane (its TMEM lane).  The tile's fp32 partial P lives
    // in shared memory (row stride 196 floats: conflict-free 16-byte accesses): each
    // segment's D (fp16: times 2^-(sA+sB), exact) is added into the row (round-to-nearest;
    // P = D for the first segment), 16 columns per tcgen05.ld, then D is released.  After
    // the tile's last segment, C = C0 + P goes out with lanes along the rows (coalesced),
    // while the MMAs already run the next tile.  Keeping P out of registers leaves the
    // transform warps the register file (a spilling transform ran sparse tiles 2x slower).
    const int q4 = warp & 3;
    const int r = 32 * q4 + lane;
    const uint32_t taddr = tbase + ((uint32_t)(q4 * 32) << 16);
    const float ia = F16 ? tc::exp2_int(-tc::f16_scale_exp(*amax)) : 1.0f;
    const float ib = F16 ? tc::exp2_int(-tc::f16_scale_exp((uint32_t)*bmax)) : 1.0f;
    float4* prow = reinterpret_cast<float4*>(&sh.p[r][0]);
    uint32_t G = 0;
    for (int64_t t = unit0; t < ntiles; t += nunits) {
      const int64_t rt = row_tile(t), tb = t / m_units;
      const int nsteps = nsteps_of(tcn[tb]);
      const int nstage = (nsteps + kSub - 1) / kSub;
      const int nseg = (nstage + kSeg - 1) / kSeg;
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
            if (F16) {
              x.x = (x.x * ia) * ib;
              x.y = (x.y * ia) * ib;
              x.z = (x.z * ia) * ib;
              x.w = (x.w * ia) * ib;
            }
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
        if (lane == 0) signal_issuer(&sh.seg_empty[d]);
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
td_done:
  tc::fence_before_sync();
  if (kPair) tc::cluster_sync_all();  // both CTAs done: no remote arrive or MMA is in flight
  else __syncthreads();
  if (warp == 0) {
    tc::fence_after_sync();
    if (kPair) tc::tmem_dealloc2(tbase, 512);
    else tc::tmem_dealloc(tbase, 512);
  }
}

}  // namespace mmmcu
