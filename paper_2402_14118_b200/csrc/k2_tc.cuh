// K2-TC — dense-tile masked GEMM on the 5th-generation tensor cores (tcgen05), for cells whose
// masks leave the 128 x 192 C tiles dense enough to pay (BASELINE north_star: "tensor cores
// only for tiles that the masks leave dense enough ... and only if the result stays inside
// tolerance").
//
// Work unit: a C tile of 192 columns (persistent CTAs).  The k loop runs only over the tile's
// LIVE k (B[k, tile] has a non-zero, from K1's tlive masks), so B's block sparsity removes
// whole k steps; A's element zeros are multiplied (the tile is dense enough by the choice of
// this path).  Two operand precisions:
//   fp16 split (MMMCU_ALGO_TC, AUTO): x = hi + lo with hi = fp16(x * 2^s), lo = fp16(x * 2^s -
//     hi), s a power-of-two scale per A ROW and per 8-column B GROUP from K1's per-row /
//     per-group max|x| (tc::f16_scale_exp), undone exactly in the segment drain;
//     kind::f16 MMAs of K = 16, and CTA pairs (cta_group::2): a pair tile is 256 rows, each
//     CTA holds its 128 A rows (TMEM) and D rows, and HALF of B's 192 columns in its shared
//     memory — the leader CTA issues M=256 MMAs that read both halves, so each SM fetches
//     half of B.
//   tf32 split (MMMCU_ALGO_TC32): hi = top 19 bits, lo = x - hi; kind::tf32 MMAs of K = 8,
//     one CTA per 128-row tile.
// Per 16 (8) live k: D += A_lo*B_hi + A_hi*B_lo + A_hi*B_hi (3 MMAs, N = 192).
//
// Pipelines (measured per-role cycle counts, TD_PROF builds, decided each of these: one
// producer warp's per-stage instruction chain and one transform warp per row group were each
// slower than a stage's MMAs; P in shared memory left room for only 4 stages):
//   smem ring (kStages): per stage the B step images of 32 (16) live k and the A^T rows of
//     those k (fp32, K1's at[(rt*kpad + k)*128 + i]).  Two producer warps (alternate
//     stages) fill it with bulk copies (B; A runs of consecutive live k).  `tma[s]` =
//     landed; `empty[s]` = the transform read A (4 arrivals) and the stage's MMAs completed
//     (1 tcgen05.commit).
//   TMEM A slots (kSlots): the transform warps split the stage's A values into hi / lo and
//     store them into slot J % kSlots (lane = row), after the slot's previous MMAs completed
//     (the empty phase of stage J - kSlots); `full[t]` tells the MMA issuer.
//   accumulation segments: the tensor core truncates its fp32 accumulation at every MMA, an
//     error that grows with the MMAs accumulated into one D (measured worst 6.7e-6 *
//     Σ|a||b| with 512 tf32 steps, 0.9e-6 with 64).  So k is cut into segments of 64 MMA
//     steps (1024 k fp16, 512 k tf32); after each, the accumulator warps add D (unscaled by
//     2^-(sA+sB) for fp16) into the tile's fp32 partial P with round-to-nearest adds.  D is
//     DOUBLE-BUFFERED in TMEM (segment G accumulates into D[G % 2]) and P lives in the
//     accumulator threads' registers (thread = tile row, 96 columns each), so the MMAs of the
//     next segment never wait for a drain (`seg_full[b]` -> `seg_empty[b]` only guards the
//     reuse of D[b] two segments later; with one D the drains stalled the MMA warp 17% of a
//     dense cell, TD_PROF).  At the end of the unit C += P by bulk reduce-adds from shared
//     memory (the L2 does the fp32 adds).
//
// Warp roles (640 threads = 5 warpgroups): WG0-1 = warps 0-7 A transform (two groups,
// alternate stages); WG2-3 = warps 8-15 accumulators (column halves of D, P in registers:
// setmaxnreg.inc to 136); WG4 = warps 16 and 18 producers (alternate stages), 17 the MMA
// issuer (the pair leader's; the follower's idles), 19 a third producer or idle
// (setmaxnreg.dec to 48).  TMEM (512 columns): D[0] [0,192), D[1] [192,384), 4 A slots
// [384,512) of 32 columns (per MMA step: hi 8 | lo 8 columns; fp16 packs 2 k per column, even
// k in the low half).
#pragma once
#include <cuda.h>  // CUtensorMap (the A^T gather descriptor)
#include <cstdint>
#include <cuda_runtime.h>

#include "tc_ptx.cuh"

namespace mmmcu {

#ifdef TD_PROF
__device__ unsigned long long* td_prof = nullptr;  // debug builds only: per-CTA cycle counters
#define TD_CLK(v) const long long v = clock64()
#define TD_ADD(i, x) (prof[i] += (x))
// kernel-phase timestamps (ns, %globaltimer) of thread 0: td_prof + 4096 + 8 * CTA
#define TD_STAMP(i)                                                     \
  if (threadIdx.x == 0 && td_prof) {                                    \
    unsigned long long t_;                                              \
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));              \
    td_prof[4096 + 8 * blockIdx.x + (i)] = t_;                          \
  }
#else
#define TD_STAMP(i)
#define TD_CLK(v)
#define TD_ADD(i, x)
#endif

#ifndef TD_TN
#define TD_TN 192
#endif
constexpr int kTdTN = TD_TN;
constexpr int kTdStepFloats = kTdTN * 8 * 2;  // one K1 step image (8 k tf32 or 16 k fp16): hi | lo, 12 KB
#ifndef TD_NPROD16
#define TD_NPROD16 2
#endif
#ifndef TD_NPROD_SPARSE
#define TD_NPROD_SPARSE 2  // 3 measured no faster on sparse-k cells (0.132 vs 0.127-0.132 ms)
#endif
constexpr int kTdAccGroups = 2;  // accumulator warpgroups (column halves of D and P)
#ifdef TD_NO_SETMAXNREG
#define TD_SETMAXNREG(op, n)
#else
#define TD_SETMAXNREG(op, n) asm volatile("setmaxnreg." op ".sync.aligned.u32 %0;" ::"n"(n))
#endif
constexpr int kTdAccRegs = 136;  // setmaxnreg of the accumulator warpgroups (P: 96 registers)
constexpr int kTdCtlRegs = 48;   // setmaxnreg of the producer / MMA warpgroup
constexpr int kTdXfRegs = 80;    // setmaxnreg of the transform warpgroups
// setmaxnreg moves registers only within the CTA's launch allocation (640 x 96): an inc that
// the decs do not cover blocks forever (measured: a hang)
static_assert(256 * kTdXfRegs + 256 * kTdAccRegs + 128 * kTdCtlRegs <= 640 * 96, "warpgroup register budget");
constexpr int kTdTM = 128;
#ifndef TD_SLOTS32
#define TD_SLOTS32 2
#endif
#ifndef TD_STAGES32
#define TD_STAGES32 4
#endif
#ifndef TD_GROUP
#define TD_GROUP 4
#endif
#ifndef TD_SEGS
#define TD_SEGS 32
#endif
#ifndef TD_ACC_SLEEP
#define TD_ACC_SLEEP 32  // ns between the accumulator warps' seg_full polls (256 measured 1% slower)
#endif
#ifndef TD_HINT
#define TD_HINT 1  // L2 evict_last on the A^T / B-image bulk copies (dense cell 0.31 -> 0.29 ms)
#endif
#ifndef TD_GATHER
#define TD_GATHER 1  // the stage's live A^T rows by TMA tile::gather4 (4 rows per instruction)
#endif
constexpr int kTdMaxTail = 256;  // >= co-resident pairs / CTAs of one launch
#ifndef TD_TAIL_SPLIT
#define TD_TAIL_SPLIT 0  // 1: the last, partial round of units cut along k across all pairs (measured slower:
                         // dense cell 0.288 vs 0.273 ms, sparse-k 0.149 vs 0.129 ms; C no longer single-writer)
#endif
#ifndef TD_GATHER_RUNS
#define TD_GATHER_RUNS 16  // stages with at most this many runs of consecutive live k use bulk copies
                           // (measured: gathers win at ~23 runs per stage, lose at ~9)
#endif
constexpr int kTdGroup = TD_GROUP;            // row units per scheduling group (L2 reuse of A^T and B)

template <bool F16>
struct TdCfg {
  static constexpr bool kPair = F16;                  // fp16: CTA pairs (cta_group::2, M=256)
  static constexpr int kSub = 2;                      // MMA steps (3 MMAs each) per stage
  static constexpr int kStepK = F16 ? 16 : 8;         // k per MMA step (one K1 step image)
  static constexpr int kStageK = kStepK * kSub;       // live k per stage: 32 / 16
  // stages per accumulation segment (64 MMA steps; 128 measured 3% faster but doubled the
  // worst error to 2.3e-6)
  static constexpr int kSeg = TD_SEGS;
  // B smem per stage: kSub step images, of which a pair CTA holds its N/2 columns
  static constexpr int kBStageFloats = kSub * kTdStepFloats / (kPair ? 2 : 1);
  static constexpr int kStages = F16 ? 6 : TD_STAGES32;  // smem ring
  static constexpr int kSlots = F16 ? 4 : TD_SLOTS32;    // TMEM A slots of 32 columns
  static_assert(kStages > kSlots, "the smem ring must run ahead of the TMEM slots");
  // Two producers and two transform groups take alternate stages, and a waiter only ever
  // observed the phases of ITS OWN earlier stages: a parity wait on the phase of stage J is
  // sound only if the phase of stage J - kStages (smem ring) / J - kSlots - kStages (slot
  // reuse) already completed, which the same-parity waiter guarantees iff both are even (odd
  // counts gave false-positive waits: corrupted A slots with 4 / 5, a hang with 2 / 3).
  static_assert(kStages % 2 == 0 && kSlots % 2 == 0, "alternating roles need even ring sizes");
  // producer warps 16, 18 (, 19): stage J goes to producer J % nprod, nprod = kProd for
  // mostly-live cells and kProdSparse for sparse-k ones (whose A rows arrive in many small
  // gathers: one more warp issuing them; TD_NPROD_SPARSE)
  static constexpr int kProd = F16 ? TD_NPROD16 : 2;
  static constexpr int kProdSparse = F16 ? TD_NPROD_SPARSE : 2;
  static_assert(kStages % kProd == 0 && kStages % kProdSparse == 0, "each producer must own whole ring slots");
  static_assert((kProd == 2 || kProd == 3) && (kProdSparse == 2 || kProdSparse == 3),
                "producers are warps 16, 18 and (optionally) 19");
  // warps 0-7 transform, 8-15 accumulators, 16 / 18 / 19 producers, 17 MMA
  static constexpr int kThreads = 640;
};

template <bool F16>
struct TdShared {
  using Cfg = TdCfg<F16>;
  // per accumulator warp: its 32 rows x 32 columns of P for the C update, the 128-byte-swizzled
  // box one TMA tensor reduce-add takes (first: the struct is 1024-byte aligned)
  float xp[4 * kTdAccGroups][32][32];
  float b[Cfg::kStages][Cfg::kBStageFloats];   // B step images (pair: this CTA's half)
  float a[Cfg::kStages][Cfg::kStageK][kTdTM];  // the stage's live A^T rows
  uint64_t tma[Cfg::kStages];    // stage data landed (TMA bytes / cp.async arrivals)
  uint64_t empty[Cfg::kStages];  // stage consumed: 4 transform arrivals (one group) + 1 tcgen05.commit
  uint64_t full[Cfg::kSlots];       // A slot written (transform warps; pair: both CTAs')
  uint64_t seg_full[2];          // segment's MMAs into D[b] done (tcgen05.commit)
  uint64_t seg_empty[2];         // D[b] drained into P (accumulator warps; pair: both CTAs')
  uint32_t tmem_base;
};
template <bool F16>
constexpr int td_smem() { return (int)sizeof(TdShared<F16>) + 1024; }

__device__ __forceinline__ void td_bulk(void* smem_dst, const void* gsrc, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   tc::smem_u32(smem_dst)),
               "l"(gsrc), "r"(bytes), "r"(tc::smem_u32(bar))
               : "memory");
}
// The same with an L2 eviction-priority policy (createpolicy): the A^T tiles and B images are
// re-read by many CTAs, the C reduce-adds are not
__device__ __forceinline__ void td_bulk_hint(void* smem_dst, const void* gsrc, uint32_t bytes, uint64_t* bar,
                                             uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          tc::smem_u32(smem_dst)),
      "l"(gsrc), "r"(bytes), "r"(tc::smem_u32(bar)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ uint64_t td_policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void td_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(tc::smem_u32(bar)), "r"(bytes)
               : "memory");
}
// Four A^T rows (row coordinates r0..r3 of the 2-D A^T tensor, 128 floats each) into 2 KB of
// shared memory with one TMA tile::gather4 (sm_100): the live rows of a sparse-k stage arrive in
// 8 instructions however they are scattered (one bulk copy per run of consecutive live k left
// the transform warps waiting 58% of their time on sparse-k cells).
__device__ __forceinline__ void td_gather4(void* smem_dst, const CUtensorMap* tmap, int r0, int r1, int r2, int r3,
                                           uint64_t* bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3, %4, %5, %6}], [%7], %8;" ::"r"(tc::smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(tc::smem_u32(bar)),
      "l"(policy)
      : "memory");
}

// A tile is "mostly live" when >= 3/4 of its k are live (scheduling groups, below).
__device__ __forceinline__ bool td_dense(int32_t live, int64_t kpad) { return 4 * (int64_t)live >= 3 * kpad; }

// Persistent: CTA (pair) u takes work units t = u, u + #units, ...; unit t = (row tile (pair)
// t % m_units, column tile t / m_units), so the CTAs running together share B column tiles
// (L2 reuse).  Every role walks the same unit sequence with running stage / slot / segment
// counters, so the producer and the transform warps run into the next tile while the
// accumulator warps update C for the previous one.  F16: the high words of rrng [M] / grng
// [ldb/8] hold the bits of max|a| per A row and max|b| per 8-column B group (K1), from which
// the operand scales and the drain's unscale follow.
template <bool F16>
__global__ void __launch_bounds__(TdCfg<F16>::kThreads, 1)
k2_tc(const float* __restrict__ AT, int64_t kpad, const float* __restrict__ tcb, const int32_t* __restrict__ tck,
      const int32_t* __restrict__ tcn, int64_t maxsteps, float* __restrict__ C, int64_t ldc, int64_t M, int64_t N,
      int64_t m_tiles, int64_t n_tiles, const unsigned long long* __restrict__ sel,
      const unsigned long long* __restrict__ rrng, const unsigned long long* __restrict__ grng,
      const __grid_constant__ CUtensorMap tmap_at, const __grid_constant__ CUtensorMap tmap_c) {
  using Cfg = TdCfg<F16>;
  constexpr int kStages = Cfg::kStages, kSub = Cfg::kSub, kStepK = Cfg::kStepK, kStageK = Cfg::kStageK,
                kSeg = Cfg::kSeg, kTdSlots = Cfg::kSlots;
  constexpr bool kPair = Cfg::kPair;
  constexpr int kNAccum = (kPair ? 8 : 4) * kTdAccGroups;  // accumulator warps signalling seg_empty
  constexpr int kNXform = kPair ? 8 : 4;    // transform warps signalling the MMA issuer (full): one group
  TD_STAMP(0);
  tc::pdl_wait();  // launched with programmatic serialization after the K1 kernels / gated K2-SIMT
  TD_STAMP(1);
  // (sel is read by both CTAs of a pair: both exit, or neither)
  if (sel && *sel != 32ull) return;  // device-side path choice (k1_finalize): 32 = TC
  extern __shared__ __align__(128) uint8_t td_raw[];
  TdShared<F16>& sh = *reinterpret_cast<TdShared<F16>*>(td_raw + ((1024 - (tc::smem_u32(td_raw) & 1023)) & 1023));
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // pair: rank r of the cluster owns row tile 2p + r of pair tile p; the leader (r = 0) issues
  const uint32_t rank = kPair ? tc::cluster_rank() : 0u;
  const bool leader = rank == 0u;
  // unit indices in 32 bits (< 2^31 units for any operand that fits the device; 32-bit
  // division in unit_rc, fewer live registers across the role branches)
  const int unit0 = kPair ? blockIdx.x / 2 : blockIdx.x, nunits = kPair ? gridDim.x / 2 : gridDim.x;
  const int m_units = (int)(kPair ? (m_tiles + 1) / 2 : m_tiles);  // (pair) row tiles per column tile
  const int ntiles = m_units * (int)n_tiles;
  // unit order: groups of `grp_rows` row units; within a group, column tile major, so the
  // units running together share both B column tiles and A^T row tiles in L2.  Measured
  // (4096^3): mostly-live cells run best with groups of 4 row units (A^T reuse, 0.32 ->
  // 0.30 ms), sparse-k cells with whole columns (their A rows are gathered per column tile)
  // the live-k total over the tiles and the tail units' stage prefix (below), computed by all
  // threads at once (a per-thread loop of dependent loads cost ~10 us at kernel start)
  __shared__ unsigned long long s_live_sum;
  __shared__ int s_tail_pre[TD_TAIL_SPLIT ? kTdMaxTail + 1 : 1];
  if (tid == 0) s_live_sum = 0ull;
  __syncthreads();
  {
    unsigned long long part = 0;
    for (int64_t i = tid; i < n_tiles; i += blockDim.x) part += (unsigned long long)tcn[i];
    if (part) atomicAdd(&s_live_sum, part);
  }
  __syncthreads();
  const int64_t live_sum = (int64_t)s_live_sum;
  const bool mostly_live = 4 * live_sum >= 3 * kpad * n_tiles;  // td_dense on the average tile
  const int grp_rows = mostly_live ? kTdGroup : m_units;
  const int nprod = mostly_live ? Cfg::kProd : Cfg::kProdSparse;  // producer warps of this launch
  auto unit_rc = [&](int t, int64_t& ru, int64_t& tb) {
    const int gsz = grp_rows * (int)n_tiles, g = t / gsz, w = t % gsz;
    const int rows_g = min(grp_rows, m_units - g * grp_rows);
    tb = w / rows_g;
    ru = g * kTdGroup + w % rows_g;
  };
  auto row_tile = [&](int64_t ru) { return kPair ? 2 * ru + rank : ru; };
  auto nsteps_of = [&](int32_t total) { return (total + kStepK - 1) / kStepK; };
  auto nstage_of = [&](int t) {
    int64_t ru, tb;
    unit_rc(t, ru, tb);
    return (nsteps_of(tcn[tb]) + kSub - 1) / kSub;
  };
  // Work items (every role walks the same sequence): the first full_rounds rounds are whole
  // units t = unit0 + r * nunits; the units of the last, partial round are cut along k so
  // that every pair (CTA) gets an equal share of their concatenated stages — item = (unit,
  // stages [jb, je)), its partial C added by the same tensor reduce-adds (352 units on 74
  // pairs left 18 pairs idle for a fifth of a dense cell).
  const int full_rounds = ntiles / nunits, tail0 = full_rounds * nunits, ntail = ntiles - tail0;
  // exclusive prefix of the tail units' stage counts (ntail < nunits <= kTdMaxTail)
  if (TD_TAIL_SPLIT) {
    if (tid < ntail) s_tail_pre[tid + 1] = nstage_of(tail0 + tid);
    if (tid == 0) s_tail_pre[0] = 0;
    __syncthreads();
    if (tid == 0)
      for (int u = 1; u <= ntail; ++u) s_tail_pre[u] += s_tail_pre[u - 1];
    __syncthreads();
  }
  const int64_t tail_total = TD_TAIL_SPLIT ? s_tail_pre[ntail] : 0;
  auto item = [&](int it, int& t, int& jb, int& je) -> bool {
    if (!TD_TAIL_SPLIT) {
      t = unit0 + it * nunits;
      if (t >= ntiles) return false;
      jb = 0;
      je = nstage_of(t);
      return true;
    }
    if (it < full_rounds) {
      t = unit0 + it * nunits;
      jb = 0;
      je = nstage_of(t);
      return true;
    }
    const int64_t lo = tail_total * unit0 / nunits, hi = tail_total * (unit0 + 1) / nunits;
    int k = it - full_rounds;
    for (int u = 0; u < ntail; ++u) {  // (shared-memory prefix: cheap)
      const int64_t base = s_tail_pre[u], b0 = max(base, lo), b1 = min((int64_t)s_tail_pre[u + 1], hi);
      if (b0 < b1) {
        if (k == 0) {
          t = tail0 + u;
          jb = (int)(b0 - base);
          je = (int)(b1 - base);
          return true;
        }
        --k;
      }
      if (s_tail_pre[u + 1] >= hi) break;
    }
    return false;
  };
  // a signal for the MMA issuer: local arrive, or (pair follower) remote arrive on the leader
  auto signal_issuer = [&](uint64_t* bar) {
    if (!kPair || leader) tc::mbar_arrive(bar);
    else tc::mbar_arrive_remote(bar, 0u);
  };

  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) {
      tc::mbar_init(&sh.tma[s], 1);
      tc::mbar_init(&sh.empty[s], 1 + 4);
    }
    for (int t = 0; t < kTdSlots; ++t) tc::mbar_init(&sh.full[t], kNXform);
    for (int b = 0; b < 2; ++b) {
      tc::mbar_init(&sh.seg_full[b], 1);
      tc::mbar_init(&sh.seg_empty[b], kNAccum);
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
  TD_STAMP(2);
  constexpr uint32_t kAcol = 2 * kTdTN;  // TMEM columns: D[0] [0,192), D[1] [192,384), then the A slots
  // register budget per warpgroup (5 x 128 threads start at 96, setmaxnreg at the top of each
  // role's branch): the accumulators hold P, the producers / MMA issuer need few
  if (warp >= 16) {
  // warpgroup 4: one setmaxnreg for the whole warpgroup, then its warps' roles
  TD_SETMAXNREG("dec", kTdCtlRegs);
  if (warp == 16 || warp == 18 || (nprod == 3 && warp == 19)) {
    // ---------------------------------------------------- producers (B and A per stage)
    // Two warps, producer p = (warp - 12) / 2 fills the stages J with J % 2 == p (one warp's
    // per-stage instruction chain, ~760 cycles, was longer than the stage's 630 MMA cycles).
    // Per stage: one bulk copy of the stage's B step images, and the stage's live A^T rows,
    // one bulk copy per run of consecutive live k (with two producers this beats per-row
    // cp.async on sparse tiles too: 0.25 vs 0.56 ms at zB = 0.8, bw = 32).  Lane
    // e < kStageK holds live k number e of the stage; the list is loaded 4 stages ahead
    // (register shift chain).
    uint32_t J = 0;
#ifdef TD_PROF
    long long prof[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    const long long p0 = clock64();
#endif
    const uint32_t pp = warp == 16 ? 0u : (uint32_t)(warp - 17);  // producer index
    const uint64_t pol = TD_HINT ? td_policy_evict_last() : 0ull;
    int t, jb, je;
    for (int it = 0; item(it, t, jb, je); ++it) {
      int64_t ru, tb;
      unit_rc(t, ru, tb);
      const int64_t rt = row_tile(ru);
      const int32_t total = tcn[tb];
      const int nsteps = nsteps_of(total);
      // pair: the tile's step images are stored per column half (K1 pack), this CTA's half
      // of a stage is one contiguous copy
      constexpr int kStepCopy = kPair ? kTdStepFloats / 2 : kTdStepFloats;  // floats per step in this CTA
      const float* bsrc = tcb + (kPair ? (tb * 2 + rank) : tb) * maxsteps * kStepCopy;
      const int32_t* kx = tck + tb * maxsteps * 8;
#if !TD_GATHER
      const float* atile = AT + rt * kpad * 128;
#endif
      const int npos = nsteps * kStepK;
      auto kload = [&](int jj) {
        const int pn = jj * kStageK + lane;
        return (lane < kStageK && pn < npos) ? __ldg(kx + pn) : -1;
      };
      // this producer's stages of the tile: j0, j0 + 2, ... (J advances by the tile's count)
      const int NP = nprod;
      const int j0 = jb + (int)((pp + NP - (J % NP)) % NP);
      int kc = kload(j0), k1 = kload(j0 + NP), k2 = kload(j0 + 2 * NP), k3 = kload(j0 + 3 * NP);
      for (int j = j0; j < je; j += NP) {
        const uint32_t Jj = J + (uint32_t)(j - jb);
        const int st = Jj % kStages;
        const int kn = k1;
        k1 = k2;
        k2 = k3;
        k3 = kload(j + 4 * NP);
        const int prev = __shfl_up_sync(0xffffffffu, kc, 1);
        const bool valid = kc >= 0;
        const bool cont = valid && lane > 0 && prev + 1 == kc;
        const uint32_t vmask = __ballot_sync(0xffffffffu, valid);
        const uint32_t cmask = __ballot_sync(0xffffffffu, cont);
#ifdef TD_BHALF  // timing variant (wrong results): half of the stage's B bytes, to see how TMA-bound a cell is
        const uint32_t bytes = (uint32_t)min(kSub, nsteps - kSub * j) * kStepCopy * 2u;
#else
        const uint32_t bytes = (uint32_t)min(kSub, nsteps - kSub * j) * kStepCopy * 4u;
#endif
        TD_CLK(q0);
        if (lane == 0 && Jj >= (uint32_t)kStages) tc::mbar_wait(&sh.empty[st], ((Jj / kStages) & 1u) ^ 1u);
        __syncwarp();
        TD_CLK(q1);
        TD_ADD(0, q1 - q0);
#if TD_GATHER
        // the stage's live A^T rows: one bulk copy per run of consecutive live k when they form at
        // most TD_GATHER_RUNS runs (dense tiles: one 16 KB copy; tiles with ~9 runs per stage
        // measured 4% faster with copies), else lane g < ceil(nvalid / 4) gathers rows 4g .. 4g+3
        // (positions past the tile's live count repeat a valid row: their B images are zero;
        // very sparse-k tiles, ~23 runs per stage, measured 7-15% faster with gathers)
        const int nv = __popc(vmask);
        const bool runs = __popc(vmask & ~cmask) <= TD_GATHER_RUNS;
        const int ng = runs ? 0 : (nv + 3) >> 2;
        if (runs) {
          const float* atile = AT + rt * kpad * 128;
          if (lane == 0) {
#ifdef TD_ANONE  // timing variant (wrong results): no A^T copies at all
            td_expect_tx(&sh.tma[st], bytes);
#else
            td_expect_tx(&sh.tma[st], bytes + 512u * (uint32_t)nv);
#endif
            if (TD_HINT) td_bulk_hint(sh.b[st], bsrc + (int64_t)kSub * j * kStepCopy, bytes, &sh.tma[st], pol);
            else td_bulk(sh.b[st], bsrc + (int64_t)kSub * j * kStepCopy, bytes, &sh.tma[st]);
          }
          __syncwarp();
#ifndef TD_ANONE
          if (valid && !cont) {  // run start: rows kc .. kc + len - 1 -> slots lane .. lane + len - 1
            const uint32_t len = lane == 31 ? 1u : (uint32_t)__ffs(~(cmask >> (lane + 1)));
            td_bulk_hint(sh.a[st][lane], atile + (int64_t)kc * 128, 512u * len, &sh.tma[st], pol);
          }
#endif
        } else if (lane == 0) {
#ifdef TD_ANONE
          td_expect_tx(&sh.tma[st], bytes);
#else
          td_expect_tx(&sh.tma[st], bytes + 2048u * (uint32_t)ng);
#endif
          if (TD_HINT) td_bulk_hint(sh.b[st], bsrc + (int64_t)kSub * j * kStepCopy, bytes, &sh.tma[st], pol);
          else td_bulk(sh.b[st], bsrc + (int64_t)kSub * j * kStepCopy, bytes, &sh.tma[st]);
        }
        __syncwarp();
        if (!runs) {  // (warp-uniform)
          const int k0 = __shfl_sync(0xffffffffu, kc, 0);
          const int rowk = (int)(rt * kpad) + (valid ? kc : k0);
          const int q0 = __shfl_sync(0xffffffffu, rowk, (4 * lane) & 31), q1 = __shfl_sync(0xffffffffu, rowk, (4 * lane + 1) & 31);
          const int q2 = __shfl_sync(0xffffffffu, rowk, (4 * lane + 2) & 31), q3 = __shfl_sync(0xffffffffu, rowk, (4 * lane + 3) & 31);
#ifndef TD_ANONE
          if (lane < ng) td_gather4(sh.a[st][4 * lane], &tmap_at, q0, q1, q2, q3, &sh.tma[st], pol);
#endif
        }
#else
        if (lane == 0) {
          td_expect_tx(&sh.tma[st], bytes + 512u * (uint32_t)__popc(vmask));
          if (TD_HINT) td_bulk_hint(sh.b[st], bsrc + (int64_t)kSub * j * kStepCopy, bytes, &sh.tma[st], pol);
          else td_bulk(sh.b[st], bsrc + (int64_t)kSub * j * kStepCopy, bytes, &sh.tma[st]);
        }
        __syncwarp();
        if (valid && !cont) {  // run start: rows kc .. kc + len - 1 -> slots lane .. lane + len - 1
          const uint32_t len = lane == 31 ? 1u : (uint32_t)__ffs(~(cmask >> (lane + 1)));
          if (TD_HINT) td_bulk_hint(sh.a[st][lane], atile + (int64_t)kc * 128, 512u * len, &sh.tma[st], pol);
          else td_bulk(sh.a[st][lane], atile + (int64_t)kc * 128, 512u * len, &sh.tma[st]);
        }
#endif
        kc = kn;
      }
      J += (uint32_t)(je - jb);
    }
#ifdef TD_PROF
    if (lane == 0 && td_prof && warp == 16) {
      unsigned long long* q = td_prof + 16 * blockIdx.x;
      q[8] = prof[0];
      q[9] = clock64() - p0;
    }
#endif
  } else if (warp == 17) {
    if (!leader) goto td_done;  // pair follower: the leader issues the pair's MMAs
    // ------------------------------------------------------------------ MMA issuer
    // The whole warp runs the loop (warp-uniform operands stay in uniform registers); one
    // elected lane issues.  Each tcgen05.commit costs the tensor pipe ~50 cycles, so a stage
    // carries 6 MMAs and ONE commit, which frees its smem (producer) and, through the same
    // barrier phase, its TMEM A slot (transform).
    const uint32_t idesc = F16 ? tc::idesc_f16_m256(kTdTN) : tc::idesc_tf32_m128(kTdTN);
    uint32_t J = 0, G = 0;
#ifdef TD_PROF
    long long prof[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    const long long p0 = clock64();
#endif
    int t, jb, je;
    for (int it = 0; item(it, t, jb, je); ++it) {
      int64_t ru, tb;
      unit_rc(t, ru, tb);
      const int nsteps = nsteps_of(tcn[tb]);
      for (int j = jb; j < je; ++j, ++J) {
        const int jl = j - jb;  // stage within the item (segments start at the item's first stage)
        const int st = J % kStages, sl = J % kTdSlots;
        TD_CLK(c0);
        // D[G % 2] was drained (segment G - 2) before this segment overwrites it
        if (jl % kSeg == 0 && G >= 2) tc::mbar_wait(&sh.seg_empty[G & 1u], ((G >> 1) - 1) & 1u);
        TD_CLK(c1);
        tc::mbar_wait(&sh.tma[st], (J / kStages) & 1u);
        TD_CLK(c15);
        tc::mbar_wait(&sh.full[sl], (J / kTdSlots) & 1u);
        TD_CLK(c2);
#ifdef TD_PROF  // pair 0: the time every stage's MMAs are issued (ns), td_prof + 8192 + J
        if (td_prof && blockIdx.x == 0 && lane == 0 && J < 4096u) {
          unsigned long long t_;
          asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));
          td_prof[8192 + J] = t_;
        }
#endif
        TD_ADD(0, c1 - c0);
        TD_ADD(1, c2 - c1);
        TD_ADD(3, c15 - c1);
        TD_ADD(4, jl < 8 ? c2 - c1 : 0);  // the waits of a unit's first 8 stages
        tc::fence_after_sync();
        const uint32_t baddr = tc::smem_u32(sh.b[st]);
        const bool seg_end = jl % kSeg == kSeg - 1 || j == je - 1;
        const uint32_t dcol = tbase + kTdTN * (G & 1u);  // this segment's D buffer
        if (tc::elect_one()) {
#pragma unroll
          for (int u = 0; u < kSub; ++u) {
            if (u == 0 || kSub * j + u < nsteps) {
              // per step: hi image then lo image (pair: of this CTA's N/2 columns)
              constexpr int kImg = kPair ? kTdTN * 16 : kTdTN * 32;  // bytes of one hi (or lo) image
              const uint32_t bu = baddr + u * 2 * kImg;
              const uint64_t bhi = tc::smem_desc(bu, 128, 256), blo = tc::smem_desc(bu + kImg, 128, 256);
              const uint32_t ahi = tbase + kAcol + 32 * sl + 16 * u, alo = ahi + 8;
              const uint32_t acc0 = (jl % kSeg != 0 || u > 0) ? 1u : 0u;
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
            if (seg_end) tc::mma_commit_pair(&sh.seg_full[G & 1u]);
          } else {
            tc::mma_commit(&sh.empty[st]);
            if (seg_end) tc::mma_commit(&sh.seg_full[G & 1u]);
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
      q[10] = prof[3];
      q[15] = prof[4];
    }
#endif
  }  // (warp 19 with two producers: idle)
  } else if (warp < 8) {
    TD_SETMAXNREG("dec", kTdXfRegs);
    // ---------------------------------------------------------------- A transform
    // Two groups of 4 warps; group g = w/4 transforms the stages J with J % 2 == g, warp w
    // owning tile rows 32*(w%4) .. +31 (its TMEM lanes), so two stages' chains of barrier
    // waits, loads and TMEM stores overlap (one stage at a time left the transform the
    // slowest stage of the pipeline).  Per stage a thread waits for the stage's A^T rows in
    // shared memory (`tma`), reads its row's values and releases the smem (`empty`), splits
    // them into hi / lo (tf32: one column each; fp16: scaled by 2^sA, two per column), waits
    // until the MMAs of the slot's previous stage are done (the `empty` phase of stage
    // J - kSlots, which includes their commit), stores them with one tcgen05.st of 32
    // columns and signals the MMA issuer (`full`).
    const int grp = warp >> 2, r = 32 * (warp & 3) + lane;
    const uint32_t lane_off = (uint32_t)(32 * (warp & 3)) << 16;
    uint32_t J = 0;
#ifdef TD_PROF
    long long prof[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    const long long p0 = clock64();
#endif
    int t, jb, je;
    for (int it = 0; item(it, t, jb, je); ++it) {
      int64_t ru, tb;
      unit_rc(t, ru, tb);
      const int32_t total = tcn[tb];
      const int j0 = jb + (int)(((uint32_t)grp + 2u - (J & 1u)) & 1u);
      // fp16: this row's power-of-two scale 2^sA (from its max|a|, K1)
      const int64_t grow = row_tile(ru) * kTdTM + r;
      const float sa = F16 ? tc::exp2_int(tc::f16_scale_exp(grow < M ? (uint32_t)(__ldg(rrng + grow) >> 32) : 0u)) : 1.0f;
      for (int j = j0; j < je; j += 2) {
        const uint32_t Jj = J + (uint32_t)(j - jb);
        const int st = Jj % kStages, sl = Jj % kTdSlots;
        const int nvalid = min(kStageK, total - kStageK * j);
        TD_CLK(q0);
        tc::mbar_wait(&sh.tma[st], (Jj / kStages) & 1u);
        TD_CLK(q1);
        float vals[kStageK];
#pragma unroll
        for (int q = 0; q < kStageK; ++q) vals[q] = q < nvalid ? sh.a[st][q][r] : 0.0f;
        tc::fence_async_smem();  // these generic-proxy reads before the producer's async-proxy refill
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(&sh.empty[st]);  // A smem read (the MMA commit completes the phase)
        uint32_t v[32];  // per step u: hi at 16u .. 16u+7, lo at 16u+8 ..
#pragma unroll
        for (int u = 0; u < kSub; ++u) {
          if (F16) {
#pragma unroll
            for (int e = 0; e < 8; ++e)
              tc::split_f16x2_scaled(vals[16 * u + 2 * e], vals[16 * u + 2 * e + 1], sa, v[16 * u + e],
                                     v[16 * u + 8 + e]);
          } else {
#pragma unroll
            for (int e = 0; e < 8; ++e) tc::split_tf32(vals[8 * u + e], v[16 * u + e], v[16 * u + 8 + e]);
          }
        }
        TD_CLK(q15);
        if (Jj >= (uint32_t)kTdSlots) {  // the slot's previous MMAs (stage Jj - kSlots) are done
          const uint32_t Jp = Jj - kTdSlots;
          tc::mbar_wait(&sh.empty[Jp % kStages], (Jp / kStages) & 1u);
        }
        TD_CLK(q2);
        TD_ADD(2, q2 - q15);
        tc::fence_after_sync();
        tc::tmem_st32(tbase + lane_off + kAcol + 32 * sl, v);
        tc::tmem_st_wait();
        tc::fence_before_sync();
        __syncwarp();
        if (lane == 0) signal_issuer(&sh.full[sl]);
        TD_CLK(q3);
        TD_ADD(0, q1 - q0);
        TD_ADD(1, q3 - q1);
      }
      J += (uint32_t)(je - jb);
    }
#ifdef TD_PROF
    if (tid == 0 && td_prof) {
      unsigned long long* q = td_prof + 16 * blockIdx.x;
      q[4] = prof[0];
      q[5] = prof[1];
      q[6] = clock64() - p0;
      q[7] = prof[2];
    }
#endif
  } else if (warp < 16) {
    TD_SETMAXNREG("inc", kTdAccRegs);
    // ------------------------------------------------------- accumulator warps 8..15
    // Thread = tile row r = 32*(w%4) + lane (its TMEM lane); warpgroup ag = columns
    // [96 ag, 96 ag + 96) of the tile.  Per segment G: wait for D[G % 2], add it (fp16: times
    // 2^-(sA+sB), exact) into the row's partial P in REGISTERS with round-to-nearest adds
    // (P = D for the unit's first segment), 16 columns per tcgen05.ld, then release D[G % 2]
    // (its MMAs two segments later may start).  After the item's last segment: C += P by TMA
    // tensor reduce-adds (below); an item that is a k-range of a unit adds its partial sum.
    const int q4 = warp & 3;
    const int ag = (warp >> 2) & 1;                  // accumulator group: columns [96 ag, 96 ag + 96)
    constexpr int kCh = kTdTN / 32 / kTdAccGroups;   // 32-column chunks per group (3)
    const int c0 = ag * kCh;
    const uint32_t taddr = tbase + ((uint32_t)(q4 * 32) << 16);
    float P[kCh * 32];
    uint32_t G = 0, R = 0;  // segments drained, C chunks reduced
#ifdef TD_PROF
    long long prof[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    const long long p0 = clock64();
#endif
    int t, jb, je;
    for (int it = 0; item(it, t, jb, je); ++it) {
      int64_t ru, tb;
      unit_rc(t, ru, tb);
      const int64_t rt = row_tile(ru);
      const int nseg = (je - jb + kSeg - 1) / kSeg;
      if (nseg == 0) continue;
      // fp16: undo this row's scale 2^sA and each 8-column group's 2^sB (exact powers of two)
      const int64_t grow = rt * kTdTM + 32 * q4 + lane;
      const float ia = F16 ? tc::exp2_int(-tc::f16_scale_exp(grow < M ? (uint32_t)(__ldg(rrng + grow) >> 32) : 0u)) : 1.0f;
      // lane q < 12 holds the unscale of 8-column group q of this group's 96 columns (read by
      // shuffles in the drain: 12 fewer live registers beside P)
      float ibl = 1.0f;
      if (F16 && lane < kCh * 4) {
        const int64_t gc = tb * kTdTN + 32 * c0 + 8 * lane;
        ibl = tc::exp2_int(-tc::f16_scale_exp(gc < N ? (uint32_t)(__ldg(grng + (gc >> 3)) >> 32) : 0u));
      }
      for (int g = 0; g < nseg; ++g, ++G) {
        const uint32_t b = G & 1u;
        TD_CLK(a0);
        if (TD_ACC_SLEEP > 0) tc::mbar_wait_sleep_ns(&sh.seg_full[b], (G >> 1) & 1u, TD_ACC_SLEEP);
        else tc::mbar_wait(&sh.seg_full[b], (G >> 1) & 1u);
        tc::fence_after_sync();
        TD_CLK(a1);
        TD_ADD(0, a1 - a0);
        const bool first = g == 0;
#pragma unroll
        for (int h = 0; h < 2 * kCh; ++h) {  // 16-column pieces
          uint32_t d[16];
          tc::tmem_ld16(taddr + kTdTN * b + 32 * c0 + 16 * h, d);
          tc::tmem_ld_wait();
          const float s0 = __shfl_sync(0xffffffffu, ibl, 2 * h), s1 = __shfl_sync(0xffffffffu, ibl, 2 * h + 1);
#pragma unroll
          for (int e = 0; e < 16; ++e) {
            float x = __uint_as_float(d[e]);
            if (F16) x *= ia;  // exact (power of two)
            const float s = e < 8 ? s0 : s1;
            // p + x*ib in one rounding (x*ib exact): the same value as the add of the product
            P[16 * h + e] = first ? x * s : fmaf(x, s, P[16 * h + e]);
          }
        }
        tc::fence_before_sync();
        __syncwarp();
        if (lane == 0) signal_issuer(&sh.seg_empty[b]);
        TD_CLK(a2);
        TD_ADD(1, a2 - a1);
      }
      TD_CLK(a3);
      // C += P: per 32 columns one TMA tensor reduce-add of the warp's 32 x 32 box (the L2
      // performs the fp32 adds, one writer per element; rows / columns past M / N are clipped
      // by the tensor map).  128-byte-swizzled staging: thread = row, its 16-byte chunk q at
      // chunk q ^ (row % 8), so the 32 rows' stores spread over the banks.  (One 128-byte bulk
      // reduce per thread and 32 columns queued 16x more TMA operations, which delayed the
      // operand loads of sparse-k cells.)
      const int64_t row0 = rt * kTdTM + 32 * q4, n0 = tb * kTdTN;
      float* box = &sh.xp[4 * ag + q4][0][0];
#pragma unroll
      for (int c = 0; c < kCh; ++c, ++R) {
        if (R > 0) {  // the previous reduce of this box has read it
          if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
          __syncwarp();
        }
#pragma unroll
        for (int q = 0; q < 8; ++q)
          *reinterpret_cast<float4*>(box + 32 * lane + 4 * (q ^ (lane & 7))) =
              make_float4(P[32 * c + 4 * q], P[32 * c + 4 * q + 1], P[32 * c + 4 * q + 2], P[32 * c + 4 * q + 3]);
        tc::fence_async_smem();  // generic-proxy stores before the tensor (async-proxy) read
        __syncwarp();
        if (lane == 0 && row0 < M) {
          const int32_t col = (int32_t)(n0 + 32 * (c0 + c));
          asm volatile(
              "cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                  reinterpret_cast<uint64_t>(&tmap_c)),
              "r"(col), "r"((int32_t)row0), "r"(tc::smem_u32(box))
              : "memory");
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
      }
      TD_CLK(a4);
      TD_ADD(2, a4 - a3);
    }
#ifdef TD_PROF
    if (lane == 0 && td_prof && warp == 8) {
      unsigned long long* q = td_prof + 16 * blockIdx.x;
      q[11] = prof[0];
      q[12] = prof[1];
      q[13] = prof[2];
      q[14] = clock64() - p0;
    }
#endif
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");  // reduces done before the CTA exits
    __syncwarp();
  }
td_done:
  TD_STAMP(3);  // thread 0 (a transform thread): its role loop is done
  tc::fence_before_sync();
  if (kPair) tc::cluster_sync_all();  // both CTAs done: no remote arrive or MMA is in flight
  else __syncthreads();
  TD_STAMP(4);
  if (warp == 0) {
    tc::fence_after_sync();
    if (kPair) tc::tmem_dealloc2(tbase, 512);
    else tc::tmem_dealloc(tbase, 512);
  }
}

}  // namespace mmmcu
