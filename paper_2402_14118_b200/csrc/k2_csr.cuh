// K2-CSR — the masked multiply driven by A's non-zero index ("the middle loop
// iterates only the non-zeros of A"; PAPER Fig. 4 / Fig. 11), for
// short, very sparse A (BASELINE configs[3], the skinny decode shape); forced with
// MMMCU_ALGO_CSR.  Measured on configs[3] it is 3.7x slower than K2-SIMT (3.6 vs 0.98 ms:
// latency-bound at 8 warps per SM, the 192 KB ring and C tile leave no room for more), so
// AUTO does not select it.
//
// K2-SIMT walks B's live (k, slice) rows and predicates every lane on a_ik != 0, so its issue
// slots scale with M x N x K_live whatever A's density; K2-TC multiplies A's zeros outright.
// Here the work is only the surviving (a_ik, B block) pairs:
//
//   unit  = 128 rows x 128 columns of C, held in SHARED memory (64 KB) for the whole k loop,
//           so any row can be updated at any k (register tiles cannot be indexed by a row that
//           changes with k).
//   chunk = 32 k: the A^T rows of the chunk (K1's A^T tile; only the tile's rows below M) and
//           ONLY the live 16-column blocks of B's chunk rows (per-thread cp.async, gated by K1's
//           group k-masks, which are prefetched a chunk ahead) are staged in a 4-deep ring.
//   warp  = 32 columns (lane = column) x half of the unit's 32-row groups.  Per chunk it visits
//           only the k where one of its four 8-column groups is live; per such k its rows with
//           a_ik != 0 come from a ballot over the staged A^T column (the per-row index lists of
//           K1, transposed per chunk), and per row c = fmaf(a_ik, b_kj, c) on the lanes whose
//           group's code bit is set (kernel_table.cpp:17-20), four rows in flight.
//
// Every C element therefore receives fmaf(a_ik, b_kj, c) over its surviving k in ascending
// order — the oracle's chain — so K2-CSR is bit-identical to the reference kernel table, like
// K2-SIMT.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace mmmcu {

constexpr int kCsKC = 32;    // k per chunk (one bitmap / group-mask word)
constexpr int kCsTM = 128;   // rows per unit (an A^T tile)
constexpr int kCsTN = 128;   // columns per unit
constexpr int kCsStages = 4;
constexpr int kCsThreads = 256;

struct CsStage {
  float at[kCsKC][kCsTM];  // 16 KB: A^T rows k0 .. k0+31 of the row tile
  float b[kCsKC][kCsTN];   // 16 KB: B chunk rows, live 16-column blocks only
};
struct CsShared {
  float c[kCsTM][kCsTN];             // 64 KB: the C tile
  CsStage st[kCsStages];             // 128 KB
};
constexpr int kCsSmem = (int)sizeof(CsShared) + 128;

__device__ __forceinline__ void cs_cp_async16(void* smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(smem)),
               "l"(gmem)
               : "memory");
}

// One unit (row tile rt, 128-column tile tb); 256 threads; sh in dynamic shared memory.
__device__ __forceinline__ void k2_csr_unit(CsShared& sh, const float* __restrict__ AT, int64_t kpad,
                                            const float* __restrict__ B, int64_t ldb, const uint32_t* __restrict__ bgrp,
                                            int64_t kw, float* __restrict__ C, int64_t ldc, int64_t M, int64_t K,
                                            int64_t N, int64_t rt, int64_t tb) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t m0 = rt * kCsTM, n0 = tb * kCsTN;
  const int cq = warp & 3, half = warp >> 2;  // columns 32 cq .. +31, row groups half, half + 2
  const int64_t ngrp_all = ldb >> 3;
  const int rows_tile = (int)(M - m0 < kCsTM ? M - m0 : kCsTM);
  const int rgroups = (rows_tile + 31) >> 5;  // 32-row groups of the tile that hold rows

  // ---- C tile into shared memory (c += a*b: the chain starts from C)
  for (int e = tid; e < kCsTM * (kCsTN / 4); e += kCsThreads) {
    const int r = e / (kCsTN / 4), q = e % (kCsTN / 4);
    const int64_t row = m0 + r, col = n0 + 4 * q;
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (row < M && col < N) {
      if (col + 4 <= N) v = *reinterpret_cast<const float4*>(C + row * ldc + col);
      else {
        float t[4] = {0.f, 0.f, 0.f, 0.f};
        for (int u = 0; u < 4 && col + u < N; ++u) t[u] = C[row * ldc + col + u];
        v = make_float4(t[0], t[1], t[2], t[3]);
      }
    }
    *reinterpret_cast<float4*>(&sh.c[r][4 * q]) = v;
  }

  // staging: thread t owns the (k = t / 8, 16-column block t % 8) pair of every chunk; its two
  // group words are loaded one chunk ahead of the copies they gate
  const int skk = tid >> 3, sblk = tid & 7;
  const int64_t scol = n0 + 16 * sblk, sg = scol >> 3;
  auto gate_words = [&](int64_t x) -> uint32_t {
    if (x >= kw || scol >= ldb) return 0u;
    return bgrp[sg * kw + x] | (sg + 1 < ngrp_all ? bgrp[(sg + 1) * kw + x] : 0u);
  };
  auto stage = [&](int64_t x, uint32_t gate) {  // chunk x into ring slot x % kCsStages
    if (x < kw) {
      CsStage& S = sh.st[x % kCsStages];
      const float* src = AT + (rt * kpad + x * kCsKC) * kCsTM;
      const int per_k = rgroups * 8;  // 16-byte pieces of one k's rows
      for (int e = tid; e < kCsKC * per_k; e += kCsThreads) {
        const int kk = e / per_k, p = e % per_k;
        cs_cp_async16(&S.at[kk][4 * p], src + kk * kCsTM + 4 * p);
      }
      const int64_t k = x * kCsKC + skk;
      if (k < K && ((gate >> skk) & 1u)) {
        const float* bs = B + k * ldb + scol;
#pragma unroll
        for (int q = 0; q < 4; ++q) cs_cp_async16(&S.b[skk][16 * sblk + 4 * q], bs + 4 * q);
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");  // (an empty group past the end)
  };
  // this warp's four 8-column groups: their k-mask words of chunk x (lane j < 4 loads group j)
  auto group_words = [&](int64_t x, uint32_t& mine, uint32_t& any) {
    const int64_t col = n0 + 32 * cq + 8 * (lane & 3), g = col >> 3;
    const uint32_t w = (lane < 4 && col < ldb) ? bgrp[g * kw + x] : 0u;
    const uint32_t w0 = __shfl_sync(0xffffffffu, w, 0), w1 = __shfl_sync(0xffffffffu, w, 1);
    const uint32_t w2 = __shfl_sync(0xffffffffu, w, 2), w3 = __shfl_sync(0xffffffffu, w, 3);
    const int j = lane >> 3;
    mine = j == 0 ? w0 : j == 1 ? w1 : j == 2 ? w2 : w3;
    any = w0 | w1 | w2 | w3;
  };

  // prologue: chunks 0 .. S-2 in flight, the gate words of chunk S-1 in registers
#pragma unroll
  for (int x = 0; x < kCsStages - 1; ++x) stage(x, gate_words(x));
  uint32_t gate_next = gate_words(kCsStages - 1);
  uint32_t mine, any;
  group_words(0, mine, any);
  const int col = 32 * cq + lane;
  for (int64_t x = 0; x < kw; ++x) {
    const int s = (int)(x % kCsStages);
    asm volatile("cp.async.wait_group %0;" ::"n"(kCsStages - 2) : "memory");  // chunk x landed (this thread)
    __syncthreads();  // ... for every thread; slot (x - 1) % S is free, the masks of x - 1 are read
    // refill the freed slot with chunk x + S - 1 (gate words loaded one iteration ago)
    stage(x + kCsStages - 1, gate_next);
    gate_next = gate_words(x + kCsStages);
    uint32_t mine_n, any_n;
    group_words(x + 1 < kw ? x + 1 : x, mine_n, any_n);  // next chunk's, latency hidden by this one
    const CsStage& S = sh.st[s];
    // ---- the surviving (a_ik, B block) pairs of this warp, ascending k: the k where one of the
    // warp's groups is live; per k the warp's rows with a_ik != 0 by ballot over the staged A^T
    // column (row groups q = half, half + 2 of the tile: balanced for 64-row tiles too)
    const int64_t kvalid = K - x * kCsKC;
    uint32_t mk = any;
    if (kvalid < 32) mk &= (1u << kvalid) - 1u;
    while (mk) {
      const int kk = __ffs(mk) - 1;
      mk &= mk - 1;
      const float b = S.b[kk][col];
      const bool live = (mine >> kk) & 1u;
#pragma unroll
      for (int qq = 0; qq < 2; ++qq) {
        const int q = half + 2 * qq;
        if (q >= rgroups) break;
        uint32_t rm = __ballot_sync(0xffffffffu, S.at[kk][32 * q + lane] != 0.0f);
        const int rbase = 32 * q;
        while (rm) {  // up to four rows per iteration (independent chains)
          int r[4];
          int n = 0;
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            r[u] = rm ? rbase + __ffs(rm) - 1 : -1;
            if (rm) {
              rm &= rm - 1;
              ++n;
            }
          }
          float a[4], c[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int ru = r[u] < 0 ? r[0] : r[u];
            a[u] = S.at[kk][ru];
            c[u] = sh.c[ru][col];
          }
          if (live) {
#pragma unroll
            for (int u = 0; u < 4; ++u)
              if (u < n) sh.c[r[u]][col] = fmaf(a[u], b, c[u]);
          }
        }
      }
    }
    mine = mine_n;
    any = any_n;
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  __syncthreads();
  // ---- C tile back
  for (int e = tid; e < kCsTM * (kCsTN / 4); e += kCsThreads) {
    const int r = e / (kCsTN / 4), q = e % (kCsTN / 4);
    const int64_t row = m0 + r, colg = n0 + 4 * q;
    if (row >= M || colg >= N) continue;
    const float4 v = *reinterpret_cast<const float4*>(&sh.c[r][4 * q]);
    if (colg + 4 <= N) *reinterpret_cast<float4*>(C + row * ldc + colg) = v;
    else {
      const float t[4] = {v.x, v.y, v.z, v.w};
      for (int u = 0; u < 4 && colg + u < N; ++u) C[row * ldc + colg + u] = t[u];
    }
  }
  __syncthreads();  // the next unit reuses the C tile and the ring
}

__device__ __forceinline__ CsShared& cs_shared() {
  extern __shared__ __align__(128) uint8_t cs_raw[];
  return *reinterpret_cast<CsShared*>(cs_raw + ((128 - ((uint32_t)__cvta_generic_to_shared(cs_raw) & 127)) & 127));
}

// Persistent over the units t = blockIdx.x, + gridDim.x, ...; sel (AUTO): runs iff *sel == 48.
__global__ void __launch_bounds__(kCsThreads, 1)
k2_csr(const float* __restrict__ AT, int64_t kpad, const float* __restrict__ B, int64_t ldb,
       const uint32_t* __restrict__ bgrp, int64_t kw, float* __restrict__ C, int64_t ldc, int64_t M, int64_t K,
       int64_t N, int64_t n_tb, int64_t n_rt, const unsigned long long* __restrict__ sel) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (sel && *sel != 48ull) return;
  CsShared& sh = cs_shared();
  for (int64_t t = blockIdx.x; t < n_tb * n_rt; t += gridDim.x)
    k2_csr_unit(sh, AT, kpad, B, ldb, bgrp, kw, C, ldc, M, K, N, t / n_tb, t % n_tb);
}

}  // namespace mmmcu
