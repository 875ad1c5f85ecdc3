// mmmcu.cu — the C ABI (include/mmmcu.h) over the sm_100a kernels K1 / K2.
//
// Host runtime of the drop-in boundary: validation with the reference's
// error semantics, a context that owns every device buffer (grow-only, reused across
// calls), the plan/version staleness contract (matrix.hpp:115), and
// stream-ordered launches.  No CPU compute path exists: without a CUDA device every entry
// point fails with MMMCU_ERR_NO_DEVICE.
#include "../../include/mmmcu.h"

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <utility>
#include <vector>

#include "gen.cuh"
#include "k1_preprocess.cuh"
#include "k2_csr.cuh"
#include "k2_simt.cuh"
#include "k2_tc.cuh"
#include "kgen.cuh"

// K1 pass ring for ordinary operand mixes: stages x CTAs per SM (measured best of 2x3, 3x2, 1x6)
#ifndef K1_SMALL_ST
#define K1_SMALL_ST (16 / K1_SR)  // 64 KB ring per CTA
#define K1_SMALL_CTAS 3
#endif
#ifndef K1_BIG_ST
#define K1_BIG_ST (48 / K1_SR)    // 192 KB ring, 1 CTA per SM
#endif

namespace {

thread_local std::string g_err;

struct DevBuf {
  void* p = nullptr;
  size_t cap = 0;
  cudaError_t ensure(size_t bytes) {
    if (bytes <= cap) return cudaSuccess;
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
    const size_t want = std::max<size_t>((bytes + 255) & ~size_t(255), 256);  // whole 16-byte words for k1_zero
    cudaError_t e = cudaMalloc(&p, want);
    if (e == cudaSuccess) cap = want;
    return e;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
  }
  template <typename T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

int64_t round_up(int64_t x, int64_t m) { return (x + m - 1) / m * m; }

}  // namespace

struct mmmcu_ctx {
  int device = 0;
  int num_sms = 0;
  cudaStream_t stream = nullptr;
  std::string err;
  mmmcu_algo algo = MMMCU_ALGO_AUTO;
  mmmcu_algo last_algo = MMMCU_ALGO_AUTO;
  bool auto_pending = false;

  // ---- A plan (preprocess_a)
  bool has_a = false;
  const float* A = nullptr;
  int64_t M = 0, Ka = 0, lda = 0;
  uint64_t av = 0;
  int csr_idx_bytes = 4;
  DevBuf abits, za, tile_prefix, row_ptr, cols;  // row_ptr + cols: K1's per-row index lists (CSR)

  // ---- B plan (preprocess_b)
  bool has_b = false;
  const float* B = nullptr;
  int64_t Kb = 0, N = 0, ldb = 0;
  uint64_t bv = 0;
  DevBuf codes, bgrp, zb;
  DevBuf ctl;

  // ---- K2 operands emitted by K1 (which ones depends on the algorithm, see ops_for)
  bool op_at = false, op_rows = false, op_tcb = false;
  bool rows_fresh = false, tcb_fresh = false;  // packed without the device gate (valid for a forced path)
  bool tcb_f16 = true;                          // format of the packed K2-TC step images (fp16 / tf32 split)
  int ops_b = 0;                                // operand sets B was staged for
  int64_t kpad = 0, m_at = 0, n_tb = 0, n_tc = 0, tc_steps = 0;
  int tc_pairs = 0;  // co-resident K2-TC CTA pairs (cudaOccupancyMaxActiveClusters), 0 = not queried
  // K1 scratch (zeroed, atomically accumulated) is double-buffered: a plan uses half p of za /
  // zb while its K1 pass zeroes the other half for the next plan, so no zeroing launch or
  // memset sits in the per-call chain.  clean[h]: half h is known to be zero.
  size_t za_half = 0, zb_half = 0;  // bytes per half
  int pa = 0, pb = 0;
  bool za_clean[2] = {false, false}, zb_clean[2] = {false, false};
  bool zero_a_next = false, zero_b_next = false;  // the coming K1 pass zeroes the other half
  DevBuf at, tcb, tck, tcn, tc_pre, brows, row_off;
  // TMA descriptor of A^T as a 2-D tensor [m_at / 128 * kpad rows][128 floats] (K2-TC gather4)
  CUtensorMap tmap_at;
  const void* tmap_at_ptr = nullptr;
  int64_t tmap_at_rows = 0;
  // TMA descriptor of C (K2-TC's tensor reduce-adds), cached by (C, ldc, M, N)
  CUtensorMap tmap_c;
  const void* tmap_c_ptr = nullptr;
  int64_t tmap_c_key[3] = {0, 0, 0};

  // ---- statistics: u64 [16] = {inv, lanes, skipped, zreg, nnzA, pop, zero_codes, span, slice_nz}
  DevBuf stats;

  // ---- host-operand staging (mmmcu_multiply_host)
  DevBuf hA, hB, hC;

  // ---- export scratch
  DevBuf scratch0, scratch1;

  // ---- lane-general / f64 plans (kgen.cuh): every (dtype, lane config) but the f32 default
  // lane, whose fused K1 / K2 path is above.  A plan built by them shares abits / row_ptr /
  // cols / tile_prefix / stats with the fast path; gen_a / gen_b say which path built it.
  bool gen_a = false, gen_b = false;
  mmmcu_dtype a_dt = MMMCU_F32, b_dt = MMMCU_F32;
  int gen_G = 8, gen_P = 8;                     // the B plan's group width and pattern bits
  const void* gA = nullptr;                     // typed operand pointers of the plan
  const void* gB = nullptr;
  DevBuf gcodes, gza, gzb;  // uint16 codes [K][ldb/R]; A scratch arow | tile_sum | acol; B scratch bpop | bnz
};

namespace {

mmmcu_status fail(mmmcu_ctx* ctx, mmmcu_status st, const std::string& msg) {
  if (ctx) ctx->err = msg;
  g_err = msg;
  return st;
}

#define MMMCU_CUDA(call)                                                                        \
  do {                                                                                          \
    cudaError_t e_ = (call);                                                                    \
    if (e_ != cudaSuccess) return fail(ctx, MMMCU_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
  } while (0)

#define MMMCU_LAUNCHED()                                                                       \
  do {                                                                                          \
    cudaError_t e_ = cudaGetLastError();                                                        \
    if (e_ != cudaSuccess) return fail(ctx, MMMCU_ERR_CUDA, std::string("kernel launch: ") + cudaGetErrorString(e_)); \
  } while (0)

#define MMMCU_TRY(expr)               \
  do {                                \
    mmmcu_status s_ = (expr);         \
    if (s_ != MMMCU_OK) return s_;    \
  } while (0)

// Launch with programmatic stream serialization (PDL): the kernel's CTAs may be scheduled
// before the previous kernel in the stream completes; the kernel waits for it in
// griddepcontrol.wait (tc::pdl_wait) before reading its outputs.  Used for the kernels that
// follow another kernel of the call chain (CSR, packs, K2).
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k, std::forward<Args>(args)...);
}

// Every kernel of the per-call chain asks for the maximum shared-memory carveout, so that
// consecutive kernels (K1 pass: 3 x 66 KB per SM, K2-TC: 210 KB, packs / CSR: small) never
// make the SMs drain and reconfigure L1 / shared memory between launches.
template <typename F>
void max_carveout(F* f) {
  cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout, (int)cudaSharedmemCarveoutMaxShared);
}
void set_carveouts(int device) {
  static bool done[64] = {false};
  if (device < 0 || device >= 64 || done[device]) return;
  done[device] = true;
  max_carveout(mmmcu::k1_pass<K1_SMALL_ST, K1_SMALL_CTAS>);
  max_carveout(mmmcu::k1_pass<K1_BIG_ST, 1>);
  max_carveout(mmmcu::k1_pack_auto);
  max_carveout(mmmcu::k1_csr);
  max_carveout(mmmcu::k1_pack_tc);
  max_carveout(mmmcu::k1_pack_rows);
  max_carveout(mmmcu::k1_row_off);
  max_carveout(mmmcu::k2_simt2_any);
  max_carveout(mmmcu::k2_csr);
  max_carveout(mmmcu::k2_simt2<8>);
  max_carveout(mmmcu::k2_simt2<16>);
  max_carveout(mmmcu::k2_tc<true>);
  max_carveout(mmmcu::k2_tc<false>);
  cudaGetLastError();  // attribute hints only
}

mmmcu_status bind(mmmcu_ctx* ctx) {
  if (!ctx) return fail(nullptr, MMMCU_ERR_INVALID_ARG, "null context");
  MMMCU_CUDA(cudaSetDevice(ctx->device));
  set_carveouts(ctx->device);
  return MMMCU_OK;
}

// KernelTable<T>::build (kernel_table.cpp:64-72) + Matrix ctor lane checks (matrix.hpp:73-74),
// with the reference's messages (dtype_name: "f32" / "f64").
mmmcu_status validate_lane(mmmcu_ctx* ctx, mmmcu_lane lane, mmmcu_dtype dt) {
  if (dt != MMMCU_F32 && dt != MMMCU_F64) return fail(ctx, MMMCU_ERR_UNSUPPORTED, "unknown dtype");
  if (lane.w <= 0 || lane.p <= 0 || lane.v <= 0)
    return fail(ctx, MMMCU_ERR_INVALID_ARG, "lane config fields must be positive");
  if (lane.p < 1 || lane.p > 16)
    return fail(ctx, MMMCU_ERR_INVALID_ARG, "pattern size must lie in [1, 16], got " + std::to_string(lane.p));
  const int g = lane.w * lane.v;
  if (g != 1 && g != 2 && g != 4 && g != 8 && g != 16 && g != 32 && g != 64)
    return fail(ctx, MMMCU_ERR_INVALID_ARG, "unsupported lane configuration: group width " + std::to_string(g) +
                                                " for " + (dt == MMMCU_F64 ? "f64" : "f32"));
  return MMMCU_OK;
}
mmmcu_status check_lane(mmmcu_ctx* ctx, mmmcu_lane lane) { return validate_lane(ctx, lane, MMMCU_F32); }
// the fused K1 / K2 kernels: f32 with the default lane config {W=8, P=8, V=1}
bool fast_lane(mmmcu_lane lane, mmmcu_dtype dt) { return dt == MMMCU_F32 && lane.w == 8 && lane.p == 8 && lane.v == 1; }

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// Zeroed scratch of the fused K1 launch: za = [arow M | acol K], zb = [slice_nz u64 |
// bpop K | bnz K]; ctl = the last-block counter, which the last block resets itself.
// (the per-row fp16 range words first: 8-byte aligned)
uint8_t* za_base(mmmcu_ctx* ctx) { return ctx->za.as<uint8_t>() + ctx->pa * ctx->za_half; }
uint8_t* zb_base(mmmcu_ctx* ctx) { return ctx->zb.as<uint8_t>() + ctx->pb * ctx->zb_half; }
unsigned long long* za_rrng(mmmcu_ctx* ctx) { return reinterpret_cast<unsigned long long*>(za_base(ctx)); }
uint32_t* za_arow(mmmcu_ctx* ctx) { return reinterpret_cast<uint32_t*>(za_rrng(ctx) + ctx->M); }
uint32_t* za_acol(mmmcu_ctx* ctx) { return za_arow(ctx) + ctx->M; }
uint32_t* za_tiles(mmmcu_ctx* ctx) { return za_acol(ctx) + ctx->Ka; }
int64_t n_row_tiles(int64_t M) { return (M + mmmcu::kK1Rows - 1) / mmmcu::kK1Rows; }
unsigned long long* zb_slice(mmmcu_ctx* ctx) { return reinterpret_cast<unsigned long long*>(zb_base(ctx)); }
uint32_t* zb_bpop(mmmcu_ctx* ctx) {  // after the head and the group range words (zb_grng)
  return reinterpret_cast<uint32_t*>(zb_slice(ctx) + 6) + 2 * (ctx->ldb / 8);
}
// one word after the A scratch: set iff A holds an Inf / NaN (zeroed with za)
uint32_t* za_nonfinite(mmmcu_ctx* ctx) { return za_tiles(ctx) + n_row_tiles(ctx->M); }
uint32_t* za_wide(mmmcu_ctx* ctx) { return za_nonfinite(ctx) + 1; }  // fp16-split range flag
int64_t za_words(int64_t M, int64_t K) { return 2 * M + M + K + n_row_tiles(M) + 1 + 1; }
// zb starts with 6 u64 B totals (k1_preprocess.cuh K1Scratch::btot), then per-8-column-group
// max|b| bits and min-complements, then bpop [K], bnz [K], ...
constexpr int kZbHead = 6;
unsigned long long* zb_grng(mmmcu_ctx* ctx) { return zb_slice(ctx) + kZbHead; }
uint32_t* zb_bnz(mmmcu_ctx* ctx) { return zb_bpop(ctx) + ctx->Kb; }
// Operand sets K1 emits for K2: A^T tiles (SIMT v2, TC), raw B rows (SIMT v2), tf32 B step
// images + live-k lists (TC).
enum { OP_AT = 1, OP_ROWS = 2, OP_TCB = 4 };
int ops_for(const mmmcu_ctx* ctx) {
  switch (ctx->algo) {
    case MMMCU_ALGO_AUTO: return OP_AT | OP_ROWS | OP_TCB;  // K1's last CTA picks (k1_choose_path)
    case MMMCU_ALGO_TC:
    case MMMCU_ALGO_TC32: return OP_AT | OP_TCB;
    case MMMCU_ALGO_DENSE: return 0;
    case MMMCU_ALGO_CSR: return OP_AT;  // A^T + the group masks; B is read as is
    default: return OP_AT | OP_ROWS;
  }
}
uint32_t* zb_tlive(mmmcu_ctx* ctx) { return zb_bnz(ctx) + ctx->Kb; }
int64_t n_cnt_tc(const mmmcu_ctx* ctx) { return ctx->n_tc * ((ctx->Kb + 31) / 32); }
// after the TC live-k words: the K2-SIMT record counts
uint32_t* zb_row_cnt(mmmcu_ctx* ctx) {
  return zb_tlive(ctx) + ((ctx->ops_b & OP_TCB) ? n_cnt_tc(ctx) : 0);
}

// Switch a double-buffered K1 scratch to its other half (zeroed by the previous K1 pass), or
// (re)allocate both halves zeroed when the size changes.  A half that is not known to be
// clean (the pass that should have zeroed it never ran) is zeroed here.
mmmcu_status next_half(mmmcu_ctx* ctx, DevBuf& buf, size_t& half, int& p, bool (&clean)[2], size_t bytes) {
  const size_t want = (bytes + 255) & ~size_t(255);
  if (want > half || !buf.p) {
    MMMCU_CUDA(buf.ensure(2 * want));
    half = want;
    MMMCU_CUDA(cudaMemsetAsync(buf.p, 0, 2 * want, ctx->stream));
    clean[0] = clean[1] = true;
    p = 0;
  } else {
    p ^= 1;
    if (!clean[p]) MMMCU_CUDA(cudaMemsetAsync(static_cast<uint8_t*>(buf.p) + p * half, 0, half, ctx->stream));
  }
  clean[p] = false;  // the coming K1 pass accumulates into it
  return MMMCU_OK;
}

mmmcu_status stage_a(mmmcu_ctx* ctx, const float* A, int64_t M, int64_t K, int64_t lda, uint64_t av) {
  if (M <= 0 || K <= 0) return fail(ctx, MMMCU_ERR_INVALID_ARG, "matrix dimensions must be positive");
  if (!A) return fail(ctx, MMMCU_ERR_INVALID_ARG, "A is null");
  if (lda < K || lda % 4 != 0 || !aligned16(A))
    return fail(ctx, MMMCU_ERR_INVALID_ARG, "A must be 16-byte aligned with lda >= K and lda % 4 == 0");
  const int64_t kw = (K + 31) / 32;
  ctx->has_a = false;
  ctx->gen_a = false;
  ctx->a_dt = MMMCU_F32;
  ctx->csr_idx_bytes = K <= 65536 ? 2 : 4;
  MMMCU_CUDA(ctx->abits.ensure(sizeof(uint32_t) * M * kw));
  MMMCU_TRY(next_half(ctx, ctx->za, ctx->za_half, ctx->pa, ctx->za_clean, sizeof(uint32_t) * za_words(M, K)));
  MMMCU_CUDA(ctx->tile_prefix.ensure(sizeof(int64_t) * (n_row_tiles(M) + 1)));
  MMMCU_CUDA(ctx->row_ptr.ensure(sizeof(int64_t) * (M + 1)));
  MMMCU_CUDA(ctx->cols.ensure((size_t)ctx->csr_idx_bytes * M * K));
  ctx->zero_a_next = true;
  ctx->op_at = false;
  if (ops_for(ctx) & OP_AT) {
    ctx->kpad = round_up(K, 32);
    ctx->m_at = round_up(M, 256);  // K2-TC pairs take row tiles two at a time
    MMMCU_CUDA(ctx->at.ensure(sizeof(float) * ctx->m_at * ctx->kpad));
  }
  ctx->A = A;
  ctx->M = M;
  ctx->Ka = K;
  ctx->lda = lda;
  ctx->av = av;
  return MMMCU_OK;
}

mmmcu_status stage_b(mmmcu_ctx* ctx, const float* B, int64_t K, int64_t N, int64_t ldb, uint64_t bv) {
  if (K <= 0 || N <= 0) return fail(ctx, MMMCU_ERR_INVALID_ARG, "matrix dimensions must be positive");
  if (!B) return fail(ctx, MMMCU_ERR_INVALID_ARG, "B is null");
  if (ldb < N || ldb % 64 != 0 || !aligned16(B))
    return fail(ctx, MMMCU_ERR_INVALID_ARG,
                "B must be 16-byte aligned with ldb >= N and ldb a multiple of the region width 64");
  const int64_t kw = (K + 31) / 32;
  const int64_t nreg = ldb / 64, ngrp = ldb / 8;
  ctx->has_b = false;
  ctx->gen_b = false;
  ctx->b_dt = MMMCU_F32;
  ctx->ldb = ldb;  // the zb_* scratch offsets depend on it
  ctx->Kb = K;
  MMMCU_CUDA(ctx->codes.ensure((size_t)K * nreg));
  MMMCU_CUDA(ctx->bgrp.ensure(sizeof(uint32_t) * ngrp * kw));
  ctx->op_rows = ctx->op_tcb = false;
  ctx->rows_fresh = ctx->tcb_fresh = false;
  const int ops = ops_for(ctx);
  ctx->ops_b = ops;
  const int64_t n_tb = (ldb + 255) / 256;
  const int64_t n_cnt = n_tb * kw;
  const int64_t n_tc = (ldb + mmmcu::kTcTileN - 1) / mmmcu::kTcTileN;
  const int64_t n_extra = ((ops & OP_TCB) ? n_tc * kw + n_tc : 0) + ((ops & OP_ROWS) ? n_cnt : 0);
  const size_t zb_bytes = kZbHead * sizeof(unsigned long long) + sizeof(uint32_t) * (2 * (ldb / 8) + 2 * K + n_extra);
  MMMCU_TRY(next_half(ctx, ctx->zb, ctx->zb_half, ctx->pb, ctx->zb_clean, zb_bytes));
  ctx->zero_b_next = true;
  ctx->n_tb = n_tb;
  ctx->n_tc = n_tc;
  if (ops & OP_TCB) {
    // worst case every k live in every tile: kw*4 steps of 12 KB per tile = 2x B's bytes
    ctx->tc_steps = kw * 4;
    MMMCU_CUDA(ctx->tcb.ensure((size_t)n_tc * ctx->tc_steps * mmmcu::kTdStepFloats * 4));
    MMMCU_CUDA(ctx->tck.ensure(sizeof(int32_t) * n_tc * ctx->tc_steps * 8));
    MMMCU_CUDA(ctx->tcn.ensure(sizeof(int32_t) * n_tc));
    MMMCU_CUDA(ctx->tc_pre.ensure(sizeof(int64_t) * (n_tc + 1)));
  }
  if (ops & OP_ROWS) {
    // worst case 3 header + 16 x 32 rows of 64 B per (tile, chunk): ~B's bytes
    MMMCU_CUDA(ctx->row_off.ensure(sizeof(int64_t) * (n_cnt + 1)));
    MMMCU_CUDA(ctx->brows.ensure((size_t)n_cnt * (3 + 16 * 32) * 64));
  }
  ctx->B = B;
  ctx->Kb = K;
  ctx->N = N;
  ctx->ldb = ldb;
  ctx->bv = bv;
  return MMMCU_OK;
}

// B operand packs for K2: K2-SIMT rows, K2-TC step images, or (AUTO) both in one launch
// gated on the device by the path choice.
mmmcu::PackRowsArgs rows_args(mmmcu_ctx* ctx) {
  return mmmcu::PackRowsArgs{ctx->B, ctx->ldb, ctx->bgrp.as<uint32_t>(), (ctx->Kb + 31) / 32,
                             ctx->row_off.as<int64_t>(), ctx->brows.as<uint4>()};
}
mmmcu::PackTcArgs tc_args(mmmcu_ctx* ctx, bool f16) {
  return mmmcu::PackTcArgs{ctx->B, ctx->ldb, zb_tlive(ctx), (ctx->Kb + 31) / 32, ctx->tc_steps,
                           ctx->tcb.as<float>(), ctx->tck.as<int32_t>(), ctx->tcn.as<int32_t>(), f16 ? 1 : 0,
                           zb_grng(ctx)};
}
// AUTO and MMMCU_ALGO_TC use the fp16 split, MMMCU_ALGO_TC32 the tf32 split
bool tc_f16(const mmmcu_ctx* ctx) { return ctx->algo != MMMCU_ALGO_TC32; }
// most step images a tile can need: every k live, 16 (fp16) or 8 (tf32) per step
int64_t pack_steps(const mmmcu_ctx* ctx, bool f16) { return f16 ? (ctx->tc_steps + 1) / 2 : ctx->tc_steps; }
int pack_tc_smem(mmmcu_ctx* ctx) { return (int)(sizeof(uint32_t) * (2 * ((ctx->Kb + 31) / 32) + 1)); }

mmmcu_status pack_rows(mmmcu_ctx* ctx) {
  dim3 grid((unsigned)((ctx->Kb + 31) / 32), (unsigned)ctx->n_tb);
  mmmcu::k1_pack_rows<<<grid, mmmcu::kPackThreads, 0, ctx->stream>>>(rows_args(ctx));
  MMMCU_LAUNCHED();
  return MMMCU_OK;
}

mmmcu_status pack_tc(mmmcu_ctx* ctx) {
  const bool f16 = tc_f16(ctx);
  const int smem = pack_tc_smem(ctx);
  if (smem > 200 * 1024) return fail(ctx, MMMCU_ERR_UNSUPPORTED, "K too large for the TC packer");
  MMMCU_CUDA(cudaFuncSetAttribute(mmmcu::k1_pack_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  dim3 grid((unsigned)((pack_steps(ctx, f16) + mmmcu::kPtSteps - 1) / mmmcu::kPtSteps), (unsigned)ctx->n_tc);
  mmmcu::k1_pack_tc<<<grid, mmmcu::kPtThreads, smem, ctx->stream>>>(tc_args(ctx, f16));
  MMMCU_LAUNCHED();
  ctx->tcb_f16 = f16;
  return MMMCU_OK;
}

mmmcu::CsrArgs csr_args(mmmcu_ctx* ctx) {
  return mmmcu::CsrArgs{ctx->abits.as<uint32_t>(), za_arow(ctx), ctx->tile_prefix.as<int64_t>(), ctx->M,
                        (ctx->Ka + 31) / 32, ctx->row_ptr.as<int64_t>(), ctx->cols.p, ctx->csr_idx_bytes};
}
int64_t csr_ctas(const mmmcu_ctx* ctx) { return (ctx->M + mmmcu::kCsrRows - 1) / mmmcu::kCsrRows; }

mmmcu_status pack_auto(mmmcu_ctx* ctx, const unsigned long long* sel, bool with_csr) {
  const int smem = pack_tc_smem(ctx);
  if (smem > 200 * 1024) return fail(ctx, MMMCU_ERR_UNSUPPORTED, "K too large for the TC packer");
  const int64_t rows_x = (ctx->Kb + 31) / 32, n_rows = rows_x * ctx->n_tb;
  const int64_t tc_x = (pack_steps(ctx, true) + mmmcu::kPtSteps - 1) / mmmcu::kPtSteps, n_tc = tc_x * ctx->n_tc;
  const int64_t n_csr = with_csr ? csr_ctas(ctx) : 0;  // A's CSR CTAs ride in this launch
  const int smem_all = with_csr ? std::max(smem, mmmcu::k1_csr_smem(ctx->csr_idx_bytes)) : smem;
  if (n_rows + n_tc + n_csr > 0x7fffffff) return fail(ctx, MMMCU_ERR_UNSUPPORTED, "B too large for one pack launch");
  MMMCU_CUDA(cudaFuncSetAttribute(mmmcu::k1_pack_auto, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_all));
  // persistent: 4 CTAs per SM (the register-limited residency) walk the items of the chosen
  // pack and the CSR
  const int64_t items = std::max(n_rows, n_tc) + n_csr;
  const int64_t grid = std::max<int64_t>(1, std::min<int64_t>(items, 4 * (int64_t)ctx->num_sms));
  MMMCU_CUDA(launch_pdl(mmmcu::k1_pack_auto, dim3((unsigned)grid), dim3(mmmcu::kPtThreads), smem_all, ctx->stream,
                        rows_args(ctx), rows_x, n_rows, tc_args(ctx, true), tc_x, n_tc, sel, csr_args(ctx), n_csr,
                        (const int64_t*)ctx->tc_pre.as<int64_t>(), ctx->n_tc, ctx->ctl.as<unsigned int>() + 2));
  MMMCU_LAUNCHED();
  ctx->tcb_f16 = true;
  return MMMCU_OK;
}

// One fused K1 launch over the staged operand(s), then (for A) the CSR index lists.
mmmcu_status launch_k1(mmmcu_ctx* ctx, bool do_a, bool do_b) {
  MMMCU_CUDA(ctx->stats.ensure(sizeof(unsigned long long) * 24));
  if (ctx->ctl.cap == 0) {
    MMMCU_CUDA(ctx->ctl.ensure(256));
    MMMCU_CUDA(cudaMemsetAsync(ctx->ctl.p, 0, 256, ctx->stream));
  }
  const bool a_valid = do_a || ctx->has_a;
  const bool b_valid = do_b || ctx->has_b;
  const bool same_k = a_valid && b_valid && ctx->Ka == ctx->Kb;
  const int64_t K = do_a ? ctx->Ka : ctx->Kb;
  const int64_t kw = (K + 31) / 32;
  const int ops = ops_for(ctx);
  // AUTO builds both K2 operand sets, each pack gated on the device by the path choice; a
  // later A-only preprocess may flip the choice, so the gated packs re-run whenever B is valid
  const int ops_b = b_valid ? ctx->ops_b : 0;
  const bool gate = (ops & OP_ROWS) && (ops & OP_TCB) && (ops_b & OP_ROWS) && (ops_b & OP_TCB);
  const bool tc_a = do_a && (ops & OP_AT);
  const bool tcb_b = (ops_b & OP_TCB) && (do_b || gate);
  const bool rows_b = (ops_b & OP_ROWS) && (do_b || gate);
  const unsigned long long* sel = gate ? ctx->stats.as<unsigned long long>() + 7 : nullptr;
  const int64_t a_tx = (ctx->Ka + mmmcu::kK1Cols - 1) / mmmcu::kK1Cols;
  const int64_t a_rows = tc_a ? ctx->m_at : ctx->M;  // A^T tiles are written to the 256-row boundary
  const int64_t nA = do_a ? a_tx * ((a_rows + mmmcu::kK1Rows - 1) / mmmcu::kK1Rows) : 0;
  const int64_t b_tx = (ctx->ldb + mmmcu::kK1Cols - 1) / mmmcu::kK1Cols;
  const int64_t nB = do_b ? b_tx * ((ctx->Kb + 31) / 32) : 0;
  if (nA + nB > 0x7fffffff) return fail(ctx, MMMCU_ERR_UNSUPPORTED, "operand too large for one K1 launch");
  mmmcu::K1Scratch z;
  z.arow = a_valid ? za_arow(ctx) : nullptr;
  z.acol = a_valid ? za_acol(ctx) : nullptr;
  z.tile_sum = do_a ? za_tiles(ctx) : nullptr;
  z.nonfinite_a = a_valid ? za_nonfinite(ctx) : nullptr;
  z.tile_prefix = do_a ? ctx->tile_prefix.as<int64_t>() : nullptr;
  z.bpop = b_valid ? zb_bpop(ctx) : nullptr;
  z.bnz = b_valid ? zb_bnz(ctx) : nullptr;
  z.btot = b_valid ? zb_slice(ctx) : ctx->stats.as<unsigned long long>() + 16;
  z.rrng = a_valid ? za_rrng(ctx) : nullptr;
  z.grng = b_valid ? zb_grng(ctx) : nullptr;
  z.ngrp = b_valid ? ctx->ldb / 8 : 0;
  z.wide_a = a_valid ? za_wide(ctx) : nullptr;
  z.done = ctx->ctl.as<unsigned int>();
  z.next_tile = ctx->ctl.as<unsigned int>() + 1;
  z.at = tc_a ? ctx->at.as<float>() : nullptr;
  z.kpad = ctx->kpad;
  z.m_at = ctx->m_at;
  z.tlive = tcb_b ? zb_tlive(ctx) : nullptr;
  z.row_cnt = rows_b ? zb_row_cnt(ctx) : nullptr;
  z.row_off = rows_b ? ctx->row_off.as<int64_t>() : nullptr;
  z.n_tb = ctx->n_tb;
  z.n_tc = ctx->n_tc;
  z.tc_pre = (gate && tcb_b) ? ctx->tc_pre.as<int64_t>() : nullptr;
  z.tcn = (gate && tcb_b) ? ctx->tcn.as<int32_t>() : nullptr;
  z.choose = gate ? 1 : 0;
  if (ctx->num_sms == 0) MMMCU_CUDA(cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, ctx->device));
  z.num_sms = ctx->num_sms;
  z.K = K;
  const int has_a = a_valid && (same_k || !b_valid) ? 1 : 0;
  const int has_b = b_valid && (same_k || !a_valid) ? 1 : 0;
  if (ctx->num_sms == 0) MMMCU_CUDA(cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, ctx->device));
  const mmmcu::K1Args g{ctx->A, ctx->M, K, ctx->lda, ctx->abits.as<uint32_t>(), a_tx, nA,
                        ctx->B, ctx->ldb, ctx->ldb / 64, ctx->bgrp.as<uint32_t>(), b_tx, nB, kw};
  // ring shape: 2 stages x 3 CTAs per SM in general (the sweep's 1024 tiles: 121 vs 134 us;
  // cfg5's A-heavy 10k tiles: 0.86 vs 1.02 ms), 6 stages x 1 CTA for streams dominated by
  // many B tiles, which carry no A^T work (cfg4's 18k B tiles: 1.26 vs 1.82 ms) — measured
  const bool big = nA + nB > 4 * 3 * (int64_t)ctx->num_sms && nB > 4 * nA;
  auto k1fn = big ? mmmcu::k1_pass<K1_BIG_ST, 1> : mmmcu::k1_pass<K1_SMALL_ST, K1_SMALL_CTAS>;
  const int k1_smem = (int)(big ? sizeof(mmmcu::K1RingT<K1_BIG_ST>) : sizeof(mmmcu::K1RingT<K1_SMALL_ST>)) + 128;
  MMMCU_CUDA(cudaFuncSetAttribute(k1fn, cudaFuncAttributeMaxDynamicSharedMemorySize, k1_smem));
  const unsigned k1_grid =
      (unsigned)std::min<int64_t>(nA + nB, (big ? 1 : K1_SMALL_CTAS) * (int64_t)ctx->num_sms);
#ifdef K1_EVT
  cudaEvent_t ev0, ev1;
  cudaEventCreate(&ev0);
  cudaEventCreate(&ev1);
  cudaEventRecord(ev0, ctx->stream);
#endif
  // the K1 pass zeroes the other halves of the scratch for the next plan (double buffering)
  z.zero_a = ctx->zero_a_next ? reinterpret_cast<uint4*>(ctx->za.as<uint8_t>() + (ctx->pa ^ 1) * ctx->za_half) : nullptr;
  z.zero_a_n = ctx->zero_a_next ? (int64_t)(ctx->za_half / 16) : 0;
  z.zero_b = ctx->zero_b_next ? reinterpret_cast<uint4*>(ctx->zb.as<uint8_t>() + (ctx->pb ^ 1) * ctx->zb_half) : nullptr;
  z.zero_b_n = ctx->zero_b_next ? (int64_t)(ctx->zb_half / 16) : 0;
  MMMCU_CUDA(launch_pdl(k1fn, dim3(k1_grid), dim3(mmmcu::kK1Block), k1_smem, ctx->stream, g, z));
  MMMCU_LAUNCHED();
  // the finalize (plan totals, fp16 range guard, AUTO path choice, CSR tile prefix, K2-SIMT
  // record offsets): one CTA, programmatically serialized behind the pass
  const mmmcu::K1FinArgs fa{ctx->M, K, ctx->ldb / 64, kw, nA, nB, has_a, has_b};
  MMMCU_CUDA(cudaFuncSetAttribute(mmmcu::k1_fin, cudaFuncAttributeMaxDynamicSharedMemorySize, mmmcu::k1_fin_smem()));
  MMMCU_CUDA(launch_pdl(mmmcu::k1_fin, dim3(1), dim3(32 * mmmcu::kFinWarps), mmmcu::k1_fin_smem(), ctx->stream, z, fa,
                        ctx->stats.as<unsigned long long>()));
  if (ctx->zero_a_next) ctx->za_clean[ctx->pa ^ 1] = true;
  if (ctx->zero_b_next) ctx->zb_clean[ctx->pb ^ 1] = true;
  ctx->zero_a_next = ctx->zero_b_next = false;
#ifdef K1_EVT
  cudaEventRecord(ev1, ctx->stream);
  cudaEventSynchronize(ev1);
  float ms = 0;
  cudaEventElapsedTime(&ms, ev0, ev1);
  fprintf(stderr, "K1_EVT k1_pass %.1f us (grid %u, smem %d)\n", ms * 1e3, k1_grid, k1_smem);
#endif
#ifdef K1_PROF
  {
    static unsigned long long* dbuf = nullptr;
    if (!dbuf) cudaMalloc(&dbuf, 8 * 4 * 4096);
    cudaDeviceSynchronize();
    cudaMemset(dbuf, 0, 8 * 4 * 4096);
    cudaMemcpyToSymbol(mmmcu::k1_prof, &dbuf, sizeof(dbuf));
    // rerun (idempotent outputs; counters are re-zeroed by the caller's memsets only once, so
    // use the stamps, not the counters)
    k1fn<<<k1_grid, mmmcu::kK1Block, k1_smem, ctx->stream>>>(g, z);
    cudaDeviceSynchronize();
    cudaMemset(ctx->ctl.as<unsigned int>() + 1, 0, sizeof(unsigned int));  // the rerun's tile counter
    std::vector<unsigned long long> h(4 * k1_grid);
    cudaMemcpy(h.data(), dbuf, 8 * 4 * k1_grid, cudaMemcpyDeviceToHost);
    unsigned long long t0 = ~0ull, t1 = 0, tmax_start = 0;
    double dsum = 0;
    for (unsigned i = 0; i < k1_grid; ++i) {
      t0 = std::min(t0, h[4 * i]);
      tmax_start = std::max(tmax_start, h[4 * i]);
      t1 = std::max(t1, h[4 * i + 1]);
      dsum += (double)(h[4 * i + 1] - h[4 * i]);
    }
    unsigned long long fp[8];
    cudaMemcpyFromSymbol(fp, mmmcu::k1_fin_prof, sizeof(fp));
    fprintf(stderr, "K1_PROF k1_fin phases (us): setup %.2f | parallel part %.2f | thread-0 choice %.2f | row_off %.2f\n",
            (fp[1] - fp[0]) / 1e3, (fp[2] - fp[1]) / 1e3, (fp[3] - fp[2]) / 1e3, (fp[4] - fp[3]) / 1e3);
    fprintf(stderr, "K1_PROF: grid %u, CTA start spread %.1f us, tiles done by %.1f us (mean CTA %.1f us)\n", k1_grid,
            (tmax_start - t0) / 1e3, (t1 - t0) / 1e3, dsum / k1_grid / 1e3);
    void* zp = nullptr;
    cudaMemcpyToSymbol(mmmcu::k1_prof, &zp, sizeof(zp));
  }
#endif
#ifdef K1_CSR_SEPARATE
  const bool csr_alone = do_a;
#else
  const bool csr_alone = do_a && !gate;
#endif
  if (csr_alone) {  // A's CSR index lists on their own (in AUTO they ride in the pack launch)
    const int csmem = mmmcu::k1_csr_smem(ctx->csr_idx_bytes);
    MMMCU_CUDA(cudaFuncSetAttribute(mmmcu::k1_csr, cudaFuncAttributeMaxDynamicSharedMemorySize, csmem));
    MMMCU_CUDA(launch_pdl(mmmcu::k1_csr, dim3((unsigned)csr_ctas(ctx)), dim3(256), csmem, ctx->stream, csr_args(ctx)));
    MMMCU_LAUNCHED();
  }
  if (gate) {
    MMMCU_TRY(pack_auto(ctx, sel, do_a && !csr_alone));
    ctx->rows_fresh = ctx->tcb_fresh = false;
  } else {
    if (rows_b) {
      MMMCU_TRY(pack_rows(ctx));
      ctx->rows_fresh = true;
    }
    if (tcb_b) {
      MMMCU_TRY(pack_tc(ctx));
      ctx->tcb_fresh = true;
    }
  }
  if (do_a) {
    ctx->has_a = true;
    ctx->op_at = tc_a;
  }
  if (do_b) ctx->has_b = true;
  if (do_b || gate) {
    ctx->op_tcb = tcb_b;
    ctx->op_rows = rows_b;
  }
  return MMMCU_OK;
}

mmmcu_status check_plan(mmmcu_ctx* ctx, const float* A, const float* B, uint64_t av, uint64_t bv) {
  if (!ctx->has_a || !ctx->has_b)
    return fail(ctx, MMMCU_ERR_NOT_READY, "multiply called before preprocess_a/preprocess_b");
  if (ctx->Ka != ctx->Kb)
    return fail(ctx, MMMCU_ERR_DIM_MISMATCH, "a.cols != b.rows (" + std::to_string(ctx->Ka) + " vs " +
                                                  std::to_string(ctx->Kb) + ")");
  if (A != ctx->A || B != ctx->B || av != ctx->av || bv != ctx->bv)
    return fail(ctx, MMMCU_ERR_STALE, "stale context: operands differ from the preprocessed ones");
  return MMMCU_OK;
}

// K2-CSR, persistent over the 128 x 128 units (sel: AUTO's device-side choice, nullptr = forced).
mmmcu_status launch_csr(mmmcu_ctx* ctx, float* C, int64_t ldc, const unsigned long long* sel) {
  const int64_t n_rt = (ctx->M + 127) / 128, n_tb = (round_up(ctx->N, 64) + mmmcu::kCsTN - 1) / mmmcu::kCsTN;
  if (ctx->num_sms == 0) MMMCU_CUDA(cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, ctx->device));
  MMMCU_CUDA(cudaFuncSetAttribute(mmmcu::k2_csr, cudaFuncAttributeMaxDynamicSharedMemorySize, mmmcu::kCsSmem));
  MMMCU_CUDA(launch_pdl(mmmcu::k2_csr, dim3((unsigned)std::min<int64_t>(n_rt * n_tb, ctx->num_sms)),
                        dim3(mmmcu::kCsThreads), mmmcu::kCsSmem, ctx->stream, (const float*)ctx->at.as<float>(),
                        ctx->kpad, ctx->B, ctx->ldb, (const uint32_t*)ctx->bgrp.as<uint32_t>(), (ctx->Ka + 31) / 32, C,
                        ldc, ctx->M, ctx->Ka, ctx->N, n_tb, n_rt, sel));
  MMMCU_LAUNCHED();
  return MMMCU_OK;
}

// span_hint 8 / 16 forces a variant; 0 launches both and lets k1_finalize's device-side
// choice (stats[7]) gate them, so AUTO never synchronises the stream between K1 and K2.
mmmcu_status launch_simt(mmmcu_ctx* ctx, float* C, int64_t ldc, int span_hint, int sel_slot) {
  const int64_t M = ctx->M, K = ctx->Ka, Np = round_up(ctx->N, 64);
  const int64_t kw = (K + 31) / 32;
  const unsigned long long* sel2 = span_hint == 0 ? ctx->stats.as<unsigned long long>() + sel_slot : nullptr;
  if (ctx->op_at && ctx->op_rows) {
    const int smem = mmmcu::kS2SmemBase + (int)(sizeof(int64_t) * (kw + 1));
    if (smem > 232448) return fail(ctx, MMMCU_ERR_UNSUPPORTED, "K too large for the SIMT v2 kernel");
    const int64_t row_tiles = (M + 127) / 128;  // not m_at / 128: A^T is padded to the 256-row TC pairs
    if (row_tiles > 65535) return fail(ctx, MMMCU_ERR_UNSUPPORTED, "M larger than 8388480 rows");
    dim3 grid((unsigned)((Np + 255) / 256), (unsigned)row_tiles);
    if (span_hint == 0) {  // one launch, span (or exit) chosen on the device
      MMMCU_CUDA(cudaFuncSetAttribute(mmmcu::k2_simt2_any, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      if (ctx->num_sms == 0)
        MMMCU_CUDA(cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, ctx->device));
      const int64_t ntl = (int64_t)grid.x * grid.y;
      MMMCU_CUDA(launch_pdl(mmmcu::k2_simt2_any, dim3((unsigned)std::min<int64_t>(ntl, ctx->num_sms)),
                            dim3(mmmcu::kS2Threads), smem, ctx->stream, (const float*)ctx->at.as<float>(), ctx->kpad,
                            (const float4*)ctx->brows.as<float4>(), (const int64_t*)ctx->row_off.as<int64_t>(), kw, C,
                            ldc, M, Np, sel2, (int64_t)grid.x, (int64_t)grid.y));
      MMMCU_LAUNCHED();
    }
    if (span_hint == 8) {
      MMMCU_CUDA(cudaFuncSetAttribute(mmmcu::k2_simt2<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      mmmcu::k2_simt2<8><<<grid, mmmcu::kS2Threads, smem, ctx->stream>>>(
          ctx->at.as<float>(), ctx->kpad, ctx->brows.as<float4>(), ctx->row_off.as<int64_t>(), kw, C, ldc, M, Np, sel2);
      MMMCU_LAUNCHED();
    }
    if (span_hint == 16) {
      MMMCU_CUDA(cudaFuncSetAttribute(mmmcu::k2_simt2<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      mmmcu::k2_simt2<16><<<grid, mmmcu::kS2Threads, smem, ctx->stream>>>(
          ctx->at.as<float>(), ctx->kpad, ctx->brows.as<float4>(), ctx->row_off.as<int64_t>(), kw, C, ldc, M, Np, sel2);
      MMMCU_LAUNCHED();
    }
    return MMMCU_OK;
  }
  const int64_t row_tiles = (M + mmmcu::kK2TM - 1) / mmmcu::kK2TM;
  if (row_tiles > 65535) return fail(ctx, MMMCU_ERR_UNSUPPORTED, "M larger than 8388480 rows");
  dim3 grid((unsigned)((Np + mmmcu::kK2TN - 1) / mmmcu::kK2TN), (unsigned)row_tiles);
  // (operands prepared for K2-TC only: the v1 kernel stages its own; span 8 only, because a
  // 16-column span would FMA zero groups of the slice)
  MMMCU_CUDA(cudaFuncSetAttribute(mmmcu::k2_simt_bcast<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, mmmcu::kK2Smem));
  mmmcu::k2_simt_bcast<8><<<grid, mmmcu::kK2Threads, mmmcu::kK2Smem, ctx->stream>>>(
      ctx->A, ctx->lda, ctx->B, ctx->ldb, C, ldc, M, K, Np, ctx->bgrp.as<uint32_t>(), kw, nullptr);
  MMMCU_LAUNCHED();
  return MMMCU_OK;
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no libcuda link).
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
mmmcu_status at_tensor_map(mmmcu_ctx* ctx) {
  const int64_t rows = (ctx->m_at / 128) * ctx->kpad;
  if (ctx->tmap_at_ptr == ctx->at.p && ctx->tmap_at_rows == rows) return MMMCU_OK;
  static EncodeTiledFn encode = nullptr;
  if (!encode) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    MMMCU_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
    if (!fn || q != cudaDriverEntryPointSuccess)
      return fail(ctx, MMMCU_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    encode = reinterpret_cast<EncodeTiledFn>(fn);
  }
  const cuuint64_t dims[2] = {128, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {128 * sizeof(float)};
  const cuuint32_t box[2] = {128, 1};  // gather4 moves 4 such rows
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = encode(&ctx->tmap_at, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, ctx->at.p, dims, strides, box, estr,
                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(ctx, MMMCU_ERR_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
  ctx->tmap_at_ptr = ctx->at.p;
  ctx->tmap_at_rows = rows;
  return MMMCU_OK;
}

// C as a 2-D fp32 tensor [M rows][N columns] (stride ldc), boxes of 32 x 32 with the 128-byte
// swizzle of K2-TC's staging: the accumulators' C += P by TMA tensor reduce-adds.
mmmcu_status c_tensor_map(mmmcu_ctx* ctx, float* C, int64_t ldc) {
  if (ctx->tmap_c_ptr == C && ctx->tmap_c_key[0] == ldc && ctx->tmap_c_key[1] == ctx->M && ctx->tmap_c_key[2] == ctx->N)
    return MMMCU_OK;
  EncodeTiledFn encode = nullptr;
  {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    MMMCU_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
    if (!fn || q != cudaDriverEntryPointSuccess) return fail(ctx, MMMCU_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    encode = reinterpret_cast<EncodeTiledFn>(fn);
  }
  const cuuint64_t dims[2] = {(cuuint64_t)ctx->N, (cuuint64_t)ctx->M};
  const cuuint64_t strides[1] = {(cuuint64_t)ldc * sizeof(float)};
  const cuuint32_t box[2] = {32, 32};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = encode(&ctx->tmap_c, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, C, dims, strides, box, estr,
                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                            CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(ctx, MMMCU_ERR_CUDA, "cuTensorMapEncodeTiled (C) failed (" + std::to_string((int)r) + ")");
  ctx->tmap_c_ptr = C;
  ctx->tmap_c_key[0] = ldc;
  ctx->tmap_c_key[1] = ctx->M;
  ctx->tmap_c_key[2] = ctx->N;
  return MMMCU_OK;
}

// K2-TC over the dense-tile operands (sel: device-side path choice, nullptr = forced).
template <bool F16>
mmmcu_status launch_tc_t(mmmcu_ctx* ctx, float* C, int64_t ldc, const unsigned long long* sel) {
  const int64_t row_tiles = ctx->m_at / mmmcu::kTdTM;
  MMMCU_TRY(at_tensor_map(ctx));
  MMMCU_TRY(c_tensor_map(ctx, C, ldc));
  constexpr int smem = mmmcu::td_smem<F16>();
  MMMCU_CUDA(cudaFuncSetAttribute(mmmcu::k2_tc<F16>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  if (ctx->num_sms == 0) MMMCU_CUDA(cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, ctx->device));
  cudaLaunchConfig_t cfg = {};
  cfg.blockDim = dim3(mmmcu::TdCfg<F16>::kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = ctx->stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // PDL: k2_tc starts with pdl_wait
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (F16) {  // CTA pairs: clusters of 2, a pair tile = 256 rows
    attr[1].id = cudaLaunchAttributeClusterDimension;
    attr[1].val.clusterDim.x = 2;
    attr[1].val.clusterDim.y = 1;
    attr[1].val.clusterDim.z = 1;
    cfg.numAttrs = 2;
    // persistent: exactly as many pairs as can be co-resident (a second wave of pairs would
    // double the kernel time)
    if (ctx->tc_pairs == 0) {
      cfg.gridDim = dim3(2u * (unsigned)(ctx->num_sms / 2));
      int nc = 0;
      MMMCU_CUDA(cudaOccupancyMaxActiveClusters(&nc, mmmcu::k2_tc<F16>, &cfg));
      ctx->tc_pairs = nc > 0 ? nc : 1;
      if (getenv("MMMCU_VERBOSE")) fprintf(stderr, "mmmcu: K2-TC co-resident pairs %d (SMs %d)\n", nc, ctx->num_sms);
    }
    const int64_t units = ((row_tiles + 1) / 2) * ctx->n_tc;
    // the fewest pairs that keep the number of rounds (352 units: 5 rounds on 74 or on 71 pairs):
    // the SMs left free run the K1 chain of a cell on another stream the whole K2 long
    int64_t pairs = std::min<int64_t>(units, ctx->tc_pairs);
    static const int trim = getenv("MMMCU_TC_TRIM") ? atoi(getenv("MMMCU_TC_TRIM")) : 1;  // 0: all co-resident pairs
    if (trim && pairs > 0) {
      const int64_t rounds = (units + pairs - 1) / pairs;
      pairs = (units + rounds - 1) / rounds;
    }
    cfg.gridDim = dim3(2u * (unsigned)pairs);
  } else {
    cfg.gridDim = dim3((unsigned)std::min<int64_t>(row_tiles * ctx->n_tc, ctx->num_sms));
  }
  auto launch = [&]() {
    return cudaLaunchKernelEx(&cfg, mmmcu::k2_tc<F16>, (const float*)ctx->at.as<float>(), ctx->kpad,
                              (const float*)ctx->tcb.as<float>(), (const int32_t*)ctx->tck.as<int32_t>(),
                              (const int32_t*)ctx->tcn.as<int32_t>(), (int64_t)ctx->tc_steps, C, ldc, ctx->M, ctx->N,
                              row_tiles, ctx->n_tc, sel, (const unsigned long long*)za_rrng(ctx),
                              (const unsigned long long*)zb_grng(ctx), ctx->tmap_at, ctx->tmap_c);
  };
  MMMCU_CUDA(launch());
#ifdef TD_PROF
  {  // debug builds: rerun with the per-CTA cycle counters on, print their means
    const unsigned grid = cfg.gridDim.x;
    static unsigned long long* dbuf = nullptr;
    if (!dbuf) cudaMalloc(&dbuf, 16 * 8 * 1024);  // 1024 CTAs x 16 counters; stamps from entry 4096 on
    cudaMemset(dbuf, 0, 16 * 8 * 1024);
    cudaMemcpyToSymbol(mmmcu::td_prof, &dbuf, sizeof(dbuf));
    launch();
    cudaDeviceSynchronize();
    std::vector<unsigned long long> h(16 * grid);
    cudaMemcpy(h.data(), dbuf, 8 * 16 * grid, cudaMemcpyDeviceToHost);
    {  // kernel phases from thread 0's %globaltimer stamps (ns): entry, after pdl_wait, after setup,
       // role loop done, after the final cluster sync
      std::vector<unsigned long long> st(8 * grid);
      cudaMemcpy(st.data(), dbuf + 4096, 8 * 8 * grid, cudaMemcpyDeviceToHost);
      unsigned long long t0 = ~0ull, t4 = 0;
      double d[4] = {0, 0, 0, 0};
      for (unsigned i = 0; i < grid; ++i) {
        t0 = std::min(t0, st[8 * i]);
        t4 = std::max(t4, st[8 * i + 4]);
        for (int j = 0; j < 4; ++j) d[j] += (double)(st[8 * i + j + 1] - st[8 * i + j]) / grid;
      }
      unsigned long long first_setup = ~0ull, last_setup = 0, first_done = ~0ull;
      for (unsigned i = 0; i < grid; ++i) {
        first_setup = std::min(first_setup, st[8 * i + 2]);
        last_setup = std::max(last_setup, st[8 * i + 2]);
        first_done = std::min(first_done, st[8 * i + 3]);
      }
      fprintf(stderr,
              "TD_PROF kernel span %.1f us | per CTA (mean, us): pdl_wait %.1f setup %.1f role loops %.1f final sync %.1f | "
              "setup done %.1f .. %.1f us after the first entry, first CTA done at %.1f us\n",
              (t4 - t0) / 1e3, d[0] / 1e3, d[1] / 1e3, d[2] / 1e3, d[3] / 1e3, (first_setup - t0) / 1e3,
              (last_setup - t0) / 1e3, (first_done - t0) / 1e3);
    }
    {  // pair 0: gaps between consecutive stages' MMA issue times
      std::vector<unsigned long long> ts(4096);
      cudaMemcpy(ts.data(), dbuf + 8192, 8 * 4096, cudaMemcpyDeviceToHost);
      int n = 0;
      while (n < 4096 && ts[n]) ++n;
      if (n > 2) {
        std::vector<double> g;
        for (int i = 1; i < n; ++i) g.push_back((double)(ts[i] - ts[i - 1]) / 1e3);
        std::vector<double> sorted = g;
        std::sort(sorted.begin(), sorted.end());
        fprintf(stderr, "TD_PROF pair 0: %d stages in %.1f us, gap median %.3f us; gaps > 3x median:", n,
                (double)(ts[n - 1] - ts[0]) / 1e3, sorted[sorted.size() / 2]);
        double extra = 0;
        for (size_t i = 0; i < g.size(); ++i)
          if (g[i] > 3 * sorted[sorted.size() / 2]) {
            fprintf(stderr, " [%zu: %.1f]", i + 1, g[i]);
            extra += g[i] - sorted[sorted.size() / 2];
          }
        fprintf(stderr, " (sum over the median %.1f us)\n", extra);
      }
    }
    double a[16] = {0}, b[16] = {0};
    for (unsigned i = 0; i < grid; ++i)
      for (int j = 0; j < 16; ++j) (i % 2 == 0 ? a : b)[j] += (double)h[16 * i + j] / (grid / 2);
    for (double* x : {a, b})
      fprintf(stderr,
              "TD_PROF/CTA cycles (%s): MMA wait-seg %.0f wait-tma+full %.0f (tma %.0f; first 8 stages of units %.0f) issue %.0f total %.0f | "
              "transform wait-tma %.0f work %.0f (slot wait %.0f) total %.0f | producer wait-empty %.0f total %.0f | "
              "accumulator wait-seg %.0f drain %.0f C-write %.0f total %.0f\n",
              x == a ? "even" : "odd", x[0], x[1], x[10], x[15], x[2], x[3], x[4], x[5], x[7], x[6], x[8], x[9], x[11], x[12],
              x[13], x[14]);
    void* z = nullptr;
    cudaMemcpyToSymbol(mmmcu::td_prof, &z, sizeof(z));
  }
#endif
  return MMMCU_OK;
}
mmmcu_status launch_tc(mmmcu_ctx* ctx, float* C, int64_t ldc, const unsigned long long* sel) {
  return tc_f16(ctx) ? launch_tc_t<true>(ctx, C, ldc, sel) : launch_tc_t<false>(ctx, C, ldc, sel);
}

mmmcu_status read_stats(mmmcu_ctx* ctx, unsigned long long* host16) {
  MMMCU_CUDA(cudaMemcpyAsync(host16, ctx->stats.p, sizeof(unsigned long long) * 16, cudaMemcpyDeviceToHost, ctx->stream));
  MMMCU_CUDA(cudaStreamSynchronize(ctx->stream));
  return MMMCU_OK;
}

// acol[k] = # non-zeros of A's column k, from the bitmap (k1_bitcols)
mmmcu_status launch_acol(mmmcu_ctx* ctx, uint32_t* acol) {
  const int64_t kwa = (ctx->Ka + 31) / 32;
  MMMCU_CUDA(cudaMemsetAsync(acol, 0, sizeof(uint32_t) * ctx->Ka, ctx->stream));
  const dim3 grid((unsigned)((kwa + 31) / 32), (unsigned)((ctx->M + mmmcu::kBcRows - 1) / mmmcu::kBcRows));
  mmmcu::k1_bitcols<1><<<grid, 256, 0, ctx->stream>>>(ctx->abits.as<uint32_t>(), ctx->M, kwa, ctx->Ka, acol);
  MMMCU_LAUNCHED();
  return MMMCU_OK;
}

mmmcu_status fill_counters(mmmcu_ctx* ctx, mmmcu_counters* out) {
  if (!out) return MMMCU_OK;
  // the A-dependent sums are computed on request only (k1_counters)
  const bool a_ok = ctx->has_a, b_ok = ctx->has_b;
  const bool same_k = a_ok && b_ok && ctx->Ka == ctx->Kb;
  const int64_t K = b_ok ? ctx->Kb : ctx->Ka;
  if (b_ok) {
    const int64_t ngrp = ctx->ldb / 8, kwb = (ctx->Kb + 31) / 32;
    MMMCU_CUDA(cudaMemsetAsync(zb_bpop(ctx), 0, sizeof(uint32_t) * ctx->Kb, ctx->stream));
    MMMCU_CUDA(cudaMemsetAsync(zb_bnz(ctx), 0, sizeof(uint32_t) * ctx->Kb, ctx->stream));
    const dim3 grid((unsigned)((kwb + 31) / 32), (unsigned)((ngrp + mmmcu::kBcRows - 1) / mmmcu::kBcRows));
    mmmcu::k1_bitcols<1><<<grid, 256, 0, ctx->stream>>>(ctx->bgrp.as<uint32_t>(), ngrp, kwb, ctx->Kb, zb_bpop(ctx));
    MMMCU_LAUNCHED();
    mmmcu::k1_bitcols<8><<<grid, 256, 0, ctx->stream>>>(ctx->bgrp.as<uint32_t>(), ngrp, kwb, ctx->Kb, zb_bnz(ctx));
    MMMCU_LAUNCHED();
  }
  if (a_ok) MMMCU_TRY(launch_acol(ctx, za_acol(ctx)));
  mmmcu::k1_counters<<<1, 1024, 0, ctx->stream>>>(a_ok ? za_acol(ctx) : nullptr, b_ok ? zb_bpop(ctx) : nullptr,
                                                  b_ok ? zb_bnz(ctx) : nullptr, K, ctx->M, ctx->ldb / 64,
                                                  (a_ok && (same_k || !b_ok)) ? 1 : 0, (b_ok && (same_k || !a_ok)) ? 1 : 0,
                                                  ctx->stats.as<unsigned long long>());
  MMMCU_LAUNCHED();
  unsigned long long s[16];
  MMMCU_TRY(read_stats(ctx, s));
  out->kernel_invocations = s[0];
  out->lane_fma_ops = s[1];
  out->rows_skipped = s[2];
  out->regions_skipped_by_zero_code = s[3];
  return MMMCU_OK;
}



// ----------------------------------------------------------- lane-general / f64 plans
size_t dt_size(mmmcu_dtype dt) { return dt == MMMCU_F64 ? 8 : 4; }
// the plan's operand pointers (fast path: ctx->A / ctx->B; general path: gA / gB)
const void* plan_a(const mmmcu_ctx* ctx) { return ctx->gen_a ? ctx->gA : static_cast<const void*>(ctx->A); }
const void* plan_b(const mmmcu_ctx* ctx) { return ctx->gen_b ? ctx->gB : static_cast<const void*>(ctx->B); }
int64_t gen_nreg(const mmmcu_ctx* ctx) { return ctx->ldb / ((int64_t)ctx->gen_G * ctx->gen_P); }

// preprocess_a of an f32 / f64 A on the general path: bitmap + row counts by
// kg_abits, the 32-row tile prefix, then K1's CSR kernel over the same bitmap.
template <typename T>
mmmcu_status gen_preprocess_a(mmmcu_ctx* ctx, const T* A, int64_t M, int64_t K, int64_t lda, uint64_t av,
                              mmmcu_dtype dt) {
  if (M <= 0 || K <= 0) return fail(ctx, MMMCU_ERR_INVALID_ARG, "matrix dimensions must be positive");
  if (!A) return fail(ctx, MMMCU_ERR_INVALID_ARG, "A is null");
  if (lda < K) return fail(ctx, MMMCU_ERR_DIM_MISMATCH, "lda smaller than the row");
  const int64_t kw = (K + 31) / 32, ntile = (M + mmmcu::kK1Rows - 1) / mmmcu::kK1Rows;
  ctx->has_a = false;
  ctx->csr_idx_bytes = K <= 65536 ? 2 : 4;
  MMMCU_CUDA(ctx->abits.ensure(sizeof(uint32_t) * M * kw));
  MMMCU_CUDA(ctx->gza.ensure(sizeof(uint32_t) * (M + ntile + K)));
  MMMCU_CUDA(ctx->tile_prefix.ensure(sizeof(int64_t) * (ntile + 1)));
  MMMCU_CUDA(ctx->row_ptr.ensure(sizeof(int64_t) * (M + 1)));
  MMMCU_CUDA(ctx->cols.ensure((size_t)ctx->csr_idx_bytes * M * K));
  uint32_t* arow = ctx->gza.as<uint32_t>();
  uint32_t* tsum = arow + M;
  MMMCU_CUDA(cudaMemsetAsync(arow, 0, sizeof(uint32_t) * (M + ntile), ctx->stream));
  const int64_t oct = (kw + 7) / 8;
  mmmcu::kg_abits<T><<<dim3((unsigned)oct, (unsigned)M), 256, 0, ctx->stream>>>(A, M, K, lda, ctx->abits.as<uint32_t>(),
                                                                                 kw, arow, tsum);
  MMMCU_LAUNCHED();
  mmmcu::kg_tile_prefix<<<1, 256, 0, ctx->stream>>>(tsum, ntile, ctx->tile_prefix.as<int64_t>());
  MMMCU_LAUNCHED();
  const int csmem = mmmcu::k1_csr_smem(ctx->csr_idx_bytes);
  MMMCU_CUDA(cudaFuncSetAttribute(mmmcu::k1_csr, cudaFuncAttributeMaxDynamicSharedMemorySize, csmem));
  const mmmcu::CsrArgs ca{ctx->abits.as<uint32_t>(), arow, ctx->tile_prefix.as<int64_t>(), M, kw,
                          ctx->row_ptr.as<int64_t>(), ctx->cols.p, ctx->csr_idx_bytes};
  mmmcu::k1_csr<<<(unsigned)((M + mmmcu::kCsrRows - 1) / mmmcu::kCsrRows), 256, csmem, ctx->stream>>>(ca);
  MMMCU_LAUNCHED();
  ctx->gA = A;
  ctx->A = dt == MMMCU_F32 ? reinterpret_cast<const float*>(A) : nullptr;
  ctx->M = M;
  ctx->Ka = K;
  ctx->lda = lda;
  ctx->av = av;
  ctx->a_dt = dt;
  ctx->gen_a = true;
  ctx->op_at = false;
  ctx->has_a = true;
  return MMMCU_OK;
}

// preprocess_b for any lane: P-bit codes per region, per-row factors, totals.
template <typename T>
mmmcu_status gen_preprocess_b(mmmcu_ctx* ctx, const T* B, int64_t K, int64_t N, int64_t ldb, mmmcu_lane lane,
                              uint64_t bv, mmmcu_dtype dt) {
  if (K <= 0 || N <= 0) return fail(ctx, MMMCU_ERR_INVALID_ARG, "matrix dimensions must be positive");
  if (!B) return fail(ctx, MMMCU_ERR_INVALID_ARG, "B is null");
  const int64_t R = (int64_t)lane.w * lane.p * lane.v;
  if (ldb < N || ldb % R != 0)
    return fail(ctx, MMMCU_ERR_INVALID_ARG, "B needs ldb >= N and ldb a multiple of the region width " +
                                                std::to_string(R) + " (Matrix padding)");
  ctx->has_b = false;
  const int64_t nreg = ldb / R;
  MMMCU_CUDA(ctx->gcodes.ensure(sizeof(uint16_t) * K * nreg));
  MMMCU_CUDA(ctx->gzb.ensure(sizeof(uint32_t) * 2 * K));
  MMMCU_CUDA(ctx->stats.ensure(sizeof(unsigned long long) * 24));
  const int64_t n = K * nreg;
  mmmcu::kg_codes<T><<<(unsigned)((n + 255) / 256), 256, 0, ctx->stream>>>(B, K, ldb, nreg, lane.w * lane.v, lane.p,
                                                                          ctx->gcodes.as<uint16_t>());
  MMMCU_LAUNCHED();
  uint32_t* bpop = ctx->gzb.as<uint32_t>();
  mmmcu::kg_bcounts<<<(unsigned)((K + 255) / 256), 256, 0, ctx->stream>>>(ctx->gcodes.as<uint16_t>(), K, nreg, bpop,
                                                                         bpop + K);
  MMMCU_LAUNCHED();
  mmmcu::kg_plan_totals<<<1, 1024, 0, ctx->stream>>>(bpop, bpop + K, K, nreg, ctx->stats.as<unsigned long long>());
  MMMCU_LAUNCHED();
  ctx->gB = B;
  ctx->B = dt == MMMCU_F32 ? reinterpret_cast<const float*>(B) : nullptr;
  ctx->Kb = K;
  ctx->N = N;
  ctx->ldb = ldb;
  ctx->bv = bv;
  ctx->b_dt = dt;
  ctx->gen_G = lane.w * lane.v;
  ctx->gen_P = lane.p;
  ctx->gen_b = true;
  ctx->op_rows = ctx->op_tcb = false;
  ctx->has_b = true;
  return MMMCU_OK;
}

// Exact WorkCounters of a general-path plan: lane_fma_ops = Σ_k acol[k]·G·bpop[k].
mmmcu_status gen_counters(mmmcu_ctx* ctx, mmmcu_counters* out) {
  if (!out) return MMMCU_OK;
  if (!ctx->has_a || !ctx->has_b) return fail(ctx, MMMCU_ERR_NOT_READY, "counters need both plans");
  const int64_t K = ctx->Kb;
  MMMCU_CUDA(ctx->scratch0.ensure(sizeof(uint32_t) * ctx->Ka));
  uint32_t* acol = ctx->scratch0.as<uint32_t>();
  MMMCU_TRY(launch_acol(ctx, acol));
  const uint32_t* bpop = ctx->gzb.as<uint32_t>();
  mmmcu::kg_counters<<<1, 1024, 0, ctx->stream>>>(acol, bpop, bpop + K, K, ctx->M, gen_nreg(ctx), ctx->gen_G,
                                                  ctx->stats.as<unsigned long long>());
  MMMCU_LAUNCHED();
  unsigned long long s[16];
  MMMCU_TRY(read_stats(ctx, s));
  out->kernel_invocations = s[0];
  out->lane_fma_ops = s[1];
  out->rows_skipped = s[2];
  out->regions_skipped_by_zero_code = s[3];
  return MMMCU_OK;
}

// C += A*B over a general-path B plan (kg_mul: the reference's per-element fma chain).
template <typename T>
mmmcu_status gen_multiply(mmmcu_ctx* ctx, T* C, int64_t ldc, const T* A) {
  const int64_t nreg = gen_nreg(ctx);
  dim3 grid((unsigned)((ctx->ldb + mmmcu::kKgTile - 1) / mmmcu::kKgTile),
            (unsigned)((ctx->M + mmmcu::kKgTile - 1) / mmmcu::kKgTile));
  mmmcu::kg_mul<T, false><<<grid, 256, 0, ctx->stream>>>(A, ctx->lda, static_cast<const T*>(ctx->gB), ctx->ldb, C, ldc,
                                                         ctx->M, ctx->Ka, ctx->ldb, ctx->gcodes.as<uint16_t>(), nreg,
                                                         ctx->gen_G, ctx->gen_P);
  MMMCU_LAUNCHED();
  return MMMCU_OK;
}

}  // namespace

extern "C" {

int mmmcu_abi_version(void) { return MMMCU_ABI_VERSION; }

const char* mmmcu_last_error(const mmmcu_ctx* ctx) { return ctx ? ctx->err.c_str() : g_err.c_str(); }

mmmcu_status mmmcu_ctx_create(int device, mmmcu_ctx** out) {
  if (!out) return fail(nullptr, MMMCU_ERR_INVALID_ARG, "out is null");
  *out = nullptr;
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0) {
    cudaGetLastError();
    return fail(nullptr, MMMCU_ERR_NO_DEVICE, "no CUDA device (the masked multiply has no CPU fallback)");
  }
  if (device < 0 || device >= n) return fail(nullptr, MMMCU_ERR_INVALID_ARG, "device ordinal out of range");
  e = cudaSetDevice(device);
  if (e != cudaSuccess) return fail(nullptr, MMMCU_ERR_CUDA, std::string("cudaSetDevice: ") + cudaGetErrorString(e));
  mmmcu_ctx* ctx = new mmmcu_ctx();
  ctx->device = device;
  *out = ctx;
  return MMMCU_OK;
}

mmmcu_status mmmcu_ctx_destroy(mmmcu_ctx* ctx) {
  if (!ctx) return MMMCU_OK;
  cudaSetDevice(ctx->device);
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  for (DevBuf* b : {&ctx->abits, &ctx->za, &ctx->tile_prefix, &ctx->row_ptr, &ctx->cols, &ctx->codes, &ctx->bgrp, &ctx->zb,
                    &ctx->ctl, &ctx->at, &ctx->tcb, &ctx->tck, &ctx->tcn, &ctx->tc_pre, &ctx->brows, &ctx->row_off,
                    &ctx->stats, &ctx->hA, &ctx->hB, &ctx->hC, &ctx->scratch0, &ctx->scratch1, &ctx->gcodes,
                    &ctx->gza, &ctx->gzb})
    b->release();
  delete ctx;
  return MMMCU_OK;
}

mmmcu_status mmmcu_set_stream(mmmcu_ctx* ctx, void* stream) {
  MMMCU_TRY(bind(ctx));
  ctx->stream = static_cast<cudaStream_t>(stream);
  return MMMCU_OK;
}

mmmcu_status mmmcu_validate_lane(mmmcu_ctx* ctx, mmmcu_lane lane) { return check_lane(ctx, lane); }

mmmcu_status mmmcu_preprocess_a(mmmcu_ctx* ctx, const float* A, int64_t M, int64_t K, int64_t lda, uint64_t av) {
  MMMCU_TRY(bind(ctx));
  MMMCU_TRY(stage_a(ctx, A, M, K, lda, av));
  return launch_k1(ctx, true, false);
}

mmmcu_status mmmcu_preprocess_b(mmmcu_ctx* ctx, const float* B, int64_t K, int64_t N, int64_t ldb, mmmcu_lane lane,
                                uint64_t bv) {
  MMMCU_TRY(bind(ctx));
  MMMCU_TRY(check_lane(ctx, lane));
  if (!fast_lane(lane, MMMCU_F32)) return gen_preprocess_b(ctx, B, K, N, ldb, lane, bv, MMMCU_F32);
  MMMCU_TRY(stage_b(ctx, B, K, N, ldb, bv));
  return launch_k1(ctx, false, true);
}

mmmcu_status mmmcu_preprocess(mmmcu_ctx* ctx, const float* A, int64_t M, int64_t K, int64_t lda, const float* B,
                              int64_t N, int64_t ldb, mmmcu_lane lane, uint64_t av, uint64_t bv) {
  MMMCU_TRY(bind(ctx));
  MMMCU_TRY(check_lane(ctx, lane));
  if (!fast_lane(lane, MMMCU_F32)) {  // the lane-general path (kgen.cuh)
    MMMCU_TRY(gen_preprocess_a(ctx, A, M, K, lda, av, MMMCU_F32));
    return gen_preprocess_b(ctx, B, K, N, ldb, lane, bv, MMMCU_F32);
  }
  MMMCU_TRY(stage_a(ctx, A, M, K, lda, av));
  MMMCU_TRY(stage_b(ctx, B, K, N, ldb, bv));
  return launch_k1(ctx, true, true);
}

mmmcu_status mmmcu_get_counters(mmmcu_ctx* ctx, mmmcu_counters* out) {
  MMMCU_TRY(bind(ctx));
  if (!out) return fail(ctx, MMMCU_ERR_INVALID_ARG, "out is null");
  if (!ctx->has_a && !ctx->has_b) return fail(ctx, MMMCU_ERR_NOT_READY, "no plan");
  if (ctx->gen_a || ctx->gen_b) return gen_counters(ctx, out);
  return fill_counters(ctx, out);
}

mmmcu_status mmmcu_get_plan_stats(mmmcu_ctx* ctx, mmmcu_plan_stats* out) {
  MMMCU_TRY(bind(ctx));
  if (!out) return fail(ctx, MMMCU_ERR_INVALID_ARG, "out is null");
  if (!ctx->has_b) return fail(ctx, MMMCU_ERR_NOT_READY, "no B plan");
  unsigned long long s[16];
  MMMCU_TRY(read_stats(ctx, s));
  const int64_t n = ctx->Kb * (ctx->gen_b ? gen_nreg(ctx) : ctx->ldb / 64);
  out->region_count = n;
  out->zero_region_fraction = n ? (double)s[6] / (double)n : 0.0;
  out->mean_popcount = n ? (double)s[5] / (double)n : 0.0;
  return MMMCU_OK;
}

// The region codes are not materialised by K1's hot pass; rebuild them from the group masks.
mmmcu_status build_codes(mmmcu_ctx* ctx) {
  if (ctx->gen_b) {  // P <= 8 (callers check): the uint16 codes narrowed
    const int64_t n = ctx->Kb * gen_nreg(ctx);
    MMMCU_CUDA(ctx->codes.ensure((size_t)n));
    std::vector<uint16_t> w((size_t)n);
    std::vector<uint8_t> b((size_t)n);
    MMMCU_CUDA(cudaMemcpyAsync(w.data(), ctx->gcodes.p, sizeof(uint16_t) * n, cudaMemcpyDeviceToHost, ctx->stream));
    MMMCU_CUDA(cudaStreamSynchronize(ctx->stream));
    for (int64_t t = 0; t < n; ++t) b[(size_t)t] = (uint8_t)w[(size_t)t];
    MMMCU_CUDA(cudaMemcpyAsync(ctx->codes.p, b.data(), (size_t)n, cudaMemcpyHostToDevice, ctx->stream));
    MMMCU_CUDA(cudaStreamSynchronize(ctx->stream));
    return MMMCU_OK;
  }
  const int64_t n = ctx->Kb * (ctx->ldb / 64);
  mmmcu::k1_codes_export<<<(unsigned)((n + 255) / 256), 256, 0, ctx->stream>>>(
      ctx->bgrp.as<uint32_t>(), ctx->Kb, ctx->ldb / 64, (ctx->Kb + 31) / 32, ctx->codes.as<uint8_t>());
  MMMCU_LAUNCHED();
  return MMMCU_OK;
}

mmmcu_status mmmcu_export_b_codes(mmmcu_ctx* ctx, uint8_t* codes_host, int64_t capacity) {
  MMMCU_TRY(bind(ctx));
  if (!ctx->has_b) return fail(ctx, MMMCU_ERR_NOT_READY, "no B plan");
  if (ctx->gen_b && ctx->gen_P > 8)
    return fail(ctx, MMMCU_ERR_UNSUPPORTED, "codes wider than 8 bits: use mmmcu_export_b_codes16");
  const int64_t n = ctx->Kb * (ctx->gen_b ? gen_nreg(ctx) : ctx->ldb / 64);
  if (!codes_host || capacity < n) return fail(ctx, MMMCU_ERR_INVALID_ARG, "codes buffer too small");
  MMMCU_TRY(build_codes(ctx));
  MMMCU_CUDA(cudaMemcpyAsync(codes_host, ctx->codes.p, (size_t)n, cudaMemcpyDeviceToHost, ctx->stream));
  MMMCU_CUDA(cudaStreamSynchronize(ctx->stream));
  return MMMCU_OK;
}

extern "C++" {
// BPlan leaf order of row-major codes [K][nreg]
template <typename C>
void leaf_order(const std::vector<C>& codes, int64_t K, int64_t nreg, int64_t leaf_dim, int64_t rpl, C* plans_host,
                int64_t* plan_off_host) {
  const int64_t n_lr = (K + leaf_dim - 1) / leaf_dim, n_lc = (nreg + rpl - 1) / rpl;
  int64_t pos = 0, p = 0;
  for (int64_t lr = 0; lr < n_lr; ++lr)
    for (int64_t lc = 0; lc < n_lc; ++lc) {
      plan_off_host[p++] = pos;
      const int64_t k1 = std::min((lr + 1) * leaf_dim, K);
      const int64_t r0 = lc * rpl, r1 = std::min(r0 + rpl, nreg);
      for (int64_t k = lr * leaf_dim; k < k1; ++k)
        for (int64_t r = r0; r < r1; ++r) plans_host[pos++] = codes[(size_t)(k * nreg + r)];
    }
  plan_off_host[p] = pos;
}

template <typename C>
mmmcu_status export_bplans_t(mmmcu_ctx* ctx, int64_t leaf_dim, C* plans_host, int64_t plans_capacity,
                             int64_t* plan_off_host, int64_t off_capacity, int64_t* n_plans) {
  MMMCU_TRY(bind(ctx));
  if (!ctx->has_b) return fail(ctx, MMMCU_ERR_NOT_READY, "no B plan");
  if (sizeof(C) == 1 && ctx->gen_b && ctx->gen_P > 8)
    return fail(ctx, MMMCU_ERR_UNSUPPORTED, "codes wider than 8 bits: use mmmcu_export_bplans16");
  const int64_t R = ctx->gen_b ? (int64_t)ctx->gen_G * ctx->gen_P : 64;
  if (leaf_dim <= 0 || leaf_dim % R != 0)
    return fail(ctx, MMMCU_ERR_INVALID_ARG,
                "leaf_dim must be a positive multiple of the region width " + std::to_string(R));
  const int64_t K = ctx->Kb, nreg = ctx->ldb / R, rpl = leaf_dim / R;
  const int64_t n_lr = (K + leaf_dim - 1) / leaf_dim, n_lc = (nreg + rpl - 1) / rpl;
  if (n_plans) *n_plans = n_lr * n_lc;
  if (!plans_host || plans_capacity < K * nreg || !plan_off_host || off_capacity < n_lr * n_lc + 1)
    return fail(ctx, MMMCU_ERR_INVALID_ARG, "plan buffers too small");
  std::vector<C> codes((size_t)(K * nreg));
  if (ctx->gen_b) {
    std::vector<uint16_t> w((size_t)(K * nreg));
    MMMCU_CUDA(cudaMemcpyAsync(w.data(), ctx->gcodes.p, sizeof(uint16_t) * w.size(), cudaMemcpyDeviceToHost, ctx->stream));
    MMMCU_CUDA(cudaStreamSynchronize(ctx->stream));
    for (size_t t = 0; t < w.size(); ++t) codes[t] = (C)w[t];
  } else {
    std::vector<uint8_t> b((size_t)(K * nreg));
    MMMCU_TRY(build_codes(ctx));
    MMMCU_CUDA(cudaMemcpyAsync(b.data(), ctx->codes.p, b.size(), cudaMemcpyDeviceToHost, ctx->stream));
    MMMCU_CUDA(cudaStreamSynchronize(ctx->stream));
    for (size_t t = 0; t < b.size(); ++t) codes[t] = (C)b[t];
  }
  leaf_order(codes, K, nreg, leaf_dim, rpl, plans_host, plan_off_host);
  return MMMCU_OK;
}
}  // extern "C++"

mmmcu_status mmmcu_export_bplans(mmmcu_ctx* ctx, int64_t leaf_dim, uint8_t* plans_host, int64_t plans_capacity,
                                 int64_t* plan_off_host, int64_t off_capacity, int64_t* n_plans) {
  return export_bplans_t<uint8_t>(ctx, leaf_dim, plans_host, plans_capacity, plan_off_host, off_capacity, n_plans);
}

mmmcu_status mmmcu_export_bplans16(mmmcu_ctx* ctx, int64_t leaf_dim, uint16_t* plans_host, int64_t plans_capacity,
                                   int64_t* plan_off_host, int64_t off_capacity, int64_t* n_plans) {
  return export_bplans_t<uint16_t>(ctx, leaf_dim, plans_host, plans_capacity, plan_off_host, off_capacity, n_plans);
}

mmmcu_status mmmcu_export_b_codes16(mmmcu_ctx* ctx, uint16_t* codes_host, int64_t capacity) {
  MMMCU_TRY(bind(ctx));
  if (!ctx->has_b) return fail(ctx, MMMCU_ERR_NOT_READY, "no B plan");
  const int64_t n = ctx->Kb * (ctx->gen_b ? gen_nreg(ctx) : ctx->ldb / 64);
  if (!codes_host || capacity < n) return fail(ctx, MMMCU_ERR_INVALID_ARG, "codes buffer too small");
  if (ctx->gen_b) {
    MMMCU_CUDA(cudaMemcpyAsync(codes_host, ctx->gcodes.p, sizeof(uint16_t) * n, cudaMemcpyDeviceToHost, ctx->stream));
    MMMCU_CUDA(cudaStreamSynchronize(ctx->stream));
    return MMMCU_OK;
  }
  std::vector<uint8_t> b((size_t)n);
  MMMCU_TRY(build_codes(ctx));
  MMMCU_CUDA(cudaMemcpyAsync(b.data(), ctx->codes.p, (size_t)n, cudaMemcpyDeviceToHost, ctx->stream));
  MMMCU_CUDA(cudaStreamSynchronize(ctx->stream));
  for (int64_t t = 0; t < n; ++t) codes_host[t] = b[(size_t)t];
  return MMMCU_OK;
}

mmmcu_status mmmcu_export_a_bitmap(mmmcu_ctx* ctx, uint32_t* bits_host, int64_t capacity) {
  MMMCU_TRY(bind(ctx));
  if (!ctx->has_a) return fail(ctx, MMMCU_ERR_NOT_READY, "no A plan");
  const int64_t n = ctx->M * ((ctx->Ka + 31) / 32);
  if (!bits_host || capacity < n) return fail(ctx, MMMCU_ERR_INVALID_ARG, "bitmap buffer too small");
  MMMCU_CUDA(cudaMemcpyAsync(bits_host, ctx->abits.p, sizeof(uint32_t) * n, cudaMemcpyDeviceToHost, ctx->stream));
  MMMCU_CUDA(cudaStreamSynchronize(ctx->stream));
  return MMMCU_OK;
}

mmmcu_status mmmcu_export_a_csr(mmmcu_ctx* ctx, int64_t* row_ptr_host, uint32_t* cols_host, int64_t cols_capacity,
                                int64_t* nnz) {
  MMMCU_TRY(bind(ctx));
  if (!ctx->has_a) return fail(ctx, MMMCU_ERR_NOT_READY, "no A plan");
  if (!row_ptr_host) return fail(ctx, MMMCU_ERR_INVALID_ARG, "row_ptr buffer is null");
  MMMCU_CUDA(cudaMemcpyAsync(row_ptr_host, ctx->row_ptr.p, sizeof(int64_t) * (ctx->M + 1), cudaMemcpyDeviceToHost,
                             ctx->stream));
  MMMCU_CUDA(cudaStreamSynchronize(ctx->stream));
  const int64_t total = row_ptr_host[ctx->M];
  if (nnz) *nnz = total;
  if (!cols_host) return MMMCU_OK;
  if (cols_capacity < total) return fail(ctx, MMMCU_ERR_INVALID_ARG, "cols buffer too small");
  if (ctx->csr_idx_bytes == 4) {
    MMMCU_CUDA(cudaMemcpyAsync(cols_host, ctx->cols.p, sizeof(uint32_t) * total, cudaMemcpyDeviceToHost, ctx->stream));
    MMMCU_CUDA(cudaStreamSynchronize(ctx->stream));
  } else {
    std::vector<uint16_t> tmp((size_t)total);
    MMMCU_CUDA(cudaMemcpyAsync(tmp.data(), ctx->cols.p, sizeof(uint16_t) * total, cudaMemcpyDeviceToHost, ctx->stream));
    MMMCU_CUDA(cudaStreamSynchronize(ctx->stream));
    for (int64_t t = 0; t < total; ++t) cols_host[t] = tmp[(size_t)t];
  }
  return MMMCU_OK;
}

mmmcu_status mmmcu_export_ablock_index(mmmcu_ctx* ctx, int64_t block_dim, uint8_t* counts_host, int64_t counts_capacity,
                                       uint8_t* offsets_host, int64_t offsets_capacity, int64_t* n_segments) {
  MMMCU_TRY(bind(ctx));
  if (!ctx->has_a) return fail(ctx, MMMCU_ERR_NOT_READY, "no A plan");
  if (block_dim <= 0 || block_dim % 8 != 0)
    return fail(ctx, MMMCU_ERR_INVALID_ARG, "block_dim must be a positive multiple of the segment width 8");
  const int64_t M = ctx->M, K = ctx->Ka, kw = (K + 31) / 32;
  const int64_t nseg = M * ((K + 7) / 8);
  if (n_segments) *n_segments = nseg;
  if (!counts_host || counts_capacity < nseg || !offsets_host || offsets_capacity < 8 * nseg)
    return fail(ctx, MMMCU_ERR_INVALID_ARG, "ABlockIndex buffers too small");
  MMMCU_CUDA(ctx->scratch0.ensure((size_t)nseg));
  MMMCU_CUDA(ctx->scratch1.ensure((size_t)nseg * 8));
  const unsigned blocks = (unsigned)((nseg + 255) / 256);
  mmmcu::k1_ablock_export<<<blocks, 256, 0, ctx->stream>>>(ctx->abits.as<uint32_t>(), M, K, kw, block_dim,
                                                           (K + block_dim - 1) / block_dim, ctx->scratch0.as<uint8_t>(),
                                                           ctx->scratch1.as<uint8_t>());
  MMMCU_LAUNCHED();
  MMMCU_CUDA(cudaMemcpyAsync(counts_host, ctx->scratch0.p, (size_t)nseg, cudaMemcpyDeviceToHost, ctx->stream));
  MMMCU_CUDA(cudaMemcpyAsync(offsets_host, ctx->scratch1.p, (size_t)nseg * 8, cudaMemcpyDeviceToHost, ctx->stream));
  MMMCU_CUDA(cudaStreamSynchronize(ctx->stream));
  return MMMCU_OK;
}

mmmcu_status mmmcu_set_algo(mmmcu_ctx* ctx, mmmcu_algo algo) {
  MMMCU_TRY(bind(ctx));
  if (algo < MMMCU_ALGO_AUTO || algo > MMMCU_ALGO_CSR)
    return fail(ctx, MMMCU_ERR_INVALID_ARG, "unknown algorithm");
  ctx->algo = algo;
  return MMMCU_OK;
}

mmmcu_status mmmcu_last_algo(mmmcu_ctx* ctx, mmmcu_algo* algo) {
  if (!ctx || !algo) return fail(ctx, MMMCU_ERR_INVALID_ARG, "null argument");
  if (ctx->auto_pending || ctx->last_algo == MMMCU_ALGO_SIMT_BCAST) {  // resolved on the device: read it
    MMMCU_TRY(bind(ctx));
    unsigned long long s[16];
    MMMCU_TRY(read_stats(ctx, s));
    if (ctx->auto_pending)
      ctx->last_algo = s[7] == 32   ? MMMCU_ALGO_TC
                       : s[7] == 48 ? MMMCU_ALGO_CSR
                       : s[7] == 8  ? MMMCU_ALGO_SIMT_SPAN8
                                    : MMMCU_ALGO_SIMT_SPAN16;
    else if (ctx->op_at && ctx->op_rows)  // the K2-SIMT span K1 chose (the v1 fallback runs span 8)
      ctx->last_algo = s[8] == 8 ? MMMCU_ALGO_SIMT_SPAN8 : MMMCU_ALGO_SIMT_SPAN16;
    else
      ctx->last_algo = MMMCU_ALGO_SIMT_SPAN8;
    ctx->auto_pending = false;
  }
  *algo = ctx->last_algo;
  return MMMCU_OK;
}

mmmcu_status mmmcu_multiply(mmmcu_ctx* ctx, float* C, int64_t ldc, const float* A, const float* B, uint64_t av,
                            uint64_t bv, mmmcu_counters* counters) {
  if (ctx && (ctx->gen_a || ctx->gen_b)) return mmmcu_multiply_t(ctx, MMMCU_F32, C, ldc, A, B, av, bv, counters);
  MMMCU_TRY(bind(ctx));
  MMMCU_TRY(check_plan(ctx, A, B, av, bv));
  if (!C) return fail(ctx, MMMCU_ERR_INVALID_ARG, "C is null");
  if (ldc < round_up(ctx->N, 64) || ldc % 4 != 0 || !aligned16(C))
    return fail(ctx, MMMCU_ERR_INVALID_ARG,
                "C must be 16-byte aligned with ldc >= round_up(N, 64) (Matrix padding) and ldc % 4 == 0");
  ctx->auto_pending = false;
  if (ctx->algo == MMMCU_ALGO_AUTO && ctx->op_at && ctx->op_rows && ctx->op_tcb) {
    // both operand sets are built; every variant is launched and all but the chosen one
    // exit at entry (stats[7]: 8 / 16 = K2-SIMT span, 32 = K2-TC) — no host round trip
    ctx->last_algo = MMMCU_ALGO_AUTO;
    ctx->auto_pending = true;
    MMMCU_TRY(launch_simt(ctx, C, ldc, 0, 7));
    MMMCU_TRY(launch_tc(ctx, C, ldc, ctx->stats.as<unsigned long long>() + 7));
  } else if (ctx->algo == MMMCU_ALGO_TC || ctx->algo == MMMCU_ALGO_TC32) {
    if (!ctx->op_at || !ctx->op_tcb)
      return fail(ctx, MMMCU_ERR_NOT_READY, "the TC operands were not built: preprocess with algo TC");
    ctx->last_algo = ctx->algo;
    if (!ctx->tcb_fresh || ctx->tcb_f16 != tc_f16(ctx)) {
      MMMCU_TRY(pack_tc(ctx));
      ctx->tcb_fresh = true;
    }
    MMMCU_TRY(launch_tc(ctx, C, ldc, nullptr));
  } else if (ctx->algo == MMMCU_ALGO_CSR) {
    if (!ctx->op_at) return fail(ctx, MMMCU_ERR_NOT_READY, "the CSR operands were not built: preprocess with algo CSR");
    ctx->last_algo = MMMCU_ALGO_CSR;
    MMMCU_TRY(launch_csr(ctx, C, ldc, nullptr));
  } else if (ctx->algo == MMMCU_ALGO_DENSE) {
    ctx->last_algo = MMMCU_ALGO_DENSE;
    dim3 grid((unsigned)((ctx->N + 63) / 64), (unsigned)((ctx->M + 63) / 64));
    mmmcu::k2_dense<<<grid, 256, 0, ctx->stream>>>(ctx->A, ctx->lda, ctx->B, ctx->ldb, C, ldc, ctx->M, ctx->Ka, ctx->N);
    MMMCU_LAUNCHED();
  } else {
    const int span = ctx->algo == MMMCU_ALGO_SIMT_SPAN8 ? 8 : ctx->algo == MMMCU_ALGO_SIMT_SPAN16 ? 16 : 0;
    ctx->last_algo = span == 8 ? MMMCU_ALGO_SIMT_SPAN8 : span == 16 ? MMMCU_ALGO_SIMT_SPAN16 : MMMCU_ALGO_SIMT_BCAST;
    if (ctx->op_rows && !ctx->rows_fresh) {
      mmmcu::k1_row_off<<<1, mmmcu::kK1Threads, 0, ctx->stream>>>(zb_row_cnt(ctx), ctx->n_tb * ((ctx->Kb + 31) / 32),
                                                                   ctx->row_off.as<int64_t>());
      MMMCU_LAUNCHED();
      MMMCU_TRY(pack_rows(ctx));
      ctx->rows_fresh = true;
    }
    MMMCU_TRY(launch_simt(ctx, C, ldc, span, 8));
  }
  return fill_counters(ctx, counters);
}

mmmcu_status mmmcu_multiply_parallel(mmmcu_ctx* ctx, float* C, int64_t ldc, const float* A, const float* B,
                                     uint64_t av, uint64_t bv, int worker_count, mmmcu_counters* counters) {
  if (worker_count <= 0) return fail(ctx, MMMCU_ERR_WORKERS, "worker_count must be positive");
  return mmmcu_multiply(ctx, C, ldc, A, B, av, bv, counters);
}

mmmcu_status mmmcu_multiply_simple(mmmcu_ctx* ctx, float* C, int64_t ldc, const float* A, int64_t lda, const float* B,
                                   int64_t ldb, int64_t M, int64_t K, int64_t N) {
  MMMCU_TRY(bind(ctx));
  if (M <= 0 || K <= 0 || N <= 0) return fail(ctx, MMMCU_ERR_INVALID_ARG, "matrix dimensions must be positive");
  if (!A || !B || !C) return fail(ctx, MMMCU_ERR_INVALID_ARG, "null operand");
  if (lda < K || ldb < N || ldc < N) return fail(ctx, MMMCU_ERR_DIM_MISMATCH, "leading dimension smaller than the row");
  dim3 grid((unsigned)((N + 63) / 64), (unsigned)((M + 63) / 64));
  mmmcu::k2_dense<<<grid, 256, 0, ctx->stream>>>(A, lda, B, ldb, C, ldc, M, K, N);
  MMMCU_LAUNCHED();
  return MMMCU_OK;
}

mmmcu_status mmmcu_multiply_host_t(mmmcu_ctx* ctx, mmmcu_dtype dt, void* C_host, int64_t ldc, const void* A_host,
                                   int64_t lda, const void* B_host, int64_t ldb, int64_t M, int64_t K, int64_t N,
                                   mmmcu_lane lane, mmmcu_counters* counters) {
  MMMCU_TRY(bind(ctx));
  if (M <= 0 || K <= 0 || N <= 0) return fail(ctx, MMMCU_ERR_INVALID_ARG, "matrix dimensions must be positive");
  if (!A_host || !B_host || !C_host) return fail(ctx, MMMCU_ERR_INVALID_ARG, "null operand");
  if (dt != MMMCU_F32 && dt != MMMCU_F64) return fail(ctx, MMMCU_ERR_UNSUPPORTED, "unknown dtype");
  const size_t es = dt_size(dt);
  MMMCU_CUDA(ctx->hA.ensure(es * M * lda));
  MMMCU_CUDA(ctx->hB.ensure(es * K * ldb));
  MMMCU_CUDA(ctx->hC.ensure(es * M * ldc));
  MMMCU_CUDA(cudaMemcpyAsync(ctx->hA.p, A_host, es * M * lda, cudaMemcpyHostToDevice, ctx->stream));
  MMMCU_CUDA(cudaMemcpyAsync(ctx->hB.p, B_host, es * K * ldb, cudaMemcpyHostToDevice, ctx->stream));
  MMMCU_CUDA(cudaMemcpyAsync(ctx->hC.p, C_host, es * M * ldc, cudaMemcpyHostToDevice, ctx->stream));
  // host operands carry no version: tag the staging copies with a per-call counter
  static thread_local uint64_t tag = 0;
  ++tag;
  MMMCU_TRY(mmmcu_preprocess_t(ctx, dt, ctx->hA.p, M, K, lda, ctx->hB.p, N, ldb, lane, tag, tag));
  MMMCU_TRY(mmmcu_multiply_t(ctx, dt, ctx->hC.p, ldc, ctx->hA.p, ctx->hB.p, tag, tag, nullptr));
  MMMCU_CUDA(cudaMemcpyAsync(C_host, ctx->hC.p, es * M * ldc, cudaMemcpyDeviceToHost, ctx->stream));
  MMMCU_CUDA(cudaStreamSynchronize(ctx->stream));
  return counters ? mmmcu_get_counters(ctx, counters) : MMMCU_OK;
}

mmmcu_status mmmcu_multiply_host(mmmcu_ctx* ctx, float* C_host, int64_t ldc, const float* A_host, int64_t lda,
                                 const float* B_host, int64_t ldb, int64_t M, int64_t K, int64_t N,
                                 mmmcu_counters* counters) {
  return mmmcu_multiply_host_t(ctx, MMMCU_F32, C_host, ldc, A_host, lda, B_host, ldb, M, K, N, mmmcu_lane{8, 8, 1},
                               counters);
}

mmmcu_status mmmcu_preprocess_host_t(mmmcu_ctx* ctx, mmmcu_dtype dt, const void* A_host, int64_t M, int64_t K,
                                     int64_t lda, const void* B_host, int64_t N, int64_t ldb, mmmcu_lane lane,
                                     uint64_t av, uint64_t bv) {
  MMMCU_TRY(bind(ctx));
  MMMCU_TRY(validate_lane(ctx, lane, dt));
  if (M <= 0 || K <= 0 || N <= 0) return fail(ctx, MMMCU_ERR_INVALID_ARG, "matrix dimensions must be positive");
  if (!A_host || !B_host) return fail(ctx, MMMCU_ERR_INVALID_ARG, "null operand");
  if (lda < K || ldb < N) return fail(ctx, MMMCU_ERR_DIM_MISMATCH, "leading dimension smaller than the row");
  const size_t es = dt_size(dt);
  MMMCU_CUDA(ctx->hA.ensure(es * M * lda));
  MMMCU_CUDA(ctx->hB.ensure(es * K * ldb));
  MMMCU_CUDA(cudaMemcpyAsync(ctx->hA.p, A_host, es * M * lda, cudaMemcpyHostToDevice, ctx->stream));
  MMMCU_CUDA(cudaMemcpyAsync(ctx->hB.p, B_host, es * K * ldb, cudaMemcpyHostToDevice, ctx->stream));
  MMMCU_TRY(mmmcu_preprocess_t(ctx, dt, ctx->hA.p, M, K, lda, ctx->hB.p, N, ldb, lane, av, bv));
  MMMCU_CUDA(cudaStreamSynchronize(ctx->stream));  // the host buffers may change after return
  return MMMCU_OK;
}

mmmcu_status mmmcu_preprocess_host(mmmcu_ctx* ctx, const float* A_host, int64_t M, int64_t K, int64_t lda,
                                   const float* B_host, int64_t N, int64_t ldb, mmmcu_lane lane, uint64_t av,
                                   uint64_t bv) {
  return mmmcu_preprocess_host_t(ctx, MMMCU_F32, A_host, M, K, lda, B_host, N, ldb, lane, av, bv);
}

mmmcu_status mmmcu_multiply_planned_host_t(mmmcu_ctx* ctx, mmmcu_dtype dt, void* C_host, int64_t ldc, uint64_t av,
                                           uint64_t bv, int worker_count, mmmcu_counters* counters) {
  MMMCU_TRY(bind(ctx));
  if (worker_count <= 0) return fail(ctx, MMMCU_ERR_WORKERS, "worker_count must be positive");
  if (!C_host) return fail(ctx, MMMCU_ERR_INVALID_ARG, "C is null");
  if (!ctx->has_a || !ctx->has_b || plan_a(ctx) != ctx->hA.p || plan_b(ctx) != ctx->hB.p)
    return fail(ctx, MMMCU_ERR_NOT_READY, "no host-operand plan: call mmmcu_preprocess_host first");
  if (av != ctx->av || bv != ctx->bv)
    return fail(ctx, MMMCU_ERR_STALE, "stale context: operands changed since preprocessing (Matrix::version)");
  const size_t es = dt_size(dt);
  const int64_t M = ctx->M;
  MMMCU_CUDA(ctx->hC.ensure(es * M * ldc));
  MMMCU_CUDA(cudaMemcpyAsync(ctx->hC.p, C_host, es * M * ldc, cudaMemcpyHostToDevice, ctx->stream));
  MMMCU_TRY(mmmcu_multiply_t(ctx, dt, ctx->hC.p, ldc, ctx->hA.p, ctx->hB.p, av, bv, nullptr));
  MMMCU_CUDA(cudaMemcpyAsync(C_host, ctx->hC.p, es * M * ldc, cudaMemcpyDeviceToHost, ctx->stream));
  MMMCU_CUDA(cudaStreamSynchronize(ctx->stream));
  return counters ? mmmcu_get_counters(ctx, counters) : MMMCU_OK;
}

mmmcu_status mmmcu_multiply_simple_host_t(mmmcu_ctx* ctx, mmmcu_dtype dt, void* C_host, int64_t ldc, const void* A_host,
                                          int64_t lda, const void* B_host, int64_t ldb, int64_t M, int64_t K, int64_t N) {
  MMMCU_TRY(bind(ctx));
  if (M <= 0 || K <= 0 || N <= 0) return fail(ctx, MMMCU_ERR_INVALID_ARG, "matrix dimensions must be positive");
  if (!A_host || !B_host || !C_host) return fail(ctx, MMMCU_ERR_INVALID_ARG, "null operand");
  if (dt != MMMCU_F32 && dt != MMMCU_F64) return fail(ctx, MMMCU_ERR_UNSUPPORTED, "unknown dtype");
  const size_t es = dt_size(dt);
  MMMCU_CUDA(ctx->hA.ensure(es * M * lda));
  MMMCU_CUDA(ctx->hB.ensure(es * K * ldb));
  MMMCU_CUDA(ctx->hC.ensure(es * M * ldc));
  MMMCU_CUDA(cudaMemcpyAsync(ctx->hA.p, A_host, es * M * lda, cudaMemcpyHostToDevice, ctx->stream));
  MMMCU_CUDA(cudaMemcpyAsync(ctx->hB.p, B_host, es * K * ldb, cudaMemcpyHostToDevice, ctx->stream));
  MMMCU_CUDA(cudaMemcpyAsync(ctx->hC.p, C_host, es * M * ldc, cudaMemcpyHostToDevice, ctx->stream));
  MMMCU_TRY(mmmcu_multiply_simple_t(ctx, dt, ctx->hC.p, ldc, ctx->hA.p, lda, ctx->hB.p, ldb, M, K, N));
  MMMCU_CUDA(cudaMemcpyAsync(C_host, ctx->hC.p, es * M * ldc, cudaMemcpyDeviceToHost, ctx->stream));
  MMMCU_CUDA(cudaStreamSynchronize(ctx->stream));
  return MMMCU_OK;
}

mmmcu_status mmmcu_multiply_planned_host(mmmcu_ctx* ctx, float* C_host, int64_t ldc, uint64_t av, uint64_t bv,
                                         int worker_count, mmmcu_counters* counters) {
  return mmmcu_multiply_planned_host_t(ctx, MMMCU_F32, C_host, ldc, av, bv, worker_count, counters);
}

mmmcu_status mmmcu_generate(mmmcu_ctx* ctx, float* out, int64_t rows, int64_t cols, int64_t ld, int64_t row0, uint64_t seed,
                            int value_kind, double sigma, double thresh, int mask_kind, double p, int64_t block) {
  MMMCU_TRY(bind(ctx));
  if (rows <= 0 || cols <= 0 || ld < cols || row0 < 0 || !out) return fail(ctx, MMMCU_ERR_INVALID_ARG, "bad generator shape");
  if (value_kind < 0 || value_kind > 2 || mask_kind < 0 || mask_kind > 2 || (mask_kind == 2 && block <= 0) ||
      !(p >= 0.0 && p <= 1.0))
    return fail(ctx, MMMCU_ERR_INVALID_ARG, "bad generator spec");
  const int64_t total = rows * ld;
  if (ctx->num_sms == 0) MMMCU_CUDA(cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, ctx->device));
  const unsigned blocks = (unsigned)std::min<int64_t>((total + 255) / 256, (int64_t)ctx->num_sms * 64);
  mmmcu::k_generate<<<blocks, 256, 0, ctx->stream>>>(out, rows, cols, ld, row0, seed, value_kind, sigma, thresh, mask_kind, p,
                                                     block);
  MMMCU_LAUNCHED();
  return MMMCU_OK;
}

mmmcu_status mmmcu_shard_rows(int64_t M, int world, int rank, int64_t* row0, int64_t* row1) {
  if (M <= 0 || world <= 0 || rank < 0 || rank >= world || !row0 || !row1)
    return fail(nullptr, MMMCU_ERR_INVALID_ARG, "bad shard arguments");
  *row0 = M * rank / world;
  *row1 = M * (rank + 1) / world;
  return MMMCU_OK;
}


// ---------------------------------------------------- every (dtype, lane config) (kgen.cuh)
mmmcu_status mmmcu_validate_lane_t(mmmcu_ctx* ctx, mmmcu_dtype dt, mmmcu_lane lane) {
  return validate_lane(ctx, lane, dt);
}

mmmcu_status mmmcu_preprocess_a_t(mmmcu_ctx* ctx, mmmcu_dtype dt, const void* A, int64_t M, int64_t K, int64_t lda,
                                  uint64_t av) {
  MMMCU_TRY(bind(ctx));
  if (dt == MMMCU_F32) return mmmcu_preprocess_a(ctx, static_cast<const float*>(A), M, K, lda, av);
  if (dt != MMMCU_F64) return fail(ctx, MMMCU_ERR_UNSUPPORTED, "unknown dtype");
  return gen_preprocess_a(ctx, static_cast<const double*>(A), M, K, lda, av, dt);
}

mmmcu_status mmmcu_preprocess_b_t(mmmcu_ctx* ctx, mmmcu_dtype dt, const void* B, int64_t K, int64_t N, int64_t ldb,
                                  mmmcu_lane lane, uint64_t bv) {
  MMMCU_TRY(bind(ctx));
  MMMCU_TRY(validate_lane(ctx, lane, dt));
  if (dt == MMMCU_F32) return mmmcu_preprocess_b(ctx, static_cast<const float*>(B), K, N, ldb, lane, bv);
  return gen_preprocess_b(ctx, static_cast<const double*>(B), K, N, ldb, lane, bv, dt);
}

mmmcu_status mmmcu_preprocess_t(mmmcu_ctx* ctx, mmmcu_dtype dt, const void* A, int64_t M, int64_t K, int64_t lda,
                                const void* B, int64_t N, int64_t ldb, mmmcu_lane lane, uint64_t av, uint64_t bv) {
  MMMCU_TRY(bind(ctx));
  MMMCU_TRY(validate_lane(ctx, lane, dt));
  if (dt == MMMCU_F32)
    return mmmcu_preprocess(ctx, static_cast<const float*>(A), M, K, lda, static_cast<const float*>(B), N, ldb, lane,
                            av, bv);
  MMMCU_TRY(gen_preprocess_a(ctx, static_cast<const double*>(A), M, K, lda, av, dt));
  return gen_preprocess_b(ctx, static_cast<const double*>(B), K, N, ldb, lane, bv, dt);
}

mmmcu_status mmmcu_multiply_t(mmmcu_ctx* ctx, mmmcu_dtype dt, void* C, int64_t ldc, const void* A, const void* B,
                              uint64_t av, uint64_t bv, mmmcu_counters* counters) {
  MMMCU_TRY(bind(ctx));
  if (dt != MMMCU_F32 && dt != MMMCU_F64) return fail(ctx, MMMCU_ERR_UNSUPPORTED, "unknown dtype");
  if (!(ctx->gen_a || ctx->gen_b)) {
    if (dt != MMMCU_F32) return fail(ctx, MMMCU_ERR_NOT_READY, "no f64 plan: preprocess with mmmcu_preprocess_t");
    return mmmcu_multiply(ctx, static_cast<float*>(C), ldc, static_cast<const float*>(A),
                          static_cast<const float*>(B), av, bv, counters);
  }
  if (!ctx->has_a || !ctx->has_b)
    return fail(ctx, MMMCU_ERR_NOT_READY, "multiply called before preprocess_a/preprocess_b");
  if (ctx->a_dt != dt || ctx->b_dt != dt)
    return fail(ctx, MMMCU_ERR_INVALID_ARG, "operand dtype differs from the preprocessed plan's");
  if (ctx->Ka != ctx->Kb)
    return fail(ctx, MMMCU_ERR_DIM_MISMATCH, "a.cols != b.rows (" + std::to_string(ctx->Ka) + " vs " +
                                                  std::to_string(ctx->Kb) + ")");
  if (A != plan_a(ctx) || B != plan_b(ctx) || av != ctx->av || bv != ctx->bv)
    return fail(ctx, MMMCU_ERR_STALE, "stale context: operands differ from the preprocessed ones");
  if (!C) return fail(ctx, MMMCU_ERR_INVALID_ARG, "C is null");
  if (ldc < ctx->ldb)
    return fail(ctx, MMMCU_ERR_INVALID_ARG, "C needs ldc >= the padded width of B (the regions cover the padding)");
  if (!ctx->gen_b) return fail(ctx, MMMCU_ERR_NOT_READY, "B plan missing for the general path");
  if (dt == MMMCU_F64)
    MMMCU_TRY(gen_multiply(ctx, static_cast<double*>(C), ldc, static_cast<const double*>(A)));
  else
    MMMCU_TRY(gen_multiply(ctx, static_cast<float*>(C), ldc, static_cast<const float*>(A)));
  ctx->last_algo = MMMCU_ALGO_SIMT_BCAST;
  return gen_counters(ctx, counters);
}

mmmcu_status mmmcu_multiply_simple_t(mmmcu_ctx* ctx, mmmcu_dtype dt, void* C, int64_t ldc, const void* A, int64_t lda,
                                     const void* B, int64_t ldb, int64_t M, int64_t K, int64_t N) {
  MMMCU_TRY(bind(ctx));
  if (dt == MMMCU_F32)
    return mmmcu_multiply_simple(ctx, static_cast<float*>(C), ldc, static_cast<const float*>(A), lda,
                                 static_cast<const float*>(B), ldb, M, K, N);
  if (dt != MMMCU_F64) return fail(ctx, MMMCU_ERR_UNSUPPORTED, "unknown dtype");
  if (M <= 0 || K <= 0 || N <= 0) return fail(ctx, MMMCU_ERR_INVALID_ARG, "matrix dimensions must be positive");
  if (!A || !B || !C) return fail(ctx, MMMCU_ERR_INVALID_ARG, "null operand");
  if (lda < K || ldb < N || ldc < N) return fail(ctx, MMMCU_ERR_DIM_MISMATCH, "leading dimension smaller than the row");
  dim3 grid((unsigned)((N + mmmcu::kKgTile - 1) / mmmcu::kKgTile), (unsigned)((M + mmmcu::kKgTile - 1) / mmmcu::kKgTile));
  mmmcu::kg_mul<double, true><<<grid, 256, 0, ctx->stream>>>(static_cast<const double*>(A), lda,
                                                             static_cast<const double*>(B), ldb, static_cast<double*>(C),
                                                             ldc, M, K, N, nullptr, 1, 1, 1);
  MMMCU_LAUNCHED();
  return MMMCU_OK;
}

mmmcu_status mmmcu_plan_info(mmmcu_ctx* ctx, mmmcu_dtype* dt, mmmcu_lane* lane) {
  if (!ctx) return fail(nullptr, MMMCU_ERR_INVALID_ARG, "null context");
  if (!ctx->has_b) return fail(ctx, MMMCU_ERR_NOT_READY, "no B plan");
  if (dt) *dt = ctx->b_dt;
  if (lane) *lane = ctx->gen_b ? mmmcu_lane{ctx->gen_G, ctx->gen_P, 1} : mmmcu_lane{8, 8, 1};
  return MMMCU_OK;
}

}  // extern "C"
