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
#include <cstring>
#include <string>
#include <vector>

#include "gen.cuh"
#include "k1_preprocess.cuh"
#include "k2_simt.cuh"

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
    const size_t want = std::max<size_t>(bytes, 256);
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
  cudaStream_t stream = nullptr;
  std::string err;
  mmmcu_algo algo = MMMCU_ALGO_AUTO;
  mmmcu_algo last_algo = MMMCU_ALGO_AUTO;

  // ---- A plan (preprocess_a)
  bool has_a = false;
  const float* A = nullptr;
  int64_t M = 0, Ka = 0, lda = 0;
  uint64_t av = 0;
  int csr_idx_bytes = 4;
  DevBuf abits, arow, acol, row_ptr, cols;

  // ---- B plan (preprocess_b)
  bool has_b = false;
  const float* B = nullptr;
  int64_t Kb = 0, N = 0, ldb = 0;
  uint64_t bv = 0;
  DevBuf codes, bgrp, bpop, bnz;

  // ---- statistics: u64 [16] = {inv, lanes, skipped, zreg, nnzA, pop, zero_codes, span, slice_nz}
  DevBuf stats;

  // ---- host-operand staging (mmmcu_multiply_host)
  DevBuf hA, hB, hC;

  // ---- export scratch
  DevBuf scratch0, scratch1;
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

mmmcu_status bind(mmmcu_ctx* ctx) {
  if (!ctx) return fail(nullptr, MMMCU_ERR_INVALID_ARG, "null context");
  MMMCU_CUDA(cudaSetDevice(ctx->device));
  return MMMCU_OK;
}

// KernelTable<float>::build (kernel_table.cpp:64-72) + Matrix ctor lane checks
// (matrix.hpp:73-74), then the GPU support check.
mmmcu_status check_lane(mmmcu_ctx* ctx, mmmcu_lane lane) {
  if (lane.w <= 0 || lane.p <= 0 || lane.v <= 0)
    return fail(ctx, MMMCU_ERR_INVALID_ARG, "lane config fields must be positive");
  if (lane.p < 1 || lane.p > 16)
    return fail(ctx, MMMCU_ERR_INVALID_ARG, "pattern size must lie in [1, 16], got " + std::to_string(lane.p));
  const int g = lane.w * lane.v;
  if (g != 1 && g != 2 && g != 4 && g != 8 && g != 16 && g != 32 && g != 64)
    return fail(ctx, MMMCU_ERR_INVALID_ARG,
                "unsupported lane configuration: group width " + std::to_string(g) + " for f32");
  if (!(lane.w == 8 && lane.p == 8 && lane.v == 1))
    return fail(ctx, MMMCU_ERR_UNSUPPORTED,
                "the GPU path implements the f32 default lane config {W=8,P=8,V=1} only");
  return MMMCU_OK;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

mmmcu_status run_finalize(mmmcu_ctx* ctx) {
  const int64_t K = ctx->has_a ? ctx->Ka : ctx->Kb;
  if (ctx->has_a && ctx->has_b && ctx->Ka != ctx->Kb) return MMMCU_OK;  // mismatched: multiply rejects
  const int64_t nreg = ctx->has_b ? ctx->ldb / 64 : 0;
  mmmcu::k1_finalize<<<1, 1024, 0, ctx->stream>>>(
      ctx->has_a ? ctx->acol.as<uint32_t>() : nullptr, ctx->has_b ? ctx->bpop.as<uint32_t>() : nullptr,
      ctx->has_b ? ctx->bnz.as<uint32_t>() : nullptr, K, ctx->has_a ? ctx->M : 0, nreg, ctx->has_a ? 1 : 0,
      ctx->has_b ? 1 : 0, ctx->stats.as<unsigned long long>() + 8, ctx->stats.as<unsigned long long>());
  MMMCU_LAUNCHED();
  return MMMCU_OK;
}

mmmcu_status do_preprocess_a(mmmcu_ctx* ctx, const float* A, int64_t M, int64_t K, int64_t lda, uint64_t av) {
  if (M <= 0 || K <= 0) return fail(ctx, MMMCU_ERR_INVALID_ARG, "matrix dimensions must be positive");
  if (!A) return fail(ctx, MMMCU_ERR_INVALID_ARG, "A is null");
  if (lda < K || lda % 4 != 0 || !aligned16(A))
    return fail(ctx, MMMCU_ERR_INVALID_ARG, "A must be 16-byte aligned with lda >= K and lda % 4 == 0");
  const int64_t kw = (K + 31) / 32;
  ctx->has_a = false;
  ctx->csr_idx_bytes = K <= 65536 ? 2 : 4;
  MMMCU_CUDA(ctx->abits.ensure(sizeof(uint32_t) * M * kw));
  MMMCU_CUDA(ctx->arow.ensure(sizeof(uint32_t) * M));
  MMMCU_CUDA(ctx->acol.ensure(sizeof(uint32_t) * K));
  MMMCU_CUDA(ctx->row_ptr.ensure(sizeof(int64_t) * (M + 1)));
  MMMCU_CUDA(ctx->cols.ensure((size_t)ctx->csr_idx_bytes * M * K));
  MMMCU_CUDA(ctx->stats.ensure(sizeof(unsigned long long) * 16));
  MMMCU_CUDA(cudaMemsetAsync(ctx->arow.p, 0, sizeof(uint32_t) * M, ctx->stream));
  MMMCU_CUDA(cudaMemsetAsync(ctx->acol.p, 0, sizeof(uint32_t) * K, ctx->stream));
  // grid.y is limited to 65535 row tiles per launch: slice very tall operands
  const int64_t rows_per_launch = (int64_t)65535 * mmmcu::kK1Rows;
  for (int64_t r0 = 0; r0 < M; r0 += rows_per_launch) {
    const int64_t mr = std::min(rows_per_launch, M - r0);
    dim3 grid((unsigned)((K + mmmcu::kK1Cols - 1) / mmmcu::kK1Cols), (unsigned)((mr + mmmcu::kK1Rows - 1) / mmmcu::kK1Rows));
    mmmcu::k1_a_pass<<<grid, mmmcu::kK1Threads, 0, ctx->stream>>>(A + r0 * lda, mr, K, lda,
                                                                    ctx->abits.as<uint32_t>() + r0 * kw, kw,
                                                                    ctx->arow.as<uint32_t>() + r0, ctx->acol.as<uint32_t>());
    MMMCU_LAUNCHED();
  }
  mmmcu::k1_scan_rows<<<1, 1024, 0, ctx->stream>>>(ctx->arow.as<uint32_t>(), M, ctx->row_ptr.as<int64_t>());
  MMMCU_LAUNCHED();
  const unsigned csr_blocks = (unsigned)((M + 7) / 8);
  if (ctx->csr_idx_bytes == 2)
    mmmcu::k1_csr<uint16_t><<<csr_blocks, 256, 0, ctx->stream>>>(ctx->abits.as<uint32_t>(), M, kw,
                                                                 ctx->row_ptr.as<int64_t>(), ctx->cols.as<uint16_t>());
  else
    mmmcu::k1_csr<uint32_t><<<csr_blocks, 256, 0, ctx->stream>>>(ctx->abits.as<uint32_t>(), M, kw,
                                                                 ctx->row_ptr.as<int64_t>(), ctx->cols.as<uint32_t>());
  MMMCU_LAUNCHED();
  ctx->has_a = true;
  ctx->A = A;
  ctx->M = M;
  ctx->Ka = K;
  ctx->lda = lda;
  ctx->av = av;
  return MMMCU_OK;
}

mmmcu_status do_preprocess_b(mmmcu_ctx* ctx, const float* B, int64_t K, int64_t N, int64_t ldb, uint64_t bv) {
  if (K <= 0 || N <= 0) return fail(ctx, MMMCU_ERR_INVALID_ARG, "matrix dimensions must be positive");
  if (!B) return fail(ctx, MMMCU_ERR_INVALID_ARG, "B is null");
  if (ldb < N || ldb % 64 != 0 || !aligned16(B))
    return fail(ctx, MMMCU_ERR_INVALID_ARG,
                "B must be 16-byte aligned with ldb >= N and ldb a multiple of the region width 64");
  const int64_t kw = (K + 31) / 32;
  if (kw > 65535) return fail(ctx, MMMCU_ERR_UNSUPPORTED, "K larger than 2097120 is not supported");
  const int64_t nreg = ldb / 64, ngrp = ldb / 8;
  ctx->has_b = false;
  MMMCU_CUDA(ctx->codes.ensure((size_t)K * nreg));
  MMMCU_CUDA(ctx->bgrp.ensure(sizeof(uint32_t) * ngrp * kw));
  MMMCU_CUDA(ctx->bpop.ensure(sizeof(uint32_t) * K));
  MMMCU_CUDA(ctx->bnz.ensure(sizeof(uint32_t) * K));
  MMMCU_CUDA(ctx->stats.ensure(sizeof(unsigned long long) * 16));
  MMMCU_CUDA(cudaMemsetAsync(ctx->bpop.p, 0, sizeof(uint32_t) * K, ctx->stream));
  MMMCU_CUDA(cudaMemsetAsync(ctx->bnz.p, 0, sizeof(uint32_t) * K, ctx->stream));
  MMMCU_CUDA(cudaMemsetAsync(ctx->stats.as<unsigned long long>() + 8, 0, sizeof(unsigned long long), ctx->stream));
  dim3 grid((unsigned)((ldb + mmmcu::kK1Cols - 1) / mmmcu::kK1Cols), (unsigned)kw);
  mmmcu::k1_b_pass<<<grid, mmmcu::kK1Threads, 0, ctx->stream>>>(
      B, K, ldb, ctx->codes.as<uint8_t>(), nreg, ctx->bgrp.as<uint32_t>(), kw, ctx->bpop.as<uint32_t>(),
      ctx->bnz.as<uint32_t>(), ctx->stats.as<unsigned long long>() + 8);
  MMMCU_LAUNCHED();
  ctx->has_b = true;
  ctx->B = B;
  ctx->Kb = K;
  ctx->N = N;
  ctx->ldb = ldb;
  ctx->bv = bv;
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

// span_hint 8 / 16 forces a variant; 0 launches both and lets k1_finalize's device-side
// choice (stats[7]) gate them, so AUTO never synchronises the stream between K1 and K2.
mmmcu_status launch_simt(mmmcu_ctx* ctx, float* C, int64_t ldc, int span_hint) {
  const int64_t M = ctx->M, K = ctx->Ka, Np = round_up(ctx->N, 64);
  const int64_t kw = (K + 31) / 32;
  const int64_t row_tiles = (M + mmmcu::kK2TM - 1) / mmmcu::kK2TM;
  if (row_tiles > 65535) return fail(ctx, MMMCU_ERR_UNSUPPORTED, "M larger than 8388480 rows");
  dim3 grid((unsigned)((Np + mmmcu::kK2TN - 1) / mmmcu::kK2TN), (unsigned)row_tiles);
  MMMCU_CUDA(cudaFuncSetAttribute(mmmcu::k2_simt_bcast<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, mmmcu::kK2Smem));
  MMMCU_CUDA(cudaFuncSetAttribute(mmmcu::k2_simt_bcast<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, mmmcu::kK2Smem));
  const unsigned long long* sel = span_hint == 0 ? ctx->stats.as<unsigned long long>() + 7 : nullptr;
  if (span_hint == 0 || span_hint == 8) {
    mmmcu::k2_simt_bcast<8><<<grid, mmmcu::kK2Threads, mmmcu::kK2Smem, ctx->stream>>>(
        ctx->A, ctx->lda, ctx->B, ctx->ldb, C, ldc, M, K, Np, ctx->bgrp.as<uint32_t>(), kw, sel);
    MMMCU_LAUNCHED();
  }
  if (span_hint == 0 || span_hint == 16) {
    mmmcu::k2_simt_bcast<16><<<grid, mmmcu::kK2Threads, mmmcu::kK2Smem, ctx->stream>>>(
        ctx->A, ctx->lda, ctx->B, ctx->ldb, C, ldc, M, K, Np, ctx->bgrp.as<uint32_t>(), kw, sel);
    MMMCU_LAUNCHED();
  }
  return MMMCU_OK;
}

mmmcu_status read_stats(mmmcu_ctx* ctx, unsigned long long* host16) {
  MMMCU_CUDA(cudaMemcpyAsync(host16, ctx->stats.p, sizeof(unsigned long long) * 16, cudaMemcpyDeviceToHost, ctx->stream));
  MMMCU_CUDA(cudaStreamSynchronize(ctx->stream));
  return MMMCU_OK;
}

mmmcu_status fill_counters(mmmcu_ctx* ctx, mmmcu_counters* out) {
  if (!out) return MMMCU_OK;
  unsigned long long s[16];
  MMMCU_TRY(read_stats(ctx, s));
  out->kernel_invocations = s[0];
  out->lane_fma_ops = s[1];
  out->rows_skipped = s[2];
  out->regions_skipped_by_zero_code = s[3];
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
  for (DevBuf* b : {&ctx->abits, &ctx->arow, &ctx->acol, &ctx->row_ptr, &ctx->cols, &ctx->codes, &ctx->bgrp,
                    &ctx->bpop, &ctx->bnz, &ctx->stats, &ctx->hA, &ctx->hB, &ctx->hC, &ctx->scratch0, &ctx->scratch1})
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
  MMMCU_TRY(do_preprocess_a(ctx, A, M, K, lda, av));
  return run_finalize(ctx);
}

mmmcu_status mmmcu_preprocess_b(mmmcu_ctx* ctx, const float* B, int64_t K, int64_t N, int64_t ldb, mmmcu_lane lane,
                                uint64_t bv) {
  MMMCU_TRY(bind(ctx));
  MMMCU_TRY(check_lane(ctx, lane));
  MMMCU_TRY(do_preprocess_b(ctx, B, K, N, ldb, bv));
  return run_finalize(ctx);
}

mmmcu_status mmmcu_preprocess(mmmcu_ctx* ctx, const float* A, int64_t M, int64_t K, int64_t lda, const float* B,
                              int64_t N, int64_t ldb, mmmcu_lane lane, uint64_t av, uint64_t bv) {
  MMMCU_TRY(bind(ctx));
  MMMCU_TRY(check_lane(ctx, lane));
  MMMCU_TRY(do_preprocess_a(ctx, A, M, K, lda, av));
  MMMCU_TRY(do_preprocess_b(ctx, B, K, N, ldb, bv));
  return run_finalize(ctx);
}

mmmcu_status mmmcu_get_counters(mmmcu_ctx* ctx, mmmcu_counters* out) {
  MMMCU_TRY(bind(ctx));
  if (!out) return fail(ctx, MMMCU_ERR_INVALID_ARG, "out is null");
  if (!ctx->has_a && !ctx->has_b) return fail(ctx, MMMCU_ERR_NOT_READY, "no plan");
  return fill_counters(ctx, out);
}

mmmcu_status mmmcu_get_plan_stats(mmmcu_ctx* ctx, mmmcu_plan_stats* out) {
  MMMCU_TRY(bind(ctx));
  if (!out) return fail(ctx, MMMCU_ERR_INVALID_ARG, "out is null");
  if (!ctx->has_b) return fail(ctx, MMMCU_ERR_NOT_READY, "no B plan");
  unsigned long long s[16];
  MMMCU_TRY(read_stats(ctx, s));
  const int64_t n = ctx->Kb * (ctx->ldb / 64);
  out->region_count = n;
  out->zero_region_fraction = n ? (double)s[6] / (double)n : 0.0;
  out->mean_popcount = n ? (double)s[5] / (double)n : 0.0;
  return MMMCU_OK;
}

mmmcu_status mmmcu_export_b_codes(mmmcu_ctx* ctx, uint8_t* codes_host, int64_t capacity) {
  MMMCU_TRY(bind(ctx));
  if (!ctx->has_b) return fail(ctx, MMMCU_ERR_NOT_READY, "no B plan");
  const int64_t n = ctx->Kb * (ctx->ldb / 64);
  if (!codes_host || capacity < n) return fail(ctx, MMMCU_ERR_INVALID_ARG, "codes buffer too small");
  MMMCU_CUDA(cudaMemcpyAsync(codes_host, ctx->codes.p, (size_t)n, cudaMemcpyDeviceToHost, ctx->stream));
  MMMCU_CUDA(cudaStreamSynchronize(ctx->stream));
  return MMMCU_OK;
}

mmmcu_status mmmcu_export_bplans(mmmcu_ctx* ctx, int64_t leaf_dim, uint8_t* plans_host, int64_t plans_capacity,
                                 int64_t* plan_off_host, int64_t off_capacity, int64_t* n_plans) {
  MMMCU_TRY(bind(ctx));
  if (!ctx->has_b) return fail(ctx, MMMCU_ERR_NOT_READY, "no B plan");
  if (leaf_dim <= 0 || leaf_dim % 64 != 0)
    return fail(ctx, MMMCU_ERR_INVALID_ARG, "leaf_dim must be a positive multiple of the region width 64");
  const int64_t K = ctx->Kb, nreg = ctx->ldb / 64, rpl = leaf_dim / 64;
  const int64_t n_lr = (K + leaf_dim - 1) / leaf_dim, n_lc = (nreg + rpl - 1) / rpl;
  if (n_plans) *n_plans = n_lr * n_lc;
  if (!plans_host || plans_capacity < K * nreg || !plan_off_host || off_capacity < n_lr * n_lc + 1)
    return fail(ctx, MMMCU_ERR_INVALID_ARG, "plan buffers too small");
  std::vector<uint8_t> codes((size_t)(K * nreg));
  MMMCU_CUDA(cudaMemcpyAsync(codes.data(), ctx->codes.p, codes.size(), cudaMemcpyDeviceToHost, ctx->stream));
  MMMCU_CUDA(cudaStreamSynchronize(ctx->stream));
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
  if (algo < MMMCU_ALGO_AUTO || algo > MMMCU_ALGO_SIMT_SPAN16)
    return fail(ctx, MMMCU_ERR_INVALID_ARG, "unknown algorithm");
  ctx->algo = algo;
  return MMMCU_OK;
}

mmmcu_status mmmcu_last_algo(mmmcu_ctx* ctx, mmmcu_algo* algo) {
  if (!ctx || !algo) return fail(ctx, MMMCU_ERR_INVALID_ARG, "null argument");
  *algo = ctx->last_algo;
  return MMMCU_OK;
}

mmmcu_status mmmcu_multiply(mmmcu_ctx* ctx, float* C, int64_t ldc, const float* A, const float* B, uint64_t av,
                            uint64_t bv, mmmcu_counters* counters) {
  MMMCU_TRY(bind(ctx));
  MMMCU_TRY(check_plan(ctx, A, B, av, bv));
  if (!C) return fail(ctx, MMMCU_ERR_INVALID_ARG, "C is null");
  if (ldc < round_up(ctx->N, 64) || ldc % 4 != 0 || !aligned16(C))
    return fail(ctx, MMMCU_ERR_INVALID_ARG,
                "C must be 16-byte aligned with ldc >= round_up(N, 64) (Matrix padding) and ldc % 4 == 0");
  if (ctx->algo == MMMCU_ALGO_DENSE) {
    ctx->last_algo = MMMCU_ALGO_DENSE;
    dim3 grid((unsigned)((ctx->N + 63) / 64), (unsigned)((ctx->M + 63) / 64));
    mmmcu::k2_dense<<<grid, 256, 0, ctx->stream>>>(ctx->A, ctx->lda, ctx->B, ctx->ldb, C, ldc, ctx->M, ctx->Ka, ctx->N);
    MMMCU_LAUNCHED();
  } else {
    const int span = ctx->algo == MMMCU_ALGO_SIMT_SPAN8 ? 8 : ctx->algo == MMMCU_ALGO_SIMT_SPAN16 ? 16 : 0;
    ctx->last_algo = span == 8 ? MMMCU_ALGO_SIMT_SPAN8 : span == 16 ? MMMCU_ALGO_SIMT_SPAN16 : MMMCU_ALGO_SIMT_BCAST;
    MMMCU_TRY(launch_simt(ctx, C, ldc, span));
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

mmmcu_status mmmcu_multiply_host(mmmcu_ctx* ctx, float* C_host, int64_t ldc, const float* A_host, int64_t lda,
                                 const float* B_host, int64_t ldb, int64_t M, int64_t K, int64_t N,
                                 mmmcu_counters* counters) {
  MMMCU_TRY(bind(ctx));
  if (M <= 0 || K <= 0 || N <= 0) return fail(ctx, MMMCU_ERR_INVALID_ARG, "matrix dimensions must be positive");
  if (!A_host || !B_host || !C_host) return fail(ctx, MMMCU_ERR_INVALID_ARG, "null operand");
  MMMCU_CUDA(ctx->hA.ensure(sizeof(float) * M * lda));
  MMMCU_CUDA(ctx->hB.ensure(sizeof(float) * K * ldb));
  MMMCU_CUDA(ctx->hC.ensure(sizeof(float) * M * ldc));
  MMMCU_CUDA(cudaMemcpyAsync(ctx->hA.p, A_host, sizeof(float) * M * lda, cudaMemcpyHostToDevice, ctx->stream));
  MMMCU_CUDA(cudaMemcpyAsync(ctx->hB.p, B_host, sizeof(float) * K * ldb, cudaMemcpyHostToDevice, ctx->stream));
  MMMCU_CUDA(cudaMemcpyAsync(ctx->hC.p, C_host, sizeof(float) * M * ldc, cudaMemcpyHostToDevice, ctx->stream));
  const mmmcu_lane lane{8, 8, 1};
  const float* dA = ctx->hA.as<float>();
  const float* dB = ctx->hB.as<float>();
  // host operands carry no version: tag the staging copies with a per-call counter
  static thread_local uint64_t tag = 0;
  ++tag;
  MMMCU_TRY(mmmcu_preprocess(ctx, dA, M, K, lda, dB, N, ldb, lane, tag, tag));
  MMMCU_TRY(mmmcu_multiply(ctx, ctx->hC.as<float>(), ldc, dA, dB, tag, tag, nullptr));
  MMMCU_CUDA(cudaMemcpyAsync(C_host, ctx->hC.p, sizeof(float) * M * ldc, cudaMemcpyDeviceToHost, ctx->stream));
  MMMCU_CUDA(cudaStreamSynchronize(ctx->stream));
  return fill_counters(ctx, counters);
}

mmmcu_status mmmcu_generate(mmmcu_ctx* ctx, float* out, int64_t rows, int64_t cols, int64_t ld, uint64_t seed,
                            int value_kind, double sigma, double thresh, int mask_kind, double p, int64_t block) {
  MMMCU_TRY(bind(ctx));
  if (rows <= 0 || cols <= 0 || ld < cols || !out) return fail(ctx, MMMCU_ERR_INVALID_ARG, "bad generator shape");
  if (value_kind < 0 || value_kind > 2 || mask_kind < 0 || mask_kind > 2 || (mask_kind == 2 && block <= 0) ||
      !(p >= 0.0 && p <= 1.0))
    return fail(ctx, MMMCU_ERR_INVALID_ARG, "bad generator spec");
  const int64_t total = rows * ld;
  const unsigned blocks = (unsigned)std::min<int64_t>((total + 255) / 256, 148 * 64);
  mmmcu::k_generate<<<blocks, 256, 0, ctx->stream>>>(out, rows, cols, ld, seed, value_kind, sigma, thresh, mask_kind, p,
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

}  // extern "C"
