/*
 * mmmcu.h — C ABI of the B200-native masked matrix multiply (arXiv 2402.14118).
 *
 * This is the drop-in boundary of the hot path.  The reference's plugin
 * point is the per-region function-pointer table `KernelFn<T>` dispatched by
 * `KernelTable<T>::apply` (/root/reference/proj/include/mmm/kernel_table.hpp:12-13, :50-54);
 * per-region host function pointers cannot dispatch device work, so the boundary moves up
 * one level to the SPEC engine entry points, which the C++ drop-in
 * header include/mmm_cuda.hpp re-exposes with the SPEC signatures on top of this ABI.
 *
 * Conventions
 *   - Plain C: pointers, int64 sizes, strides in ELEMENTS.  No torch, no C++ types.
 *   - Every entry point returns an mmmcu_status; 0 is success.  The message of the last
 *     failure on a context is mmmcu_last_error(ctx) (thread-local when ctx is NULL).
 *   - Device pointers unless the name says _host.  All work is enqueued on the context's
 *     stream (mmmcu_set_stream); results are valid after that stream completes, except
 *     for calls that return host data (they synchronise the stream).
 *   - Operand layout is the reference Matrix<float> layout (matrix.hpp:61-83): row-major,
 *     element (i, j) at i*ld + j, ld a multiple of the region width R = W*P*V (64 for the
 *     f32 defaults) and columns [cols, ld) exactly zero.
 *   - The f32 default lane config {W=8, P=8, V=1} (matrix.hpp:36-38) runs the fused K1 / K2
 *     kernels; every other valid lane config (G = W*V in {1, 2, ..., 64}, P in [1, 16]) and
 *     f64 (the *_t entry points) run the lane-general kernels (kgen.cuh), bit-identical to
 *     the reference's KernelTable<T>.  There is no CPU fallback.
 */
#ifndef MMMCU_H_
#define MMMCU_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MMMCU_ABI_VERSION 1

typedef enum {
  MMMCU_OK = 0,
  MMMCU_ERR_INVALID_ARG = 1,   /* std::invalid_argument: dims <= 0, lane fields, p range (matrix.hpp:72-74, kernel_table.cpp:66-72) */
  MMMCU_ERR_DIM_MISMATCH = 2,  /* SPEC.md:262, :271 dimension mismatch */
  MMMCU_ERR_STALE = 3,         /* SPEC.md:280 stale context (content-version mismatch) */
  MMMCU_ERR_UNSUPPORTED = 4,   /* dtype / lane config without a GPU kernel */
  MMMCU_ERR_CUDA = 5,          /* CUDA runtime failure */
  MMMCU_ERR_NOT_READY = 6,     /* multiply before preprocess */
  MMMCU_ERR_OVERFLOW = 7,      /* std::overflow_error (matrix.hpp:77-80) */
  MMMCU_ERR_WORKERS = 8,       /* SPEC.md:290 worker_count == 0 */
  MMMCU_ERR_NO_DEVICE = 9,     /* no CUDA device: the product never falls back to the CPU */
  MMMCU_ERR_FILE_IO = 10,      /* IoError (matrix_io.hpp:27-29): open / write failures */
  MMMCU_ERR_FILE_FORMAT = 11,  /* BadMagicError, UnknownDtypeError, bad version (matrix_io.hpp:18-26) */
  MMMCU_ERR_FILE_TRUNCATED = 12 /* TruncatedFileError (matrix_io.hpp:21-23) */
} mmmcu_status;

typedef struct mmmcu_ctx mmmcu_ctx;

/* Dtype (matrix.hpp:13-26): f32 = 0, f64 = 1. */
typedef enum { MMMCU_F32 = 0, MMMCU_F64 = 1 } mmmcu_dtype;

/* LaneConfig (matrix.hpp:31-44). */
typedef struct {
  int32_t w, p, v;
} mmmcu_lane;

/* WorkCounters (SPEC.md:252-255; semantics :279, :297-298). */
typedef struct {
  uint64_t kernel_invocations;           /* (non-zero a_ik, region with code != 0) pairs */
  uint64_t lane_fma_ops;                 /* Σ popcount(code) * W * V over those pairs      */
  uint64_t rows_skipped;                 /* zero A elements (a whole B row skipped)        */
  uint64_t regions_skipped_by_zero_code; /* (non-zero a_ik, region with code == 0) pairs   */
} mmmcu_counters;

/* plan_stats. */
typedef struct {
  int64_t region_count;
  double zero_region_fraction;
  double mean_popcount;
} mmmcu_plan_stats;

/* Kernel-variant selection for mmmcu_multiply (all variants honour the same contract). */
typedef enum {
  MMMCU_ALGO_AUTO = 0,       /* K1's cost model picks K2-SIMT or K2-TC on the device (no
                                host round trip); C within the tolerance below           */
  MMMCU_ALGO_SIMT_BCAST = 1, /* K2-SIMT: warp-uniform k over B block masks, exact fp32
                                (bit-identical to the reference's fmaf chain); mask
                                granularity (8 or 16 columns) chosen on the device         */
  MMMCU_ALGO_DENSE = 2,      /* multiply_simple (dense i-k-j fma)            */
  MMMCU_ALGO_SIMT_SPAN8 = 3, /* K2-SIMT forced to 8-column (group) masks                  */
  MMMCU_ALGO_SIMT_SPAN16 = 4,/* K2-SIMT forced to 16-column slice masks                   */
  MMMCU_ALGO_TC = 5,         /* K2-TC: tcgen05 3-term fp16 split (kind::f16, operands
                                scaled by powers of two) on 128x192 C tiles over each
                                tile's live k; tolerance-matched (|dC| <= 1e-5 * (|c0| +
                                sum|a||b|)), not bit-exact                                 */
  MMMCU_ALGO_TC32 = 6,       /* K2-TC with the 3xTF32 split (kind::tf32): same tiles and
                                tolerance, half the k per MMA; no operand scaling          */
  MMMCU_ALGO_CSR = 7         /* K2-CSR: only the surviving (a_ik != 0, live B block) pairs,
                                C tiles in shared memory; exact fp32 (bit-identical to the
                                reference kernel table) — for very sparse / skinny A        */
} mmmcu_algo;

/* ---- context --------------------------------------------------------------------- */

/* Bind a context to CUDA device `device`.  MMMCU_ERR_NO_DEVICE when none is present. */
mmmcu_status mmmcu_ctx_create(int device, mmmcu_ctx** out);
mmmcu_status mmmcu_ctx_destroy(mmmcu_ctx* ctx);
/* Stream all subsequent work is enqueued on (a cudaStream_t; NULL = legacy default). */
mmmcu_status mmmcu_set_stream(mmmcu_ctx* ctx, void* stream);
const char* mmmcu_last_error(const mmmcu_ctx* ctx);
int mmmcu_abi_version(void);

/* KernelTable<T>::build validation (kernel_table.cpp:64-92): 0 if the lane config is
 * valid for f32, MMMCU_ERR_INVALID_ARG with the reference's message otherwise. */
mmmcu_status mmmcu_validate_lane(mmmcu_ctx* ctx, mmmcu_lane lane);

/* ---- preprocessing (K1) ------------------------------------------------------------ */

/*
 * preprocess_a + preprocess_b of SPEC.md:196-214 in one pass over A (M x K, lda) and
 * B (K x N, ldb), device pointers.  Builds, in context-owned device memory:
 *   A: per-row non-zero bitmap (uint32 [M][ceil(K/32)], LSB-first), per-row non-zero
 *      counts, per-row ascending index lists (CSR, uint32 columns), column counts;
 *   B: pattern codes (uint8 [K][ldb/64], MSB-first == BPlan codes), per-8-column-group
 *      k-bitmaps (transposed block masks), per-row code statistics;
 *   the exact WorkCounters and plan_stats of the coming multiply.
 * a_version / b_version are the operands' content versions (Matrix::version(),
 * matrix.hpp:115); mmmcu_multiply rejects other versions as stale.
 */
mmmcu_status mmmcu_preprocess(mmmcu_ctx* ctx, const float* A, int64_t M, int64_t K, int64_t lda,
                              const float* B, int64_t N, int64_t ldb, mmmcu_lane lane,
                              uint64_t a_version, uint64_t b_version);

/* Only A's half (preprocess_a): bitmap, counts, CSR, column counts. */
mmmcu_status mmmcu_preprocess_a(mmmcu_ctx* ctx, const float* A, int64_t M, int64_t K, int64_t lda,
                                uint64_t a_version);

/* Only B's half (preprocess_b): codes + group bitmaps + row statistics. */
mmmcu_status mmmcu_preprocess_b(mmmcu_ctx* ctx, const float* B, int64_t K, int64_t N, int64_t ldb,
                                mmmcu_lane lane, uint64_t b_version);

/* Counters and plan statistics of the current plan (synchronises the stream). */
mmmcu_status mmmcu_get_counters(mmmcu_ctx* ctx, mmmcu_counters* out);
mmmcu_status mmmcu_get_plan_stats(mmmcu_ctx* ctx, mmmcu_plan_stats* out);

/* ---- exports of the canonical plan formats (host destination buffers) -------------- */

/* Pattern codes, row-major uint8 [K][ldb/64] (SPEC BPlan codes before leaf ordering). */
mmmcu_status mmmcu_export_b_codes(mmmcu_ctx* ctx, uint8_t* codes_host, int64_t capacity);
/* BPlan order: per leaf_dim x leaf_dim sub-block, leaf-row-major;
 * inside a leaf, rows then regions.  plans_host has K*ldb/64 entries, plan_off_host
 * n_plans + 1; *n_plans receives the plan count. */
mmmcu_status mmmcu_export_bplans(mmmcu_ctx* ctx, int64_t leaf_dim, uint8_t* plans_host,
                                 int64_t plans_capacity, int64_t* plan_off_host,
                                 int64_t off_capacity, int64_t* n_plans);
/* A bitmap, uint32 [M][ceil(K/32)], LSB-first. */
mmmcu_status mmmcu_export_a_bitmap(mmmcu_ctx* ctx, uint32_t* bits_host, int64_t capacity);
/* A CSR: row_ptr int64 [M+1], ascending uint32 columns [nnz]; *nnz receives nnz(A). */
mmmcu_status mmmcu_export_a_csr(mmmcu_ctx* ctx, int64_t* row_ptr_host, uint32_t* cols_host,
                                int64_t cols_capacity, int64_t* nnz);
/* ABlockIndex: block_dim x block_dim blocks of A, block-major;
 * per block row, per aligned 8-element segment: count + 8 offset slots (0xFF unused; a
 * full segment stores none).  *n_segments receives the segment count. */
mmmcu_status mmmcu_export_ablock_index(mmmcu_ctx* ctx, int64_t block_dim, uint8_t* counts_host,
                                       int64_t counts_capacity, uint8_t* offsets_host,
                                       int64_t offsets_capacity, int64_t* n_segments);

/* ---- masked multiply (K2) ---------------------------------------------------------- */

/*
 * multiply_mmm: C (M x N, ldc) += A * B over the masks of the current
 * plan.  A and B must be the preprocessed operands (same pointers, same versions).
 * Accuracy depends on the algorithm (mmmcu_set_algo):
 *   MMMCU_ALGO_SIMT_*, MMMCU_ALGO_CSR and MMMCU_ALGO_DENSE: each C element receives the ascending-k fmaf
 *     chain of its surviving terms, bit-identical to the CPU oracle / reference kernel table;
 *   MMMCU_ALGO_AUTO (default), MMMCU_ALGO_TC, MMMCU_ALGO_TC32: the north_star tolerance,
 *     |dC| <= 1e-5 * (|c0| + sum_k |a_ik||b_kj|), not bit-exact (AUTO runs an exact SIMT
 *     kernel whenever its guards — Inf / NaN / subnormal operands, mixed-scale rows or
 *     groups — or its cost model say so).
 * counters may be NULL; filling it synchronises the stream.
 */
mmmcu_status mmmcu_multiply(mmmcu_ctx* ctx, float* C, int64_t ldc, const float* A, const float* B,
                            uint64_t a_version, uint64_t b_version, mmmcu_counters* counters);
/* multiply_parallel: worker_count == 0 is rejected; otherwise the same
 * computation (the GPU's parallelism is not a host worker count). */
mmmcu_status mmmcu_multiply_parallel(mmmcu_ctx* ctx, float* C, int64_t ldc, const float* A,
                                     const float* B, uint64_t a_version, uint64_t b_version,
                                     int worker_count, mmmcu_counters* counters);
/* Force a kernel variant (MMMCU_ALGO_AUTO by default). */
mmmcu_status mmmcu_set_algo(mmmcu_ctx* ctx, mmmcu_algo algo);
/* Variant the last mmmcu_multiply ran (AUTO and SIMT_BCAST resolve to the kernel the
 * device chose: TC, CSR, SIMT_SPAN8 or SIMT_SPAN16; synchronises the stream). */
mmmcu_status mmmcu_last_algo(mmmcu_ctx* ctx, mmmcu_algo* algo);

/* multiply_simple: dense i-k-j C += A*B, fmaf per term. */
mmmcu_status mmmcu_multiply_simple(mmmcu_ctx* ctx, float* C, int64_t ldc, const float* A,
                                   int64_t lda, const float* B, int64_t ldb, int64_t M, int64_t K,
                                   int64_t N);

/* ---- every dtype and lane config of the reference ---------------
 * Typed (void*) twins of the calls above: dtype MMMCU_F32 with the default lane forwards to
 * them; f32 with another lane and f64 with any lane build a lane-general plan (pattern codes
 * of P bits per region of R = W*P*V columns, MSB first; the same A bitmap / CSR) and the
 * multiply is the reference's per-element fma chain over it (exact, bit-identical to
 * KernelTable<T>).  Operands are Matrix<T> layouts: ldb a multiple of R, ldc >= ldb. */
mmmcu_status mmmcu_validate_lane_t(mmmcu_ctx* ctx, mmmcu_dtype dtype, mmmcu_lane lane);
mmmcu_status mmmcu_preprocess_a_t(mmmcu_ctx* ctx, mmmcu_dtype dtype, const void* A, int64_t M, int64_t K,
                                  int64_t lda, uint64_t a_version);
mmmcu_status mmmcu_preprocess_b_t(mmmcu_ctx* ctx, mmmcu_dtype dtype, const void* B, int64_t K, int64_t N,
                                  int64_t ldb, mmmcu_lane lane, uint64_t b_version);
mmmcu_status mmmcu_preprocess_t(mmmcu_ctx* ctx, mmmcu_dtype dtype, const void* A, int64_t M, int64_t K,
                                int64_t lda, const void* B, int64_t N, int64_t ldb, mmmcu_lane lane,
                                uint64_t a_version, uint64_t b_version);
mmmcu_status mmmcu_multiply_t(mmmcu_ctx* ctx, mmmcu_dtype dtype, void* C, int64_t ldc, const void* A,
                              const void* B, uint64_t a_version, uint64_t b_version,
                              mmmcu_counters* counters);
mmmcu_status mmmcu_multiply_simple_t(mmmcu_ctx* ctx, mmmcu_dtype dtype, void* C, int64_t ldc,
                                     const void* A, int64_t lda, const void* B, int64_t ldb,
                                     int64_t M, int64_t K, int64_t N);
/* Pattern codes of any plan as uint16 [K][ldb/R] (P up to 16), and the BPlan order of them. */
mmmcu_status mmmcu_export_b_codes16(mmmcu_ctx* ctx, uint16_t* codes_host, int64_t capacity);
mmmcu_status mmmcu_export_bplans16(mmmcu_ctx* ctx, int64_t leaf_dim, uint16_t* plans_host,
                                   int64_t plans_capacity, int64_t* plan_off_host,
                                   int64_t off_capacity, int64_t* n_plans);
/* dtype and {G, P, 1} of the current B plan. */
mmmcu_status mmmcu_plan_info(mmmcu_ctx* ctx, mmmcu_dtype* dtype, mmmcu_lane* lane);

/* ---- host-buffer convenience (the drop-in path for host Matrix<float> operands) ------- */

/*
 * preprocess + multiply with HOST operands: copies A, B and C to the device, runs K1 and
 * K2, copies C back.  Device staging buffers are owned (and reused) by the context.
 */
mmmcu_status mmmcu_multiply_host(mmmcu_ctx* ctx, float* C_host, int64_t ldc, const float* A_host,
                                 int64_t lda, const float* B_host, int64_t ldb, int64_t M,
                                 int64_t K, int64_t N, mmmcu_counters* counters);

/*
 * Plan-owning host path used by the C++ drop-in (include/mmm_cuda.hpp): copy host A and B
 * (reference Matrix<float> layout) into context-owned device buffers and preprocess them;
 * later multiplies of that plan check the operands' content versions and
 * move only C.
 */
mmmcu_status mmmcu_preprocess_host(mmmcu_ctx* ctx, const float* A_host, int64_t M, int64_t K, int64_t lda,
                                   const float* B_host, int64_t N, int64_t ldb, mmmcu_lane lane,
                                   uint64_t a_version, uint64_t b_version);
mmmcu_status mmmcu_multiply_planned_host(mmmcu_ctx* ctx, float* C_host, int64_t ldc, uint64_t a_version,
                                         uint64_t b_version, int worker_count, mmmcu_counters* counters);
/* Typed twins of the three host-buffer calls (f32 / f64, any valid lane), and multiply_simple
 * on host operands. */
mmmcu_status mmmcu_multiply_simple_host_t(mmmcu_ctx* ctx, mmmcu_dtype dtype, void* C_host, int64_t ldc,
                                          const void* A_host, int64_t lda, const void* B_host, int64_t ldb,
                                          int64_t M, int64_t K, int64_t N);
mmmcu_status mmmcu_multiply_host_t(mmmcu_ctx* ctx, mmmcu_dtype dtype, void* C_host, int64_t ldc,
                                   const void* A_host, int64_t lda, const void* B_host, int64_t ldb,
                                   int64_t M, int64_t K, int64_t N, mmmcu_lane lane,
                                   mmmcu_counters* counters);
mmmcu_status mmmcu_preprocess_host_t(mmmcu_ctx* ctx, mmmcu_dtype dtype, const void* A_host, int64_t M,
                                     int64_t K, int64_t lda, const void* B_host, int64_t N, int64_t ldb,
                                     mmmcu_lane lane, uint64_t a_version, uint64_t b_version);
mmmcu_status mmmcu_multiply_planned_host_t(mmmcu_ctx* ctx, mmmcu_dtype dtype, void* C_host, int64_t ldc,
                                           uint64_t a_version, uint64_t b_version, int worker_count,
                                           mmmcu_counters* counters);

/* ---- synthetic inputs (device generator; matgen.hpp analogue for BASELINE.json) ------ */

/*
 * Fill out (rows x ld, device) with the seeded i.i.d. generator of SURVEY.md §8(d), built
 * on the reference's counter hash (rng.hpp:8-26).  Row r of `out` is global row row0 + r
 * of the matrix the seed defines (so row shards generate their own slice):
 *   value_kind 0 uniform[-1,1], 1 N(0, sigma), 2 ReLU(N(0,1) - thresh);
 *   mask_kind  0 none, 1 element zero with prob p, 2 aligned `block`-wide runs zero with
 *              prob p.  Columns [cols, ld) are zeroed.
 */
mmmcu_status mmmcu_generate(mmmcu_ctx* ctx, float* out, int64_t rows, int64_t cols, int64_t ld,
                            int64_t row0, uint64_t seed, int value_kind, double sigma, double thresh,
                            int mask_kind, double p, int64_t block);

/* Row partition of a sharded multiply: rank r of `world` owns [*row0, *row1). */
mmmcu_status mmmcu_shard_rows(int64_t M, int world, int rank, int64_t* row0, int64_t* row1);
/* Column partition (skinny A): rank r owns columns [*col0, *col1), whole 64-column regions. */
mmmcu_status mmmcu_shard_cols(int64_t N, int world, int rank, int64_t* col0, int64_t* col1);

/* ---- multi-GPU (one process, one context + stream per GPU; csrc/mmmcu_group.cu) -------
 *
 * multiply_parallel's row partition (the reference runs it with OpenMP,
 * /root/reference/proj/include/mmm/matrix.hpp:170) spread over the GPUs of one box, as
 * north_star puts it: A/C rows are sharded (mmmcu_shard_rows), B is broadcast ONCE over
 * NVLink with NCCL (ncclCommInitAll + ncclBroadcast from devices[0]; NCCL is dlopen'ed), and
 * each GPU runs K1 + K2 on its rows with no further exchange.  A group whose device list
 * repeats a device replicates with device copies instead (NCCL rejects duplicate devices).
 */
typedef struct mmmcu_group mmmcu_group;

mmmcu_status mmmcu_group_create(int ngpus, const int* devices, mmmcu_group** out);
mmmcu_status mmmcu_group_destroy(mmmcu_group* g);
const char* mmmcu_group_last_error(const mmmcu_group* g);
int mmmcu_group_size(const mmmcu_group* g);
int mmmcu_group_uses_nccl(const mmmcu_group* g);
/* The per-rank context (device devices[rank]); owned by the group. */
mmmcu_ctx* mmmcu_group_ctx(mmmcu_group* g, int rank);
mmmcu_status mmmcu_group_set_algo(mmmcu_group* g, mmmcu_algo algo);

/*
 * Row-sharded multiply_parallel: C = C + A * B over g ranks.  A_shards[r] / C_shards[r] hold
 * rows mmmcu_shard_rows(M, g, r) on devices[r] (strides lda / ldc); B (K x N, ldb a multiple
 * of 64, Matrix layout) lives on devices[0] and is broadcast to the other ranks when its
 * pointer or b_version changed since the last call (*broadcast_ms = its wall time, 0 when
 * skipped).  Each rank re-preprocesses only when its operands or versions changed.  Returns
 * after every rank finished; counters (may be NULL) are summed over the ranks.
 */
mmmcu_status mmmcu_multiply_sharded(mmmcu_group* g, float* const* C_shards, int64_t ldc, const float* const* A_shards,
                                    int64_t lda, const float* B, int64_t ldb, int64_t M, int64_t K, int64_t N,
                                    uint64_t a_version, uint64_t b_version, mmmcu_counters* counters,
                                    double* broadcast_ms);
/*
 * Column-sharded variant for skinny A (M too small to row-shard, BASELINE configs[3]): rank r
 * owns columns mmmcu_shard_cols(N, g, r); A (M x K, lda) on devices[0] is broadcast, rank r's
 * B slab is copied peer-to-peer from B on devices[0], and C_slabs[r] (M x slab width, ldc)
 * on devices[r] receives C[:, col0:col1] += A * B[:, col0:col1].
 */
mmmcu_status mmmcu_multiply_sharded_cols(mmmcu_group* g, float* const* C_slabs, int64_t ldc, const float* A, int64_t lda,
                                         const float* B, int64_t ldb, int64_t M, int64_t K, int64_t N,
                                         uint64_t a_version, uint64_t b_version, mmmcu_counters* counters,
                                         double* broadcast_ms);

/* ---- MMMB files <-> device memory (csrc/mmmcu_io.cu) ----------------------------------
 *
 * The reference's interchange format (/root/reference/proj/include/mmm/matrix_io.hpp:11-13):
 * "MMMB" | u32 version 1 | u32 dtype (0 f32, 1 f64) | u64 rows | u64 cols | row-major payload.
 * These replace write_matrix / read_matrix / peek_dtype (matrix_io.hpp:32-49) for device
 * operands: the payload streams through pinned staging straight into the Matrix layout on the
 * device (ld columns per row, padding zeroed).  f64 files are MMMCU_ERR_UNSUPPORTED.  The
 * message of the last failure of these calls is mmmcu_io_last_error().
 */
const char* mmmcu_io_last_error(void);
mmmcu_status mmmcu_mmmb_peek(const char* path, int32_t* dtype, int64_t* rows, int64_t* cols);
/* Load into dev (max_rows x ld floats, cudaStream_t stream); *rows / *cols receive the shape.
 * Synchronises the stream before returning. */
mmmcu_status mmmcu_mmmb_load(const char* path, float* dev, int64_t ld, int64_t max_rows, void* stream, int64_t* rows,
                             int64_t* cols);
mmmcu_status mmmcu_mmmb_save(const char* path, const float* dev, int64_t rows, int64_t cols, int64_t ld, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* MMMCU_H_ */
