// mmmcu_group.cu — single-process multi-GPU entry points of the C ABI (include/mmmcu.h,
// SURVEY.md §8(e)).
//
// The reference parallelises multiply_parallel with OpenMP over C's rows inside one host
// (/root/reference/proj/include/mmm/matrix.hpp:170).  On one 8xB200 box the
// same row partition becomes a partition over GPUs (north_star): rank r of g owns A/C rows
// mmmcu_shard_rows(M, g, r), B is broadcast ONCE over NVLink with NCCL (ncclBroadcast from
// devices[0], one communicator per device from ncclCommInitAll), and every GPU runs K1 + K2
// on its own rows with no further exchange (C stays sharded).  Skinny operands (configs[3]:
// M = 64) do not row-shard: mmmcu_multiply_sharded_cols splits B / C by 64-column slabs and
// broadcasts A instead.
//
// Built only on the public per-device ABI (mmmcu_preprocess / mmmcu_multiply on one context
// and stream per GPU); ranks run concurrently, the host waits once at the end.  NCCL is
// dlopen'ed (libnccl.so.2), so the library does not pin an NCCL build and shares the one a
// host process (e.g. torch) already loaded.  A group whose device list repeats a device
// (tests on a single GPU) makes its replicas with device copies instead of NCCL, which
// rejects duplicate devices.
#include "../../include/mmmcu.h"

#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <string>
#include <vector>

namespace {

thread_local std::string g_group_err;

struct NcclApi {
  bool tried = false;
  void* h = nullptr;
  ncclResult_t (*comm_init_all)(ncclComm_t*, int, const int*) = nullptr;
  ncclResult_t (*broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*group_start)() = nullptr;
  ncclResult_t (*group_end)() = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
  bool ok() const { return comm_init_all && broadcast && group_start && group_end && comm_destroy; }
};

NcclApi& nccl() {
  static NcclApi a;
  if (!a.tried) {
    a.tried = true;
    for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
      a.h = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
      if (a.h) break;
    }
    if (a.h) {
      a.comm_init_all = reinterpret_cast<decltype(a.comm_init_all)>(dlsym(a.h, "ncclCommInitAll"));
      a.broadcast = reinterpret_cast<decltype(a.broadcast)>(dlsym(a.h, "ncclBroadcast"));
      a.group_start = reinterpret_cast<decltype(a.group_start)>(dlsym(a.h, "ncclGroupStart"));
      a.group_end = reinterpret_cast<decltype(a.group_end)>(dlsym(a.h, "ncclGroupEnd"));
      a.comm_destroy = reinterpret_cast<decltype(a.comm_destroy)>(dlsym(a.h, "ncclCommDestroy"));
      a.error_string = reinterpret_cast<decltype(a.error_string)>(dlsym(a.h, "ncclGetErrorString"));
    }
  }
  return a;
}

struct Buf {
  void* p = nullptr;
  size_t cap = 0;
  int dev = 0;
};

int64_t round_up64(int64_t x) { return (x + 63) / 64 * 64; }

}  // namespace

struct mmmcu_group {
  int n = 0;
  std::vector<int> dev;
  std::vector<mmmcu_ctx*> ctx;
  std::vector<cudaStream_t> st;
  std::vector<ncclComm_t> comm;
  bool use_nccl = false;
  std::vector<Buf> rep;   // replicas of the broadcast operand (B: row split, A: column split)
  std::vector<Buf> slab;  // column split: this rank's B slab
  // what the replicas hold (a repeated call with the same operand and version skips the broadcast)
  const void* rep_src = nullptr;
  uint64_t rep_version = 0;
  int64_t rep_elems = -1;
  int rep_kind = -1;
  // what each rank last preprocessed (plan reuse, SPEC.md:250 staleness by version)
  std::vector<const void*> plan_a, plan_b;
  std::vector<uint64_t> plan_av, plan_bv;
  std::string err;
};

namespace {

mmmcu_status gfail(mmmcu_group* g, mmmcu_status s, const std::string& m) {
  if (g) g->err = m;
  g_group_err = m;
  return s;
}

#define G_CUDA(call)                                                                                      \
  do {                                                                                                    \
    cudaError_t e_ = (call);                                                                              \
    if (e_ != cudaSuccess) return gfail(g, MMMCU_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
  } while (0)

mmmcu_status ensure(mmmcu_group* g, Buf& b, int dev, size_t bytes) {
  if (b.p && b.cap >= bytes && b.dev == dev) return MMMCU_OK;
  G_CUDA(cudaSetDevice(dev));
  if (b.p) cudaFree(b.p);
  b.p = nullptr;
  b.cap = 0;
  G_CUDA(cudaMalloc(&b.p, bytes));
  b.cap = bytes;
  b.dev = dev;
  return MMMCU_OK;
}

// Replicate `elems` floats at src (on dev[0]) into rep[r] for r >= 1 (rank 0 reads src in
// place): one ncclBroadcast per rank inside a group call, or device copies for a group that
// repeats a device.  Returns the broadcast's wall time (all streams drained) in *ms.
mmmcu_status replicate(mmmcu_group* g, const float* src, int64_t elems, uint64_t version, int kind, double* ms) {
  if (ms) *ms = 0.0;
  if (g->rep_src == src && g->rep_version == version && g->rep_elems == elems && g->rep_kind == kind) return MMMCU_OK;
  for (int r = 1; r < g->n; ++r) {
    mmmcu_status s = ensure(g, g->rep[r], g->dev[r], sizeof(float) * (size_t)elems);
    if (s != MMMCU_OK) return s;
  }
  for (int r = 0; r < g->n; ++r) {  // the operand is ready on every stream's device
    G_CUDA(cudaSetDevice(g->dev[r]));
    G_CUDA(cudaStreamSynchronize(g->st[r]));
  }
  G_CUDA(cudaSetDevice(g->dev[0]));
  G_CUDA(cudaDeviceSynchronize());  // src may have been written on another stream of device 0
  const auto t0 = std::chrono::steady_clock::now();
  if (g->use_nccl) {  // (a 1-GPU group runs the root's in-place broadcast too)
    NcclApi& api = nccl();
    if (api.group_start() != ncclSuccess) return gfail(g, MMMCU_ERR_CUDA, "ncclGroupStart failed");
    for (int r = 0; r < g->n; ++r) {
      cudaSetDevice(g->dev[r]);
      void* dst = r == 0 ? const_cast<float*>(src) : g->rep[r].p;
      const ncclResult_t e = api.broadcast(src, dst, (size_t)elems, ncclFloat32, 0, g->comm[r], g->st[r]);
      if (e != ncclSuccess) {
        api.group_end();
        return gfail(g, MMMCU_ERR_CUDA, std::string("ncclBroadcast: ") + (api.error_string ? api.error_string(e) : "error"));
      }
    }
    if (api.group_end() != ncclSuccess) return gfail(g, MMMCU_ERR_CUDA, "ncclGroupEnd failed");
  } else {
    for (int r = 1; r < g->n; ++r) {
      G_CUDA(cudaSetDevice(g->dev[r]));
      G_CUDA(cudaMemcpyAsync(g->rep[r].p, src, sizeof(float) * (size_t)elems, cudaMemcpyDefault, g->st[r]));
    }
  }
  for (int r = 0; r < g->n; ++r) {
    G_CUDA(cudaSetDevice(g->dev[r]));
    G_CUDA(cudaStreamSynchronize(g->st[r]));
  }
  if (ms) *ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  g->rep_src = src;
  g->rep_version = version;
  g->rep_elems = elems;
  g->rep_kind = kind;
  return MMMCU_OK;
}

mmmcu_status ctx_fail(mmmcu_group* g, int r, mmmcu_status s) {
  return gfail(g, s, "rank " + std::to_string(r) + ": " + mmmcu_last_error(g->ctx[r]));
}

// Per rank: (re)preprocess when its operands or versions changed, multiply (no counters:
// the ranks stay concurrent), then — after every rank was enqueued — drain and sum counters.
mmmcu_status run_ranks(mmmcu_group* g, const std::vector<const float*>& A, const std::vector<int64_t>& rows,
                       int64_t K, int64_t lda, const std::vector<const float*>& B, const std::vector<int64_t>& cols,
                       const std::vector<int64_t>& ldb, const std::vector<float*>& C, int64_t ldc, uint64_t av,
                       uint64_t bv, mmmcu_counters* counters) {
  const mmmcu_lane lane{8, 8, 1};
  for (int r = 0; r < g->n; ++r) {
    if (rows[r] <= 0 || cols[r] <= 0) continue;
    if (g->plan_a[r] != A[r] || g->plan_b[r] != B[r] || g->plan_av[r] != av || g->plan_bv[r] != bv) {
      g->plan_a[r] = nullptr;
      const mmmcu_status s = mmmcu_preprocess(g->ctx[r], A[r], rows[r], K, lda, B[r], cols[r], ldb[r], lane, av, bv);
      if (s != MMMCU_OK) return ctx_fail(g, r, s);
      g->plan_a[r] = A[r];
      g->plan_b[r] = B[r];
      g->plan_av[r] = av;
      g->plan_bv[r] = bv;
    }
    const mmmcu_status s = mmmcu_multiply(g->ctx[r], C[r], ldc, A[r], B[r], av, bv, nullptr);
    if (s != MMMCU_OK) return ctx_fail(g, r, s);
  }
  mmmcu_counters sum{0, 0, 0, 0};
  for (int r = 0; r < g->n; ++r) {
    G_CUDA(cudaSetDevice(g->dev[r]));
    G_CUDA(cudaStreamSynchronize(g->st[r]));
    if (counters && rows[r] > 0 && cols[r] > 0) {
      mmmcu_counters c;
      const mmmcu_status s = mmmcu_get_counters(g->ctx[r], &c);
      if (s != MMMCU_OK) return ctx_fail(g, r, s);
      sum.kernel_invocations += c.kernel_invocations;
      sum.lane_fma_ops += c.lane_fma_ops;
      sum.rows_skipped += c.rows_skipped;
      sum.regions_skipped_by_zero_code += c.regions_skipped_by_zero_code;
    }
  }
  if (counters) *counters = sum;
  return MMMCU_OK;
}

}  // namespace

extern "C" {

const char* mmmcu_group_last_error(const mmmcu_group* g) { return g ? g->err.c_str() : g_group_err.c_str(); }

mmmcu_status mmmcu_group_create(int ngpus, const int* devices, mmmcu_group** out) {
  if (!out || ngpus <= 0 || !devices) return gfail(nullptr, MMMCU_ERR_INVALID_ARG, "bad group arguments");
  *out = nullptr;
  mmmcu_group* g = new mmmcu_group();
  g->n = ngpus;
  g->dev.assign(devices, devices + ngpus);
  g->ctx.assign(ngpus, nullptr);
  g->st.assign(ngpus, nullptr);
  g->rep.resize(ngpus);
  g->slab.resize(ngpus);
  g->plan_a.assign(ngpus, nullptr);
  g->plan_b.assign(ngpus, nullptr);
  g->plan_av.assign(ngpus, 0);
  g->plan_bv.assign(ngpus, 0);
  auto bail = [&](mmmcu_status s, const std::string& m) {
    mmmcu_group_destroy(g);
    return gfail(nullptr, s, m);
  };
  for (int r = 0; r < ngpus; ++r) {
    mmmcu_status s = mmmcu_ctx_create(devices[r], &g->ctx[r]);
    if (s != MMMCU_OK) return bail(s, std::string("rank ") + std::to_string(r) + ": " + mmmcu_last_error(nullptr));
    if (cudaSetDevice(devices[r]) != cudaSuccess || cudaStreamCreateWithFlags(&g->st[r], cudaStreamNonBlocking) != cudaSuccess)
      return bail(MMMCU_ERR_CUDA, "stream creation failed");
    s = mmmcu_set_stream(g->ctx[r], g->st[r]);
    if (s != MMMCU_OK) return bail(s, mmmcu_last_error(g->ctx[r]));
  }
  std::vector<int> sorted(g->dev);
  std::sort(sorted.begin(), sorted.end());
  const bool distinct = std::adjacent_find(sorted.begin(), sorted.end()) == sorted.end();
  if (distinct) {
    NcclApi& api = nccl();
    if (!api.ok()) return bail(MMMCU_ERR_UNSUPPORTED, "NCCL (libnccl.so.2) not found: multi-GPU groups need it");
    g->comm.assign(ngpus, nullptr);
    const ncclResult_t e = api.comm_init_all(g->comm.data(), ngpus, g->dev.data());
    if (e != ncclSuccess)
      return bail(MMMCU_ERR_CUDA, std::string("ncclCommInitAll: ") + (api.error_string ? api.error_string(e) : "error"));
    g->use_nccl = true;
  }
  *out = g;
  return MMMCU_OK;
}

mmmcu_status mmmcu_group_destroy(mmmcu_group* g) {
  if (!g) return MMMCU_OK;
  for (int r = 0; r < (int)g->st.size(); ++r)
    if (g->st[r]) {
      cudaSetDevice(g->dev[r]);
      cudaStreamSynchronize(g->st[r]);
    }
  if (g->use_nccl)
    for (ncclComm_t c : g->comm)
      if (c) nccl().comm_destroy(c);
  for (int r = 0; r < g->n; ++r) {
    for (Buf* b : {&g->rep[r], &g->slab[r]})
      if (b->p) {
        cudaSetDevice(b->dev);
        cudaFree(b->p);
      }
    if (g->ctx[r]) mmmcu_ctx_destroy(g->ctx[r]);
    if (g->st[r]) {
      cudaSetDevice(g->dev[r]);
      cudaStreamDestroy(g->st[r]);
    }
  }
  delete g;
  return MMMCU_OK;
}

int mmmcu_group_size(const mmmcu_group* g) { return g ? g->n : 0; }

int mmmcu_group_uses_nccl(const mmmcu_group* g) { return g && g->use_nccl ? 1 : 0; }

mmmcu_ctx* mmmcu_group_ctx(mmmcu_group* g, int rank) {
  return (g && rank >= 0 && rank < g->n) ? g->ctx[rank] : nullptr;
}

mmmcu_status mmmcu_group_set_algo(mmmcu_group* g, mmmcu_algo algo) {
  if (!g) return gfail(nullptr, MMMCU_ERR_INVALID_ARG, "null group");
  for (int r = 0; r < g->n; ++r) {
    const mmmcu_status s = mmmcu_set_algo(g->ctx[r], algo);
    if (s != MMMCU_OK) return ctx_fail(g, r, s);
    g->plan_a[r] = nullptr;  // the operand sets K1 builds depend on the algorithm
  }
  return MMMCU_OK;
}

mmmcu_status mmmcu_shard_cols(int64_t N, int world, int rank, int64_t* col0, int64_t* col1) {
  if (N <= 0 || world <= 0 || rank < 0 || rank >= world || !col0 || !col1)
    return gfail(nullptr, MMMCU_ERR_INVALID_ARG, "bad shard arguments");
  const int64_t w = round_up64((N + world - 1) / world);  // whole 64-column regions per rank
  *col0 = std::min<int64_t>(N, (int64_t)rank * w);
  *col1 = std::min<int64_t>(N, (int64_t)(rank + 1) * w);
  return MMMCU_OK;
}

mmmcu_status mmmcu_multiply_sharded(mmmcu_group* g, float* const* C_shards, int64_t ldc, const float* const* A_shards,
                                    int64_t lda, const float* B, int64_t ldb, int64_t M, int64_t K, int64_t N,
                                    uint64_t a_version, uint64_t b_version, mmmcu_counters* counters,
                                    double* broadcast_ms) {
  if (!g) return gfail(nullptr, MMMCU_ERR_INVALID_ARG, "null group");
  if (!C_shards || !A_shards || !B || M <= 0 || K <= 0 || N <= 0)
    return gfail(g, MMMCU_ERR_INVALID_ARG, "bad sharded multiply arguments");
  if (ldb < N || ldb % 64 != 0) return gfail(g, MMMCU_ERR_INVALID_ARG, "ldb must be >= N and a multiple of 64");
  mmmcu_status s = replicate(g, B, K * ldb, b_version, 0, broadcast_ms);
  if (s != MMMCU_OK) return s;
  std::vector<const float*> A(g->n), Bs(g->n);
  std::vector<float*> C(g->n);
  std::vector<int64_t> rows(g->n), cols(g->n, N), ldbs(g->n, ldb);
  for (int r = 0; r < g->n; ++r) {
    int64_t r0 = 0, r1 = 0;
    mmmcu_shard_rows(M, g->n, r, &r0, &r1);
    rows[r] = r1 - r0;
    A[r] = A_shards[r];
    C[r] = C_shards[r];
    Bs[r] = r == 0 ? B : static_cast<const float*>(g->rep[r].p);
    if (rows[r] > 0 && (!A[r] || !C[r])) return gfail(g, MMMCU_ERR_INVALID_ARG, "null shard pointer");
  }
  return run_ranks(g, A, rows, K, lda, Bs, cols, ldbs, C, ldc, a_version, b_version, counters);
}

mmmcu_status mmmcu_multiply_sharded_cols(mmmcu_group* g, float* const* C_slabs, int64_t ldc, const float* A, int64_t lda,
                                         const float* B, int64_t ldb, int64_t M, int64_t K, int64_t N,
                                         uint64_t a_version, uint64_t b_version, mmmcu_counters* counters,
                                         double* broadcast_ms) {
  if (!g) return gfail(nullptr, MMMCU_ERR_INVALID_ARG, "null group");
  if (!C_slabs || !A || !B || M <= 0 || K <= 0 || N <= 0)
    return gfail(g, MMMCU_ERR_INVALID_ARG, "bad sharded multiply arguments");
  if (ldb < N || lda < K || lda % 4 != 0) return gfail(g, MMMCU_ERR_INVALID_ARG, "bad leading dimensions");
  mmmcu_status s = replicate(g, A, M * lda, a_version, 1, broadcast_ms);
  if (s != MMMCU_OK) return s;
  std::vector<const float*> As(g->n), Bs(g->n);
  std::vector<float*> C(g->n);
  std::vector<int64_t> rows(g->n, M), cols(g->n), ldbs(g->n);
  // B slabs (Matrix layout: 64-padded, zero padding) copied from devices[0], peer-to-peer
  for (int r = 0; r < g->n; ++r) {
    int64_t c0 = 0, c1 = 0;
    mmmcu_shard_cols(N, g->n, r, &c0, &c1);
    cols[r] = c1 - c0;
    As[r] = r == 0 ? A : static_cast<const float*>(g->rep[r].p);
    C[r] = C_slabs[r];
    if (cols[r] <= 0) continue;
    if (!C[r]) return gfail(g, MMMCU_ERR_INVALID_ARG, "null slab pointer");
    ldbs[r] = round_up64(cols[r]);
    s = ensure(g, g->slab[r], g->dev[r], sizeof(float) * (size_t)(K * ldbs[r]));
    if (s != MMMCU_OK) return s;
    G_CUDA(cudaSetDevice(g->dev[r]));
    if (ldbs[r] != cols[r]) G_CUDA(cudaMemsetAsync(g->slab[r].p, 0, sizeof(float) * (size_t)(K * ldbs[r]), g->st[r]));
    G_CUDA(cudaMemcpy2DAsync(g->slab[r].p, sizeof(float) * ldbs[r], B + c0, sizeof(float) * ldb,
                             sizeof(float) * cols[r], (size_t)K, cudaMemcpyDefault, g->st[r]));
    Bs[r] = static_cast<const float*>(g->slab[r].p);
    g->plan_b[r] = nullptr;  // the slab was rewritten
  }
  return run_ranks(g, As, rows, K, lda, Bs, cols, ldbs, C, ldc, a_version, b_version, counters);
}

}  // extern "C"
