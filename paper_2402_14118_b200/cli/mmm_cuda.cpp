// mmm-cuda — the SPEC bench-cli (SPEC.md "bench-cli" module: gen / bench / sweep / verify /
// analyze, CSV BenchRecord schema, exit codes 0 ok, 1 verification failure, 2 usage, 3 I/O)
// on the B200 path.  Every multiply goes through the C ABI of include/mmmcu.h; the dense
// comparators are the library's multiply_simple (i-k-j fmaf, the oracle order) and cuBLAS
// SGEMM (the vendor dense GEMM, the GPU analogue of the paper's "MKL dense").
//
//   mmm-cuda gen     --rows R --cols C [--structure random|block_random] [--sparsity s]
//                    [--block-len L] [--value uniform|normal|relu] [--sigma x] [--thresh t]
//                    [--seed S] --out FILE
//   mmm-cuda bench   (--a FILE --b FILE | --n N [--a-sparsity s] [--b-sparsity s] [--block-len L]
//                    [--seed S]) [--algo mmm|mmm_exact|mmm_tc|mmm_tc32|dense|cublas|all]
//                    [--trials T] [--workers W] [--out CSV]
//   mmm-cuda sweep   --n N [--grid-step g] [--block-len L] [--trials T] [--out CSV]
//   mmm-cuda verify  (--a FILE --b FILE | --n N ...) [--tolerance 1e-5]
//   mmm-cuda analyze --matrix FILE
//
// Timings are CUDA events on the context's stream around preprocess (K1) and multiply (K2),
// generation and file I/O excluded (SPEC bench-cli design decisions); the summary row of each
// algo is the median of its trials.  The checksum hashes C's logical range rounded to 2^-16
// relative precision, so tolerance-equivalent results of different algos hash equally.
#include "../../include/mmmcu.h"

#include <cublas_v2.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <string>
#include <vector>

namespace {

constexpr int kExitOk = 0, kExitVerify = 1, kExitUsage = 2, kExitIo = 3;

struct Usage {
  std::string msg;
};
struct IoFail {
  std::string msg;
};
struct Fatal {
  std::string msg;
};

using Args = std::map<std::string, std::string>;

Args parse(int argc, char** argv, int first) {
  Args a;
  for (int i = first; i < argc; ++i) {
    std::string k = argv[i];
    if (k.rfind("--", 0) != 0) throw Usage{"unexpected argument " + k};
    k = k.substr(2);
    if (i + 1 >= argc || std::string(argv[i + 1]).rfind("--", 0) == 0) throw Usage{"flag --" + k + " needs a value"};
    a[k] = argv[++i];
  }
  return a;
}
std::string get(const Args& a, const std::string& k, const std::string& def) {
  auto it = a.find(k);
  return it == a.end() ? def : it->second;
}
int64_t get_i(const Args& a, const std::string& k, int64_t def) {
  const std::string v = get(a, k, "");
  if (v.empty()) return def;
  char* e = nullptr;
  const long long x = std::strtoll(v.c_str(), &e, 10);
  if (!e || *e) throw Usage{"--" + k + " expects an integer, got " + v};
  return x;
}
double get_d(const Args& a, const std::string& k, double def) {
  const std::string v = get(a, k, "");
  if (v.empty()) return def;
  char* e = nullptr;
  const double x = std::strtod(v.c_str(), &e);
  if (!e || *e) throw Usage{"--" + k + " expects a number, got " + v};
  return x;
}

void cuda_ok(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw Fatal{std::string(what) + ": " + cudaGetErrorString(e)};
}
void st_ok(mmmcu_ctx* ctx, mmmcu_status s, const char* what) {
  if (s == MMMCU_OK) return;
  const std::string msg = std::string(what) + ": " + mmmcu_last_error(ctx);
  if (s == MMMCU_ERR_INVALID_ARG || s == MMMCU_ERR_DIM_MISMATCH || s == MMMCU_ERR_UNSUPPORTED) throw Usage{msg};
  throw Fatal{msg};
}
void io_ok(mmmcu_status s) {
  if (s == MMMCU_OK) return;
  const std::string msg = mmmcu_io_last_error();
  if (s == MMMCU_ERR_UNSUPPORTED || s == MMMCU_ERR_DIM_MISMATCH) throw Usage{msg};
  throw IoFail{msg};
}

int64_t round64(int64_t x) { return (x + 63) / 64 * 64; }

// A device matrix in the reference Matrix layout (ld = round_up(cols, 64), zero padding).
struct DMat {
  float* p = nullptr;
  int64_t rows = 0, cols = 0, ld = 0;
  DMat() = default;
  DMat(int64_t r, int64_t c) : rows(r), cols(c), ld(round64(c)) {
    cuda_ok(cudaMalloc(&p, sizeof(float) * rows * ld), "cudaMalloc");
    cuda_ok(cudaMemset(p, 0, sizeof(float) * rows * ld), "cudaMemset");
  }
  DMat(const DMat&) = delete;
  DMat& operator=(const DMat&) = delete;
  DMat(DMat&& o) noexcept { *this = std::move(o); }
  DMat& operator=(DMat&& o) noexcept {
    std::swap(p, o.p);
    rows = o.rows;
    cols = o.cols;
    ld = o.ld;
    return *this;
  }
  ~DMat() {
    if (p) cudaFree(p);
  }
  std::vector<float> host() const {
    std::vector<float> h((size_t)(rows * cols));
    cuda_ok(cudaMemcpy2D(h.data(), sizeof(float) * cols, p, sizeof(float) * ld, sizeof(float) * cols, rows,
                         cudaMemcpyDeviceToHost),
            "D2H");
    return h;
  }
  void upload(const std::vector<float>& h) {
    cuda_ok(cudaMemcpy2D(p, sizeof(float) * ld, h.data(), sizeof(float) * cols, sizeof(float) * cols, rows,
                         cudaMemcpyHostToDevice),
            "H2D");
  }
};

struct Ctx {
  mmmcu_ctx* c = nullptr;
  cudaStream_t st = nullptr;
  Ctx() {
    const mmmcu_status s = mmmcu_ctx_create(0, &c);
    if (s != MMMCU_OK) throw Fatal{std::string("context: ") + mmmcu_last_error(nullptr)};
    cuda_ok(cudaStreamCreate(&st), "stream");
    st_ok(c, mmmcu_set_stream(c, st), "set_stream");
  }
  ~Ctx() {
    mmmcu_ctx_destroy(c);
    if (st) cudaStreamDestroy(st);
  }
};

DMat load(const std::string& path) {
  int32_t dt = 0;
  int64_t r = 0, c = 0;
  io_ok(mmmcu_mmmb_peek(path.c_str(), &dt, &r, &c));
  if (dt != 0) throw Usage{path + " holds f64: the GPU path is f32 only"};
  DMat m(r, c);
  io_ok(mmmcu_mmmb_load(path.c_str(), m.p, m.ld, r, nullptr, &r, &c));
  return m;
}

// Synthetic operand with the device generator (uniform values, i.i.d. element
// or aligned-block masks, per-matrix seeds).
DMat synth(Ctx& ctx, int64_t rows, int64_t cols, uint64_t seed, int value_kind, double sigma, double thresh,
           int mask_kind, double p, int64_t block) {
  DMat m(rows, cols);
  st_ok(ctx.c, mmmcu_generate(ctx.c, m.p, rows, cols, m.ld, 0, seed, value_kind, sigma, thresh, mask_kind, p, block),
        "generate");
  cuda_ok(cudaStreamSynchronize(ctx.st), "generate");
  return m;
}

void operands(Ctx& ctx, const Args& a, DMat& A, DMat& B, double& sa, double& sb, std::string& sbstruct) {
  if (a.count("a") || a.count("b")) {
    if (!a.count("a") || !a.count("b")) throw Usage{"--a and --b go together"};
    A = load(get(a, "a", ""));
    B = load(get(a, "b", ""));
    sa = sb = -1;
    sbstruct = "file";
  } else {
    const int64_t n = get_i(a, "n", 0);
    if (n <= 0) throw Usage{"give --a FILE --b FILE or --n N"};
    sa = get_d(a, "a-sparsity", 0.8);
    sb = get_d(a, "b-sparsity", 0.8);
    const int64_t bl = get_i(a, "block-len", 16);
    const uint64_t seed = (uint64_t)get_i(a, "seed", 42);
    A = synth(ctx, n, n, seed * 2 + 1, 0, 1.0, 0.0, 1, sa, 1);
    B = synth(ctx, n, n, seed * 2 + 2, 0, 1.0, 0.0, 2, sb, bl);
    sbstruct = "block_random";
  }
  if (A.cols != B.rows) throw Usage{"incompatible dims: a.cols " + std::to_string(A.cols) + " != b.rows " +
                                    std::to_string(B.rows)};
}

// Quantized checksum (SPEC bench-cli decision): each element rounded to 2^-16 relative
// precision (16 of fp32's 23 mantissa bits kept, rounded half up on the bit pattern), folded
// with FNV-1a over the logical range.
uint64_t checksum(const std::vector<float>& c) {
  uint64_t h = 1469598103934665603ull;
  for (float v : c) {
    uint32_t b;
    std::memcpy(&b, &v, 4);
    if ((b & 0x7FFFFFFFu) == 0) b = 0;  // +0 / -0 alike
    b = (b + 0x40u) & 0xFFFFFF80u;
    h = (h ^ b) * 1099511628211ull;
  }
  return h;
}

struct Rec {
  std::string algo;
  int64_t n;
  double sa, sb;
  std::string sbs;
  int workers, trial;
  double pre_ns, mul_ns;
  mmmcu_counters cnt;
  uint64_t sum;
};

void csv_header(std::FILE* f) {
  std::fprintf(f,
               "algo,n,a_sparsity,b_sparsity,structure_b,dtype,workers,trial,preprocess_ns,multiply_ns,total_ns,"
               "kernel_invocations,lane_fma_ops,rows_skipped,regions_skipped,checksum\n");
}
void csv_row(std::FILE* f, const Rec& r, const std::string& trial) {
  std::fprintf(f, "%s,%lld,%.4f,%.4f,%s,f32,%d,%s,%.0f,%.0f,%.0f,%llu,%llu,%llu,%llu,%016llx\n", r.algo.c_str(),
               (long long)r.n, r.sa, r.sb, r.sbs.c_str(), r.workers, trial.c_str(), r.pre_ns, r.mul_ns,
               r.pre_ns + r.mul_ns, (unsigned long long)r.cnt.kernel_invocations,
               (unsigned long long)r.cnt.lane_fma_ops, (unsigned long long)r.cnt.rows_skipped,
               (unsigned long long)r.cnt.regions_skipped_by_zero_code, (unsigned long long)r.sum);
}

struct Timer {
  cudaEvent_t e[3];
  Timer() {
    for (auto& x : e) cuda_ok(cudaEventCreate(&x), "event");
  }
  ~Timer() {
    for (auto& x : e) cudaEventDestroy(x);
  }
};

struct Cublas {
  cublasHandle_t h = nullptr;
  explicit Cublas(cudaStream_t st) {
    if (cublasCreate(&h) != CUBLAS_STATUS_SUCCESS) throw Fatal{"cublasCreate failed"};
    cublasSetStream(h, st);
    cublasSetMathMode(h, CUBLAS_PEDANTIC_MATH);  // plain fp32 (no tf32 tensor cores)
  }
  ~Cublas() { cublasDestroy(h); }
  // C (row-major M x N, ldc) += A (M x K, lda) * B (K x N, ldb): column-major C^T = B^T A^T
  void gemm(const DMat& A, const DMat& B, DMat& C) {
    const float one = 1.0f;
    if (cublasSgemm(h, CUBLAS_OP_N, CUBLAS_OP_N, (int)B.cols, (int)A.rows, (int)A.cols, &one, B.p, (int)B.ld, A.p,
                    (int)A.ld, &one, C.p, (int)C.ld) != CUBLAS_STATUS_SUCCESS)
      throw Fatal{"cublasSgemm failed"};
  }
};

// One multiply of `algo` into a zeroed C: preprocess / multiply times (ns) and counters.
Rec run_algo(Ctx& ctx, Cublas& blas, const std::string& algo, const DMat& A, const DMat& B, DMat& C, int workers) {
  Timer t;
  Rec r{};
  r.algo = algo;
  r.workers = workers;
  cuda_ok(cudaMemsetAsync(C.p, 0, sizeof(float) * C.rows * C.ld, ctx.st), "memset");
  const mmmcu_lane lane{8, 8, 1};
  cuda_ok(cudaEventRecord(t.e[0], ctx.st), "event");
  if (algo == "cublas") {
    cuda_ok(cudaEventRecord(t.e[1], ctx.st), "event");
    blas.gemm(A, B, C);
  } else if (algo == "dense") {
    cuda_ok(cudaEventRecord(t.e[1], ctx.st), "event");
    st_ok(ctx.c, mmmcu_multiply_simple(ctx.c, C.p, C.ld, A.p, A.ld, B.p, B.ld, A.rows, A.cols, B.cols), "multiply_simple");
  } else {
    const mmmcu_algo al = algo == "mmm" ? MMMCU_ALGO_AUTO
                          : algo == "mmm_exact" ? MMMCU_ALGO_SIMT_BCAST
                          : algo == "mmm_tc" ? MMMCU_ALGO_TC
                                             : MMMCU_ALGO_TC32;
    st_ok(ctx.c, mmmcu_set_algo(ctx.c, al), "set_algo");
    static uint64_t version = 0;
    ++version;
    st_ok(ctx.c, mmmcu_preprocess(ctx.c, A.p, A.rows, A.cols, A.ld, B.p, B.cols, B.ld, lane, version, version),
          "preprocess");
    cuda_ok(cudaEventRecord(t.e[1], ctx.st), "event");
    st_ok(ctx.c, mmmcu_multiply_parallel(ctx.c, C.p, C.ld, A.p, B.p, version, version, workers, nullptr), "multiply");
  }
  cuda_ok(cudaEventRecord(t.e[2], ctx.st), "event");
  cuda_ok(cudaEventSynchronize(t.e[2]), "sync");
  float ms0 = 0, ms1 = 0;
  cudaEventElapsedTime(&ms0, t.e[0], t.e[1]);
  cudaEventElapsedTime(&ms1, t.e[1], t.e[2]);
  r.pre_ns = ms0 * 1e6;
  r.mul_ns = ms1 * 1e6;
  if (algo.rfind("mmm", 0) == 0) st_ok(ctx.c, mmmcu_get_counters(ctx.c, &r.cnt), "counters");
  return r;
}

std::vector<std::string> algo_list(const std::string& a) {
  if (a == "all") return {"mmm", "mmm_exact", "mmm_tc", "mmm_tc32", "dense", "cublas"};
  static const char* known[] = {"mmm", "mmm_exact", "mmm_tc", "mmm_tc32", "dense", "cublas"};
  for (const char* k : known)
    if (a == k) return {a};
  throw Usage{"unknown algo " + a};
}

std::FILE* open_out(const Args& a) {
  const std::string p = get(a, "out", "");
  if (p.empty()) return stdout;
  std::FILE* f = std::fopen(p.c_str(), "w");
  if (!f) throw IoFail{"cannot open " + p};
  return f;
}

int cmd_gen(const Args& a) {
  const int64_t rows = get_i(a, "rows", 0), cols = get_i(a, "cols", 0);
  if (rows <= 0 || cols <= 0) throw Usage{"--rows and --cols must be positive"};
  const std::string out = get(a, "out", "");
  if (out.empty()) throw Usage{"--out FILE is required"};
  const std::string structure = get(a, "structure", "random"), value = get(a, "value", "uniform");
  const double sp = get_d(a, "sparsity", 0.0);
  if (!(sp >= 0.0 && sp <= 1.0)) throw Usage{"--sparsity must lie in [0, 1]"};
  int mask = 0;
  if (structure == "random") mask = sp > 0 ? 1 : 0;
  else if (structure == "block_random") mask = 2;
  else throw Usage{"structure " + structure + ": the device generator draws random / block_random (i.i.d. masks)"};
  const int vk = value == "uniform" ? 0 : value == "normal" ? 1 : value == "relu" ? 2 : -1;
  if (vk < 0) throw Usage{"unknown --value " + value};
  Ctx ctx;
  DMat m = synth(ctx, rows, cols, (uint64_t)get_i(a, "seed", 42), vk, get_d(a, "sigma", 1.0), get_d(a, "thresh", 0.0),
                 mask, sp, get_i(a, "block-len", 16));
  io_ok(mmmcu_mmmb_save(out.c_str(), m.p, rows, cols, m.ld, nullptr));
  const std::vector<float> h = m.host();
  const int64_t z = std::count(h.begin(), h.end(), 0.0f);
  std::printf("wrote %s: %lld x %lld, measured sparsity %.5f\n", out.c_str(), (long long)rows, (long long)cols,
              (double)z / (double)h.size());
  return kExitOk;
}

int cmd_bench(const Args& a) {
  Ctx ctx;
  DMat A, B;
  double sa, sb;
  std::string sbs;
  operands(ctx, a, A, B, sa, sb, sbs);
  const auto algos = algo_list(get(a, "algo", "mmm"));
  // worker count: the flag, else MMM_WORKERS, else 1 (SPEC bench-cli design decisions); the
  // GPU path validates it (multiply_parallel) and records it
  const char* env_w = std::getenv("MMM_WORKERS");
  const int trials = (int)get_i(a, "trials", 10),
            workers = (int)get_i(a, "workers", env_w ? std::strtoll(env_w, nullptr, 10) : 1);
  if (trials <= 0) throw Usage{"--trials must be positive"};
  DMat C(A.rows, B.cols);
  Cublas blas(ctx.st);
  std::FILE* f = open_out(a);
  csv_header(f);
  for (const auto& al : algos) {
    run_algo(ctx, blas, al, A, B, C, workers);  // warm-up (plans, caches, lazy loads)
    std::vector<Rec> recs;
    for (int t = 0; t < trials; ++t) {
      Rec r = run_algo(ctx, blas, al, A, B, C, workers);
      r.n = A.rows;
      r.sa = sa;
      r.sb = sb;
      r.sbs = sbs;
      r.trial = t;
      r.sum = checksum(C.host());
      csv_row(f, r, std::to_string(t));
      recs.push_back(r);
    }
    std::vector<Rec> sorted(recs);
    std::sort(sorted.begin(), sorted.end(), [](const Rec& x, const Rec& y) { return x.mul_ns < y.mul_ns; });
    Rec med = sorted[sorted.size() / 2];
    csv_row(f, med, "median");
  }
  if (f != stdout) std::fclose(f);
  return kExitOk;
}

int cmd_sweep(const Args& a) {
  const int64_t n = get_i(a, "n", 2048);
  const double step = get_d(a, "grid-step", 0.1);
  const int64_t bl = get_i(a, "block-len", 16);
  const int trials = (int)get_i(a, "trials", 3);
  if (n <= 0 || !(step > 0 && step <= 1) || trials <= 0) throw Usage{"bad sweep arguments"};
  Ctx ctx;
  Cublas blas(ctx.st);
  DMat C(n, n);
  std::FILE* f = open_out(a);
  std::fprintf(f,
               "a_sparsity,b_sparsity,mmm_multiply_ns,mmm_total_ns,mmm_path,best_dense_ns,best_dense_algo,speedup_multiply,"
               "speedup_total,lane_fma_ops_per_n3\n");
  auto median = [&](const std::string& al, const DMat& A, const DMat& B, double* pre) {
    std::vector<double> m, p;
    run_algo(ctx, blas, al, A, B, C, 1);
    for (int t = 0; t < trials; ++t) {
      const Rec r = run_algo(ctx, blas, al, A, B, C, 1);
      m.push_back(r.mul_ns);
      p.push_back(r.pre_ns);
    }
    std::sort(m.begin(), m.end());
    std::sort(p.begin(), p.end());
    if (pre) *pre = p[p.size() / 2];
    return m[m.size() / 2];
  };
  const int steps = (int)std::floor(1.0 / step + 1e-9);
  for (int i = 0; i <= steps; ++i)
    for (int j = 0; j <= steps; ++j) {
      const double sa = std::min(1.0, i * step), sb = std::min(1.0, j * step);
      DMat A = synth(ctx, n, n, 1000 + i, 0, 1.0, 0.0, 1, sa, 1);
      DMat B = synth(ctx, n, n, 2000 + j, 0, 1.0, 0.0, 2, sb, bl);
      double pre = 0;
      const double mm = median("mmm", A, B, &pre);
      mmmcu_algo path;
      mmmcu_last_algo(ctx.c, &path);
      mmmcu_counters cnt;
      st_ok(ctx.c, mmmcu_get_counters(ctx.c, &cnt), "counters");
      const double cb = median("cublas", A, B, nullptr), de = median("dense", A, B, nullptr);
      const double best = std::min(cb, de);
      std::fprintf(f, "%.3f,%.3f,%.0f,%.0f,%s,%.0f,%s,%.4f,%.4f,%.6f\n", sa, sb, mm, mm + pre,
                   path == MMMCU_ALGO_TC ? "k2_tc" : "k2_simt", best, cb <= de ? "cublas" : "dense", best / mm,
                   best / (mm + pre), (double)cnt.lane_fma_ops / ((double)n * n * n));
      std::fflush(f);
    }
  if (f != stdout) std::fclose(f);
  return kExitOk;
}

int cmd_verify(const Args& a) {
  const double tol = get_d(a, "tolerance", 1e-5);
  Ctx ctx;
  DMat A, B;
  double sa, sb;
  std::string sbs;
  operands(ctx, a, A, B, sa, sb, sbs);
  Cublas blas(ctx.st);
  DMat C(A.rows, B.cols), R(A.rows, B.cols), D(A.rows, B.cols);
  // reference: multiply_simple (dense i-k-j fmaf); denominator Σ|a||b| from |A| |B|
  run_algo(ctx, blas, "dense", A, B, R, 1);
  const std::vector<float> ref = R.host();
  {
    std::vector<float> ha = A.host(), hb = B.host();
    for (float& v : ha) v = std::fabs(v);
    for (float& v : hb) v = std::fabs(v);
    DMat Aa(A.rows, A.cols), Ba(B.rows, B.cols);
    Aa.upload(ha);
    Ba.upload(hb);
    run_algo(ctx, blas, "dense", Aa, Ba, D, 1);
  }
  const std::vector<float> den = D.host();
  bool ok = true;
  for (const auto& al : algo_list("all")) {
    if (al == "dense") continue;
    run_algo(ctx, blas, al, A, B, C, 1);
    const std::vector<float> c = C.host();
    double worst = 0;
    int64_t bad = 0;
    for (size_t i = 0; i < c.size(); ++i) {
      const double e = std::fabs((double)c[i] - (double)ref[i]);
      const double d = (double)den[i] * (1.0 + 1e-6);  // the denominator's own fp32 rounding
      if (e > tol * d) ++bad;
      if (d > 0) worst = std::max(worst, e / d);
      else if (e > 0) worst = INFINITY;
    }
    const bool pass = bad == 0;
    ok = ok && pass;
    std::printf("%-10s max rel error %.3e  %s\n", al.c_str(), worst, pass ? "ok" : "FAIL");
  }
  return ok ? kExitOk : kExitVerify;
}

int cmd_analyze(const Args& a) {
  const std::string path = get(a, "matrix", "");
  if (path.empty()) throw Usage{"--matrix FILE is required"};
  Ctx ctx;
  DMat m = load(path);
  const std::vector<float> h = m.host();
  int64_t zeros = std::count(h.begin(), h.end(), 0.0f);
  // zero-region fractions at widths 8 / 16 / 32 / 64 from the pattern codes (K1, preprocess_b)
  const mmmcu_lane lane{8, 8, 1};
  st_ok(ctx.c, mmmcu_preprocess_b(ctx.c, m.p, m.rows, m.cols, m.ld, lane, 1), "preprocess_b");
  const int64_t nreg = m.ld / 64;
  std::vector<uint8_t> codes((size_t)(m.rows * nreg));
  st_ok(ctx.c, mmmcu_export_b_codes(ctx.c, codes.data(), (int64_t)codes.size()), "codes");
  const int64_t ngroups_row = (m.cols + 7) / 8;
  double zf[4] = {0, 0, 0, 0};  // widths 8, 16, 32, 64
  int64_t units[4] = {0, 0, 0, 0};
  for (int64_t k = 0; k < m.rows; ++k)
    for (int64_t r = 0; r < nreg; ++r) {
      const uint8_t c = codes[(size_t)(k * nreg + r)];
      for (int wi = 0; wi < 4; ++wi) {
        const int span = 1 << wi;  // groups per unit
        for (int g0 = 0; g0 < 8; g0 += span) {
          if (r * 8 + g0 >= ngroups_row) break;
          const int mask = ((1 << span) - 1) << (8 - g0 - span);
          zf[wi] += (c & mask) == 0;
          ++units[wi];
        }
      }
    }
  int64_t zero_cols = 0;
  for (int64_t j = 0; j < m.cols; ++j) {
    bool z = true;
    for (int64_t i = 0; i < m.rows && z; ++i) z = h[(size_t)(i * m.cols + j)] == 0.0f;
    zero_cols += z;
  }
  const double el = (double)zeros / (double)h.size();
  std::printf("matrix %s: %lld x %lld f32\n", path.c_str(), (long long)m.rows, (long long)m.cols);
  std::printf("elementwise sparsity      %.5f\n", el);
  const char* w[4] = {"8 (W)", "16", "32", "64 (R)"};
  for (int i = 0; i < 4; ++i) std::printf("zero-region fraction %-6s %.5f\n", w[i], units[i] ? zf[i] / units[i] : 0.0);
  std::printf("column sparsity           %.5f\n", (double)zero_cols / (double)m.cols);
  // measured regime map: the masked multiply pays over cuBLAS SGEMM once the product
  // of the A and B densities is low; as a B operand, region sparsity decides the masked path
  std::printf("predicted best algorithm  %s\n", (el >= 0.5 || zf[0] >= 0.5) ? "mmm" : "dense");
  return kExitOk;
}

void usage() {
  std::fprintf(stderr,
               "usage: mmm-cuda {gen|bench|sweep|verify|analyze} [--flag value ...]\n"
               "  gen     --rows R --cols C [--structure random|block_random] [--sparsity s] [--block-len L]\n"
               "          [--value uniform|normal|relu] [--sigma x] [--thresh t] [--seed S] --out FILE\n"
               "  bench   (--a FILE --b FILE | --n N [--a-sparsity s] [--b-sparsity s] [--block-len L] [--seed S])\n"
               "          [--algo mmm|mmm_exact|mmm_tc|mmm_tc32|dense|cublas|all] [--trials T] [--workers W] [--out CSV]\n"
               "  sweep   --n N [--grid-step g] [--block-len L] [--trials T] [--out CSV]\n"
               "  verify  (--a FILE --b FILE | --n N ...) [--tolerance 1e-5]\n"
               "  analyze --matrix FILE\n"
               "exit codes: 0 ok, 1 verification failure, 2 usage error, 3 I/O error\n");
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2 || !std::strcmp(argv[1], "--help") || !std::strcmp(argv[1], "-h")) {
    usage();
    return argc < 2 ? kExitUsage : kExitOk;
  }
  const std::string cmd = argv[1];
  try {
    const Args a = parse(argc, argv, 2);
    if (cmd == "gen") return cmd_gen(a);
    if (cmd == "bench") return cmd_bench(a);
    if (cmd == "sweep") return cmd_sweep(a);
    if (cmd == "verify") return cmd_verify(a);
    if (cmd == "analyze") return cmd_analyze(a);
    usage();
    return kExitUsage;
  } catch (const Usage& e) {
    std::fprintf(stderr, "mmm-cuda: %s\n", e.msg.c_str());
    return kExitUsage;
  } catch (const IoFail& e) {
    std::fprintf(stderr, "mmm-cuda: %s\n", e.msg.c_str());
    return kExitIo;
  } catch (const Fatal& e) {
    std::fprintf(stderr, "mmm-cuda: %s\n", e.msg.c_str());
    return kExitIo;
  }
}
