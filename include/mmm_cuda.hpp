// mmm_cuda.hpp — C++ drop-in for the reference's masked-multiply engine, on the B200 C ABI.
//
// A caller of the reference (namespace mmm) keeps its types and call sites:
// Matrix<T> (T = float or double) and LaneConfig come from the reference's own mmm/matrix.hpp
// (/root/reference/proj/include/mmm/matrix.hpp:31-164, on the include path of the
// integrating build), and the SPEC entry points below forward to include/mmmcu.h.
// Header-only; link libmmmcu.so.  Exceptions mirror the reference's error behaviour:
//   std::invalid_argument  bad lane config (kernel_table.cpp:66-72), bad dims, worker_count 0
//   DimensionMismatch      a.cols != b.rows or c's shape
//   StaleContextError      operands changed since the context's plans
//   UnsupportedError       lane config / dtype without a GPU kernel (no CPU fallback)
//   CudaError              device failures (including "no CUDA device")
#ifndef MMM_CUDA_HPP_
#define MMM_CUDA_HPP_

#include <cstdint>
#include <stdexcept>
#include <algorithm>
#include <string>
#include <type_traits>
#include <utility>
#include <vector>

#include "mmm/matrix.hpp"  // the reference's Matrix<T>, LaneConfig
#include "mmmcu.h"

namespace mmm {

struct DimensionMismatch : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};
struct StaleContextError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct UnsupportedError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// WorkCounters.
struct WorkCounters {
  uint64_t kernel_invocations = 0;
  uint64_t lane_fma_ops = 0;
  uint64_t rows_skipped = 0;
  uint64_t regions_skipped_by_zero_code = 0;
};

// BPlan and ABlockIndex (layout decision :229).
struct BPlan {
  int64_t submatrix_id = 0;
  std::vector<uint16_t> codes;  // one P-bit code (P <= 16) per region, multiply order
};
struct ABlockIndex {
  int64_t block_dim = 256;
  std::vector<uint8_t> counts;   // per 8-element segment, block-major
  std::vector<uint8_t> offsets;  // 8 slots per segment, 0xFF unused (full segments store none)
};
struct PlanStats {
  int64_t region_count = 0;
  double zero_region_fraction = 0.0;
  double mean_popcount = 0.0;
};

namespace cuda_detail {

inline void check(mmmcu_status st, const mmmcu_ctx* ctx) {
  if (st == MMMCU_OK) return;
  const std::string msg = mmmcu_last_error(ctx);
  switch (st) {
    case MMMCU_ERR_INVALID_ARG:
    case MMMCU_ERR_WORKERS: throw std::invalid_argument(msg);
    case MMMCU_ERR_DIM_MISMATCH: throw DimensionMismatch(msg);
    case MMMCU_ERR_STALE: throw StaleContextError(msg);
    case MMMCU_ERR_UNSUPPORTED: throw UnsupportedError(msg);
    case MMMCU_ERR_OVERFLOW: throw std::overflow_error(msg);
    default: throw CudaError(msg);
  }
}

inline mmmcu_lane lane_of(const LaneConfig& l) { return mmmcu_lane{l.w, l.p, l.v}; }

inline WorkCounters counters_of(const mmmcu_counters& c) {
  return WorkCounters{c.kernel_invocations, c.lane_fma_ops, c.rows_skipped, c.regions_skipped_by_zero_code};
}

class Handle {
 public:
  explicit Handle(int device) { check(mmmcu_ctx_create(device, &h_), nullptr); }
  ~Handle() { mmmcu_ctx_destroy(h_); }
  Handle(const Handle&) = delete;
  Handle& operator=(const Handle&) = delete;
  Handle(Handle&& o) noexcept : h_(std::exchange(o.h_, nullptr)) {}
  mmmcu_ctx* get() const { return h_; }

 private:
  mmmcu_ctx* h_ = nullptr;
};

}  // namespace cuda_detail

// MmmContext: the device plans (B codes + block masks, A bitmaps/index
// lists, MMA-ready operands) of one (a, b) pair, tagged with their content versions.
template <typename T>
class MmmContext;

enum class Accumulation { Auto, Exact };

namespace cuda_detail {
template <typename T>
constexpr mmmcu_dtype dtype_code() {
  static_assert(std::is_same_v<T, float> || std::is_same_v<T, double>, "the reference compiles f32 and f64 only");
  return std::is_same_v<T, double> ? MMMCU_F64 : MMMCU_F32;
}
}  // namespace cuda_detail

// MmmContext<T> for the reference's two dtypes and any valid LaneConfig:
// f32 with the default lane runs the fused K1 / K2 kernels (Accumulation::Auto picks K2-TC
// or the exact K2-SIMT on the device; Exact forces the bit-identical chain); every other
// (dtype, lane) runs the lane-general kernels, always bit-identical to KernelTable<T>.
template <typename T>
class MmmContext {
 public:
  MmmContext(const Matrix<T>& a, const Matrix<T>& b, LaneConfig lane = LaneConfig::defaults(dtype_of<T>()),
             int64_t leaf_dim = 256, int device = 0, Accumulation accumulation = Accumulation::Auto)
      : h_(device), lane_(lane), leaf_dim_(leaf_dim), rows_(a.rows()), inner_(a.cols()), cols_(b.cols()) {
    if (a.cols() != b.rows())
      throw DimensionMismatch("a.cols (" + std::to_string(a.cols()) + ") != b.rows (" + std::to_string(b.rows()) +
                              ")");
    constexpr mmmcu_dtype dt = cuda_detail::dtype_code<T>();
    cuda_detail::check(mmmcu_validate_lane_t(h_.get(), dt, cuda_detail::lane_of(lane)), h_.get());
    cuda_detail::check(
        mmmcu_set_algo(h_.get(), accumulation == Accumulation::Exact ? MMMCU_ALGO_SIMT_BCAST : MMMCU_ALGO_AUTO),
        h_.get());
    cuda_detail::check(mmmcu_preprocess_host_t(h_.get(), dt, a.data(), a.rows(), a.cols(), a.padded_cols(), b.data(),
                                               b.cols(), b.padded_cols(), cuda_detail::lane_of(lane), a.version(),
                                               b.version()),
                       h_.get());
    av_ = a.version();
    bv_ = b.version();
  }

  const LaneConfig& lane() const { return lane_; }
  int64_t leaf_dim() const { return leaf_dim_; }
  // counters of the last multiply
  const WorkCounters& counters() const { return counters_; }
  mmmcu_ctx* native() const { return h_.get(); }

  WorkCounters multiply(Matrix<T>& c, const Matrix<T>& a, const Matrix<T>& b, int workers) {
    if (a.rows() != rows_ || a.cols() != inner_ || b.cols() != cols_ || c.rows() != rows_ || c.cols() != cols_)
      throw DimensionMismatch("operand shapes differ from the context's plans");
    if (a.version() != av_ || b.version() != bv_)
      throw StaleContextError("stale context: operands changed since preprocessing (Matrix::version)");
    mmmcu_counters cnt{};
    // c.data() (mutable) bumps c's version: c is written, as in the reference engine
    cuda_detail::check(mmmcu_multiply_planned_host_t(h_.get(), cuda_detail::dtype_code<T>(), c.data(),
                                                     c.padded_cols(), a.version(), b.version(), workers, &cnt),
                       h_.get());
    counters_ = cuda_detail::counters_of(cnt);
    return counters_;
  }

 private:
  cuda_detail::Handle h_;
  LaneConfig lane_;
  int64_t leaf_dim_;
  int64_t rows_, inner_, cols_;
  uint64_t av_ = 0, bv_ = 0;
  WorkCounters counters_;
};

// preprocess_b: one BPlan per leaf_dim x leaf_dim sub-block of B.
template <typename T>
std::vector<BPlan> preprocess_b(const Matrix<T>& b, const LaneConfig& lane, int64_t leaf_dim = 256, int device = 0) {
  cuda_detail::Handle h(device);
  constexpr mmmcu_dtype dt = cuda_detail::dtype_code<T>();
  cuda_detail::check(mmmcu_validate_lane_t(h.get(), dt, cuda_detail::lane_of(lane)), h.get());
  // device copy of B through the host-plan path (a 1 x b.rows() zero A keeps shapes valid)
  Matrix<T> a0(1, b.rows(), lane);
  cuda_detail::check(mmmcu_preprocess_host_t(h.get(), dt, a0.data(), 1, b.rows(), a0.padded_cols(), b.data(),
                                             b.cols(), b.padded_cols(), cuda_detail::lane_of(lane), 0, b.version()),
                     h.get());
  const int64_t nreg = b.padded_cols() / lane.region_width();
  const int64_t rpl = std::max<int64_t>(leaf_dim / lane.region_width(), 1);
  const int64_t n_pl = ((b.rows() + leaf_dim - 1) / leaf_dim) * ((nreg + rpl - 1) / rpl);
  std::vector<uint16_t> flat(static_cast<size_t>(b.rows() * nreg));
  std::vector<int64_t> off(static_cast<size_t>(n_pl + 1));
  int64_t n = 0;
  cuda_detail::check(mmmcu_export_bplans16(h.get(), leaf_dim, flat.data(), static_cast<int64_t>(flat.size()),
                                           off.data(), static_cast<int64_t>(off.size()), &n),
                     h.get());
  std::vector<BPlan> plans(static_cast<size_t>(n));
  for (int64_t p = 0; p < n; ++p) {
    plans[p].submatrix_id = p;
    plans[p].codes.assign(flat.begin() + off[p], flat.begin() + off[p + 1]);
  }
  return plans;
}

// preprocess_a.
template <typename T>
ABlockIndex preprocess_a(const Matrix<T>& a, int64_t block_dim = 256, int device = 0) {
  cuda_detail::Handle h(device);
  const LaneConfig lane = LaneConfig::defaults(dtype_of<T>());
  Matrix<T> b0(a.cols(), 1, lane);
  cuda_detail::check(mmmcu_preprocess_host_t(h.get(), cuda_detail::dtype_code<T>(), a.data(), a.rows(), a.cols(),
                                             a.padded_cols(), b0.data(), 1, b0.padded_cols(),
                                             cuda_detail::lane_of(lane), a.version(), 0),
                     h.get());
  ABlockIndex idx;
  idx.block_dim = block_dim;
  const int64_t nseg = a.rows() * ((a.cols() + 7) / 8);
  idx.counts.resize(static_cast<size_t>(nseg));
  idx.offsets.resize(static_cast<size_t>(nseg * 8));
  int64_t n = 0;
  cuda_detail::check(mmmcu_export_ablock_index(h.get(), block_dim, idx.counts.data(), nseg, idx.offsets.data(),
                                               nseg * 8, &n),
                     h.get());
  return idx;
}

// plan_stats: a pure summary of the plans' codes.
inline PlanStats plan_stats(const std::vector<BPlan>& plans) {
  PlanStats s;
  int64_t zeros = 0, pop = 0;
  for (const BPlan& p : plans)
    for (uint16_t c : p.codes) {
      ++s.region_count;
      zeros += c == 0;
      pop += __builtin_popcount(c);
    }
  if (s.region_count) {
    s.zero_region_fraction = static_cast<double>(zeros) / static_cast<double>(s.region_count);
    s.mean_popcount = static_cast<double>(pop) / static_cast<double>(s.region_count);
  }
  return s;
}

// multiply_mmm / multiply_parallel.
template <typename T>
WorkCounters multiply_mmm(MmmContext<T>& ctx, Matrix<T>& c, const Matrix<T>& a, const Matrix<T>& b) {
  return ctx.multiply(c, a, b, 1);
}
template <typename T>
WorkCounters multiply_parallel(MmmContext<T>& ctx, Matrix<T>& c, const Matrix<T>& a, const Matrix<T>& b,
                               int worker_count) {
  if (worker_count <= 0) throw std::invalid_argument("worker_count must be positive");
  return ctx.multiply(c, a, b, worker_count);
}

// multiply_simple: dense i-k-j c += a*b with fma per term, on the GPU.
template <typename T>
void multiply_simple(Matrix<T>& c, const Matrix<T>& a, const Matrix<T>& b, int device = 0) {
  if (a.cols() != b.rows() || c.rows() != a.rows() || c.cols() != b.cols())
    throw DimensionMismatch("multiply_simple: shapes do not chain");
  cuda_detail::Handle h(device);
  cuda_detail::check(mmmcu_multiply_simple_host_t(h.get(), cuda_detail::dtype_code<T>(), c.data(), c.padded_cols(),
                                                  a.data(), a.padded_cols(), b.data(), b.padded_cols(), a.rows(),
                                                  a.cols(), b.cols()),
                     h.get());
}

}  // namespace mmm

#endif  // MMM_CUDA_HPP_
