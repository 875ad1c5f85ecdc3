// Drop-in check: a reference-style caller (SPEC engine API over the reference's own
// Matrix<float> / generate<float>, /root/reference/proj/include) switched to
// include/mmm_cuda.hpp.  Built by paper_2402_14118_b200/build.py when the reference headers
// are present; run on the GPU by tests/test_gpu_parity.py::test_cpp_dropin.
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "mmm/matgen.hpp"
#include "mmm_cuda.hpp"

using namespace mmm;

#define CHECK(cond)                                                          \
  do {                                                                       \
    if (!(cond)) {                                                           \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);            \
      std::exit(1);                                                          \
    }                                                                        \
  } while (0)

int main() {
  const int64_t M = 300, K = 520, N = 320;
  SparsitySpec sa{Structure::random, 0.8, 0, 11};
  SparsitySpec sb{Structure::block_random, 0.8, 16, 12};
  Matrix<float> a = generate<float>(M, K, sa);
  Matrix<float> b = generate<float>(K, N, sb);

  // oracle: ascending-k fmaf chain over the non-zero A entries and non-zero 8-wide B groups
  Matrix<float> ref(M, N);
  uint64_t lanes = 0;
  for (int64_t i = 0; i < M; ++i)
    for (int64_t k = 0; k < K; ++k) {
      const float av = a.at(i, k);
      if (av == 0.0f) continue;
      for (int64_t g = 0; g < b.padded_cols(); g += 8) {
        bool nz = false;
        for (int l = 0; l < 8; ++l) nz |= b.row(k)[g + l] != 0.0f;
        if (!nz) continue;
        lanes += 8;
        for (int l = 0; l < 8 && g + l < N; ++l) ref.row(i)[g + l] = std::fma(av, b.row(k)[g + l], ref.row(i)[g + l]);
      }
    }

  MmmContext<float> ctx(a, b, LaneConfig::defaults(Dtype::f32), 256, 0, Accumulation::Exact);
  Matrix<float> c(M, N);
  WorkCounters w = multiply_mmm(ctx, c, a, b);
  CHECK(w.lane_fma_ops == lanes);
  CHECK(w.rows_skipped + (uint64_t)((1.0 - elementwise_sparsity(a)) * M * K + 0.5) == (uint64_t)(M * K));
  for (int64_t i = 0; i < M; ++i)
    for (int64_t j = 0; j < N; ++j) CHECK(c.at(i, j) == ref.at(i, j));  // bit-exact (K2-SIMT)
  CHECK(c.padding_is_zero());

  // default accumulation (AUTO: K2-SIMT or K2-TC): within the north_star tolerance
  {
    const Matrix<float>& ca_ = a;  // const access: no version bump
    const Matrix<float>& cb_ = b;
    MmmContext<float> actx(a, b);
    Matrix<float> ca(M, N);
    WorkCounters wa = multiply_mmm(actx, ca, a, b);
    CHECK(wa.lane_fma_ops == lanes);
    for (int64_t i = 0; i < M; ++i)
      for (int64_t j = 0; j < N; ++j) {
        double den = 0.0;
        for (int64_t k = 0; k < K; ++k) den += std::fabs((double)ca_.at(i, k) * (double)cb_.at(k, j));
        CHECK(std::fabs((double)ca.at(i, j) - (double)ref.at(i, j)) <= 1e-5 * den);
      }
    CHECK(ca.padding_is_zero());
  }

  // multiply_parallel: same bits, worker_count 0 rejected
  Matrix<float> c2(M, N);
  WorkCounters w2 = multiply_parallel(ctx, c2, a, b, 8);
  CHECK(w2.lane_fma_ops == w.lane_fma_ops);
  bool threw = false;
  try {
    multiply_parallel(ctx, c2, a, b, 0);
  } catch (const std::invalid_argument&) {
    threw = true;
  }
  CHECK(threw);

  // stale context: any mutable access bumps Matrix::version
  a.at(0, 0) = 1.0f;
  threw = false;
  try {
    multiply_mmm(ctx, c, a, b);
  } catch (const StaleContextError&) {
    threw = true;
  }
  CHECK(threw);

  // bad lane config: the reference's KernelTable::build message (kernel_table.cpp:66-67)
  threw = false;
  try {
    MmmContext<float> bad(a, b, LaneConfig{8, 17, 1});
  } catch (const std::invalid_argument& e) {
    threw = std::string(e.what()).find("pattern size must lie in [1, 16]") != std::string::npos;
  }
  CHECK(threw);

  // preprocess_b / plan_stats / preprocess_a
  std::vector<BPlan> plans = preprocess_b(b, LaneConfig::defaults(Dtype::f32), 256);
  CHECK(plans.size() == 6);  // ceil(520/256) = 3 leaf rows x ceil(5 regions / 4) = 2 leaf cols
  PlanStats st = plan_stats(plans);
  CHECK(st.region_count == K * (b.padded_cols() / 64));
  ABlockIndex idx = preprocess_a(a, 256);
  int64_t nnz = 0;
  for (uint8_t cnt : idx.counts) nnz += cnt;
  int64_t direct = 0;
  for (int64_t i = 0; i < M; ++i)
    for (int64_t k = 0; k < K; ++k) direct += a.at(i, k) != 0.0f;
  CHECK(nnz == direct);

  // multiply_simple: dense fmaf chain == masked chain on finite data
  Matrix<float> c3(M, N);
  Matrix<float> a2 = generate<float>(M, K, sa);
  multiply_simple(c3, a2, b);
  for (int64_t i = 0; i < M; ++i)
    for (int64_t j = 0; j < N; ++j) CHECK(c3.at(i, j) == ref.at(i, j));

  // f64 (Dtype::f64, default lane {4, 8, 1}) and an f32 non-default lane ({2, 16, 2}: G = 4,
  // P = 16, two-part KernelTable): the reference's per-group fma chain, bit-identical
  {
    auto masked_ref = [](const auto& A, const auto& B, auto& C, int64_t G, uint64_t& lane_ops) {
      for (int64_t i = 0; i < A.rows(); ++i)
        for (int64_t k = 0; k < A.cols(); ++k) {
          const auto av = A.at(i, k);
          if (av == 0) continue;
          for (int64_t g = 0; g < B.padded_cols(); g += G) {
            bool nz = false;
            for (int64_t l = 0; l < G; ++l) nz |= B.row(k)[g + l] != 0;
            if (!nz) continue;
            lane_ops += G;
            for (int64_t l = 0; l < G && g + l < B.cols(); ++l)
              C.row(i)[g + l] = std::fma(av, B.row(k)[g + l], C.row(i)[g + l]);
          }
        }
    };
    const LaneConfig l64 = LaneConfig::defaults(Dtype::f64);
    Matrix<double> a64 = generate<double>(130, 200, SparsitySpec{Structure::random, 0.7, 0, 21}, l64);
    Matrix<double> b64 = generate<double>(200, 150, SparsitySpec{Structure::block_random, 0.6, 0, 22}, l64);
    Matrix<double> r64(130, 150, l64);
    uint64_t ops64 = 0;
    masked_ref(a64, b64, r64, 4, ops64);
    MmmContext<double> c64ctx(a64, b64, l64);
    Matrix<double> c64(130, 150, l64);
    WorkCounters w64 = multiply_mmm(c64ctx, c64, a64, b64);
    CHECK(w64.lane_fma_ops == ops64);
    for (int64_t i = 0; i < 130; ++i)
      for (int64_t j = 0; j < 150; ++j) CHECK(c64.at(i, j) == r64.at(i, j));
    CHECK(c64.padding_is_zero());
    std::vector<BPlan> p64 = preprocess_b(b64, l64, 256);
    CHECK(plan_stats(p64).region_count == 200 * (b64.padded_cols() / 32));
    Matrix<double> s64(130, 150, l64), sr(130, 150, l64);
    multiply_simple(s64, a64, b64);
    for (int64_t i = 0; i < 130; ++i)
      for (int64_t k = 0; k < 200; ++k)
        for (int64_t j = 0; j < 150; ++j) sr.row(i)[j] = std::fma(a64.at(i, k), b64.at(k, j), sr.row(i)[j]);
    for (int64_t i = 0; i < 130; ++i)
      for (int64_t j = 0; j < 150; ++j) CHECK(s64.at(i, j) == sr.at(i, j));

    const LaneConfig l16{2, 16, 2};
    Matrix<float> a16 = generate<float>(90, 120, SparsitySpec{Structure::random, 0.6, 0, 31}, l16);
    Matrix<float> b16 = generate<float>(120, 200, SparsitySpec{Structure::block_random, 0.5, 0, 32}, l16);
    Matrix<float> r16(90, 200, l16);
    uint64_t ops16 = 0;
    masked_ref(a16, b16, r16, 4, ops16);
    MmmContext<float> c16ctx(a16, b16, l16);
    Matrix<float> c16(90, 200, l16);
    WorkCounters w16 = multiply_mmm(c16ctx, c16, a16, b16);
    CHECK(w16.lane_fma_ops == ops16);
    for (int64_t i = 0; i < 90; ++i)
      for (int64_t j = 0; j < 200; ++j) CHECK(c16.at(i, j) == r16.at(i, j));
    std::vector<BPlan> p16 = preprocess_b(b16, l16, 256);
    bool wide_code = false;
    for (const BPlan& p : p16)
      for (uint16_t code : p.codes) wide_code |= code > 0xFF;  // P = 16 codes exceed a byte
    CHECK(wide_code);
  }

  std::printf("DROPIN OK lane_fma_ops=%llu\n", (unsigned long long)w.lane_fma_ops);
  return 0;
}
