// The reference's own unit tests (test_fast.cpp, test_core.cpp,
// test_baseline.cpp, test_partition.cpp, acceptance.cpp) restated against the
// source-compatible C++ headers in include/cvgram/, which run on the B200.
// Catch2 is absent, so a tiny harness stands in.  The oracle's baseline engine
// (oracle/, test infrastructure) is the checker for the seeded equivalences.
//
//   test_header_api            all cases (needs an sm_100 device)
//   test_header_api --host     host-only cases (partition predicates, types)
#include <cstdio>
#include <cstring>
#include <functional>
#include <random>
#include <string>
#include <vector>

#include "cvgram/cvgram.hpp"

extern "C" int orc_baseline_all_folds(const double* x, const double* y, int64_t n, int64_t k, int64_t m,
                                      const int32_t* labels, int64_t n_labels, int32_t p, uint32_t cfg, int n_threads,
                                      double* xtx, double* xty, double* mean_x, double* mean_y, double* std_x,
                                      double* std_y, int64_t* n_train, int64_t* n_val, char* err, size_t errlen);

using namespace cvgram;

static int g_fail = 0, g_checks = 0;
#define CHECK(cond)                                                        \
  do {                                                                     \
    ++g_checks;                                                            \
    if (!(cond)) {                                                         \
      ++g_fail;                                                            \
      std::printf("  CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #cond); \
    }                                                                      \
  } while (0)
#define CHECK_THROWS_AS(expr, type) \
  do {                              \
    bool thrown_ = false;           \
    try {                           \
      (void)(expr);                 \
    } catch (const type&) {         \
      thrown_ = true;               \
    } catch (...) {                 \
    }                               \
    CHECK(thrown_);                 \
  } while (0)
static bool near(double a, double b, double margin) { return std::abs(a - b) <= margin; }

namespace {

DatasetPair micro_case() {
  Matrix x(3, 1), y(3, 1);
  x << 1, 3, 5;
  y << 2, 4, 6;
  return DatasetPair(x, y);
}
const PreprocessConfig kAllOn{true, true, true, true};
PreprocessConfig from_bits(int b) { return PreprocessConfig{(b & 8) != 0, (b & 4) != 0, (b & 2) != 0, (b & 1) != 0}; }

struct Base {
  std::vector<Matrix> xtx, xty;
  std::vector<Vector> mx, my, sx, sy;
};
Base oracle_baseline(const DatasetPair& d, const Partitioning& part, const PreprocessConfig& cfg) {
  const Index n = d.n_rows(), k = d.n_features(), m = d.n_responses();
  const int p = part.p;
  std::vector<double> xtx(p * k * k), xty(p * k * m), mx(p * k), my(p * m), sx(p * k), sy(p * m);
  std::vector<int64_t> nt(p), nv(p);
  std::vector<int32_t> l(part.labels.begin(), part.labels.end());
  char err[256];
  if (orc_baseline_all_folds(d.x().data(), d.y().data(), n, k, m, l.data(), n, p, cfg.mask(), 1, xtx.data(),
                             xty.data(), mx.data(), my.data(), sx.data(), sy.data(), nt.data(), nv.data(), err,
                             sizeof err))
    throw std::runtime_error(err);
  Base b;
  for (int f = 0; f < p; ++f) {
    Matrix a(k, k), c(k, m);
    std::copy_n(xtx.data() + f * k * k, k * k, a.data());
    std::copy_n(xty.data() + f * k * m, k * m, c.data());
    b.xtx.push_back(a);
    b.xty.push_back(c);
    Vector v1(k), v2(m), v3(k), v4(m);
    std::copy_n(mx.data() + f * k, k, v1.data());
    std::copy_n(my.data() + f * m, m, v2.data());
    std::copy_n(sx.data() + f * k, k, v3.data());
    std::copy_n(sy.data() + f * m, m, v4.data());
    b.mx.push_back(v1);
    b.my.push_back(v2);
    b.sx.push_back(v3);
    b.sy.push_back(v4);
  }
  return b;
}

// ------------------------------------------------------------ test_fast.cpp
void precompute_global_worked_values() {  // 25-38
  const auto cache = precompute_global(micro_case(), kAllOn);
  CHECK(cache.xtx(0, 0) == 35.0);
  CHECK(cache.xty(0, 0) == 44.0);
  CHECK(near(cache.mean_x(0), 3.0, 1e-12));
  CHECK(near(cache.mean_y(0), 4.0, 1e-12));
  CHECK(cache.sum_x(0) == 9.0);
  CHECK(cache.sum_y(0) == 12.0);
  CHECK(cache.sum_sq_x(0) == 35.0);
  CHECK(cache.sum_sq_y(0) == 56.0);
  CHECK(cache.n_rows == 3);
  CHECK(cache.sum_x(0) == 3.0 * cache.mean_x(0));
}

void precompute_global_degenerate() {  // 40-54
  const DatasetPair zero(Matrix::Zero(3, 2), Matrix::Zero(3, 1));
  const auto cache = precompute_global(zero, kAllOn);
  CHECK(cache.xtx.isZero(0.0));
  CHECK(cache.xty.isZero(0.0));
  CHECK(cache.mean_x.isZero(0.0));
  CHECK(cache.sum_sq_y.isZero(0.0));
  Matrix eye = Matrix::Identity(2, 2);
  const auto cache2 = precompute_global(DatasetPair(eye, Matrix::Ones(2, 1)), {});
  CHECK(cache2.xtx == Matrix::Identity(2, 2));
  CHECK(cache2.xty == Matrix::Ones(2, 1));
  CHECK(cache2.mean_x.size() == 0);
  CHECK(cache2.sum_sq_x.size() == 0);
}

void training_mean_worked_values() {  // 56-68
  Vector g(1), v(1);
  g << 3;
  v << 5;
  CHECK(near(training_mean(g, v, 3, 1)(0), 2.0, 1e-15));
  g << 4;
  v << 6;
  CHECK(near(training_mean(g, v, 3, 1)(0), 3.0, 1e-15));
  g << 1.25;
  v << 1.25;
  CHECK(near(training_mean(g, v, 10, 4)(0), 1.25, 1e-15));
  CHECK_THROWS_AS(training_mean(g, v, 3, 3), std::invalid_argument);
}

void training_std_worked_values() {  // 70-95
  Vector m(1), s(1), q(1);
  m << 2;
  s << 4;
  q << 10;
  CHECK(near(training_std(m, s, q, 2)(0), std::sqrt(2.0), 1e-15));
  m << 4;
  s << 8;
  q << 32;
  CHECK(training_std(m, s, q, 2)(0) == 1.0);
  m << 3;
  s << 6;
  q << 26;
  CHECK(near(training_std(m, s, q, 2)(0), 2.0 * std::sqrt(2.0), 1e-15));
  CHECK_THROWS_AS(training_std(m, s, q, 1), scalability_error);
  const double v0 = 0.1;
  m << v0;
  s << 3 * v0;
  q << 3 * v0 * v0 * (1.0 - 1e-16);
  CHECK(training_std(m, s, q, 3)(0) == 1.0);
}

void fold_products_micro() {  // 97-122
  const auto data = micro_case();
  const std::vector<Index> v_rows{2};
  PreprocessConfig center{true, true, false, false};
  auto r = fold_products(precompute_global(data, center), data, v_rows, center, 2);
  CHECK(r.fold_id == 2);
  CHECK(near(r.xtx_t(0, 0), 2.0, 1e-12));
  CHECK(near(r.xty_t(0, 0), 2.0, 1e-12));
  r = fold_products(precompute_global(data, kAllOn), data, v_rows, kAllOn);
  CHECK(near(r.xtx_t(0, 0), 1.0, 1e-12));
  CHECK(near(r.xty_t(0, 0), 1.0, 1e-12));
  r = fold_products(precompute_global(data, {}), data, v_rows, {});
  CHECK(near(r.xtx_t(0, 0), 10.0, 1e-12));
  CHECK(near(r.xty_t(0, 0), 14.0, 1e-12));
  PreprocessConfig cx{true, false, false, false};
  PreprocessConfig cy{false, true, false, false};
  CHECK(near(fold_products(precompute_global(data, cx), data, v_rows, cx).xty_t(0, 0), 2.0, 1e-12));
  CHECK(near(fold_products(precompute_global(data, cy), data, v_rows, cy).xty_t(0, 0), 2.0, 1e-12));
}

void fold_products_rejects() {  // 124-132
  const auto data = micro_case();
  const auto cache = precompute_global(data, {});
  CHECK_THROWS_AS(fold_products(cache, data, {}, {}), std::invalid_argument);
  CHECK_THROWS_AS(fold_products(cache, data, {0, 1, 2}, {}), std::invalid_argument);
  PreprocessConfig scale{false, false, true, true};
  const auto cache2 = precompute_global(data, scale);
  CHECK_THROWS_AS(fold_products(cache2, data, {0, 1}, scale), scalability_error);
}

void fast_matches_baseline_all_16() {  // 134-158
  std::mt19937_64 rng(8);
  const auto data = random_dataset(40, 5, 3, rng);
  const auto part = random_partitioning(40, 7, rng);
  for (int bits = 0; bits < 16; ++bits) {
    const auto cfg = from_bits(bits);
    const auto fast = run_all_folds(data, part, cfg);
    const auto base = oracle_baseline(data, part, cfg);
    CHECK(fast.size() == base.xtx.size());
    for (size_t f = 0; f < fast.size(); ++f) {
      CHECK(fast[f].fold_id == static_cast<int>(f) + 1);
      CHECK(max_rel_diff(fast[f].xtx_t, base.xtx[f]) <= 1e-8);
      CHECK(max_rel_diff(fast[f].xty_t, base.xty[f]) <= 1e-8);
      if (cfg.any()) {
        CHECK(max_rel_diff(fast[f].stats.mean_x_t, base.mx[f]) <= 1e-12);
        CHECK(max_rel_diff(fast[f].stats.mean_y_t, base.my[f]) <= 1e-12);
      }
      if (cfg.scale_x) CHECK(max_rel_diff(fast[f].stats.std_x_t, base.sx[f]) <= 1e-10);
      if (cfg.scale_y) CHECK(max_rel_diff(fast[f].stats.std_y_t, base.sy[f]) <= 1e-10);
    }
  }
}

void leave_one_out_boundary() {  // 160-165
  const auto results = run_all_folds(micro_case(), {{1, 2, 3}, 3}, kAllOn);
  CHECK(results.size() == 3);
  for (const auto& r : results) CHECK(r.stats.n_train == 2);
}

void statistic_reconstruction() {  // 167-190
  std::mt19937_64 rng(9);
  const auto data = random_dataset(50, 4, 2, rng);
  const auto cache = precompute_global(data, kAllOn);
  for (int trial = 0; trial < 100; ++trial) {
    std::vector<Index> v_rows;
    for (Index i = 0; i < 50; ++i)
      if (rng() % 3 == 0) v_rows.push_back(i);
    if (v_rows.empty() || v_rows.size() > 48) continue;
    const auto r = fold_products(cache, data, v_rows, kAllOn);
    const Matrix xt = gather_rows(data.x(), complement_rows(v_rows, 50));
    const double nt = static_cast<double>(xt.rows());
    Vector mean(4);
    for (Index j = 0; j < 4; ++j) {
      double s = 0;
      for (Index i = 0; i < xt.rows(); ++i) s += xt(i, j);
      mean(j) = s / nt;
    }
    CHECK(max_rel_diff(r.stats.mean_x_t, mean) <= 1e-12);
    for (Index j = 0; j < 4; ++j) {
      double v = 0;
      for (Index i = 0; i < xt.rows(); ++i) v += (xt(i, j) - mean(j)) * (xt(i, j) - mean(j));
      v /= (nt - 1.0);
      if (v > 1e-20) CHECK(std::abs(r.stats.std_x_t(j) - std::sqrt(v)) <= 1e-10 * std::sqrt(v));
    }
  }
}

void thread_count_invariance() {  // 217-229
  std::mt19937_64 rng(12);
  const auto data = random_dataset(60, 6, 2, rng);
  const auto part = random_partitioning(60, 9, rng);
  const auto serial = run_all_folds(data, part, kAllOn, 1);
  const auto parallel = run_all_folds(data, part, kAllOn, 4);
  for (size_t f = 0; f < serial.size(); ++f) {
    CHECK(std::memcmp(serial[f].xtx_t.data(), parallel[f].xtx_t.data(), sizeof(double) * serial[f].xtx_t.size()) == 0);
    CHECK(std::memcmp(serial[f].xty_t.data(), parallel[f].xty_t.data(), sizeof(double) * serial[f].xty_t.size()) == 0);
  }
}

// ------------------------------------------------------------ test_core.cpp
void hadamard_values() {  // 9-67
  Matrix m2(2, 2);
  m2 << 6, 4, 2, 8;
  Vector l2(2), r2(2);
  l2 << 2, 1;
  r2 << 3, 2;
  const Matrix out = hadamard_outer_divide(m2, l2, r2);
  for (Index i = 0; i < 2; ++i)
    for (Index j = 0; j < 2; ++j) CHECK(out(i, j) == m2(i, j) / (l2(i) * r2(j)));
  CHECK(out(1, 1) == 4.0);
  Matrix ones = Matrix::Ones(2, 2);
  Vector ok = Vector::Ones(2), bad(2);
  bad << 1.0, 0.0;
  CHECK_THROWS_AS(hadamard_outer_divide(ones, bad, ok), std::invalid_argument);
  bad << 1.0, -2.0;
  CHECK_THROWS_AS(hadamard_outer_divide(ones, ok, bad), std::invalid_argument);
}

void dataset_pair_invariants() {  // test_core.cpp:69-80 (host)
  CHECK_THROWS_AS(DatasetPair(Matrix::Ones(3, 2), Matrix::Ones(4, 1)), dimension_error);
  CHECK_THROWS_AS(DatasetPair(Matrix::Ones(1, 2), Matrix::Ones(1, 1)), dimension_error);
  Matrix bad = Matrix::Ones(3, 2);
  bad(1, 1) = std::numeric_limits<double>::quiet_NaN();
  CHECK_THROWS_AS(DatasetPair(bad, Matrix::Ones(3, 1)), dimension_error);
  const DatasetPair data(Matrix::Ones(3, 2), Matrix::Ones(3, 1));
  CHECK(data.n_rows() == 3 && data.n_features() == 2 && data.n_responses() == 1);
}

// -------------------------------------------------------- test_baseline.cpp
void zero_variance_column() {  // 55-66
  Matrix x(4, 1), y(4, 1);
  x << 4, 9, 4, 4;
  y << 1, 2, 3, 4;
  PreprocessConfig cfg;
  cfg.center_x = cfg.scale_x = true;
  for (const auto& results : {run_all_folds(DatasetPair(x, y), {{1, 1, 2, 2}, 2}, cfg),
                              baseline_fold_products(DatasetPair(x, y), {{1, 1, 2, 2}, 2}, cfg)}) {
    CHECK(results[0].stats.std_x_t(0) == 1.0);
    CHECK(std::abs(results[0].xtx_t(0, 0)) <= 1e-15);
  }
}

void device_baseline_micro_and_errors() {  // test_baseline.cpp:23-53, 136-148
  const auto data = micro_case();
  const Partitioning micro_part{{1, 1, 2}, 2};
  auto r0 = baseline_fold_products(data, micro_part, {});
  CHECK(r0.size() == 2 && r0[1].fold_id == 2);
  CHECK(near(r0[1].xtx_t(0, 0), 10.0, 1e-12) && near(r0[1].xty_t(0, 0), 14.0, 1e-12));
  PreprocessConfig cc{true, true, false, false};
  auto r1 = baseline_fold_products(data, micro_part, cc);
  CHECK(near(r1[1].xtx_t(0, 0), 2.0, 1e-12) && near(r1[1].xty_t(0, 0), 2.0, 1e-12));
  CHECK_THROWS_AS(baseline_fold_products(data, micro_part, kAllOn), scalability_error);
  const auto r = baseline_single_fold(data, {2}, kAllOn, 2);
  CHECK(near(r.xtx_t(0, 0), 1.0, 1e-12) && near(r.xty_t(0, 0), 1.0, 1e-12));
  CHECK(near(r.stats.std_x_t(0), std::sqrt(2.0), 1e-15) && near(r.stats.std_y_t(0), std::sqrt(2.0), 1e-15));
  CHECK_THROWS_AS(baseline_fold_products(data, {{1, 1, 3}, 3}, {}), partition_error);
  CHECK_THROWS_AS(baseline_fold_products(data, {{1, 2}, 2}, {}), dimension_error);
}

void errors_like_the_reference() {  // 136-148
  const DatasetPair data(Matrix::Ones(2, 1) * 2.0, Matrix::Ones(2, 1));
  PreprocessConfig cfg;
  cfg.scale_x = true;
  CHECK_THROWS_AS(run_all_folds(data, {{1, 2}, 2}, cfg), scalability_error);
  CHECK_THROWS_AS(run_all_folds(micro_case(), {{1, 1, 3}, 3}, {}), partition_error);
  CHECK_THROWS_AS(run_all_folds(micro_case(), {{1, 2}, 2}, {}), dimension_error);
}

// ------------------------------------------------------- test_partition.cpp
void partition_predicates() {  // 11-91 (host)
  const auto idx = build_validation_partitions({{1, 2, 1}, 2});
  CHECK((idx.sets[0] == std::vector<Index>{0, 2}) && (idx.sets[1] == std::vector<Index>{1}));
  CHECK(!validate_partitioning({1, 2}, 2).has_value());
  auto e = validate_partitioning({1, 3, 1}, 3);
  CHECK(e.has_value() && e->find("fold 2") != std::string::npos);
  e = validate_partitioning({1, 2, 0}, 2);
  CHECK(e.has_value() && e->find("outside") != std::string::npos);
  CHECK(validate_partitioning({1}, 1).has_value());
  CHECK(validate_partitioning({1, 2, 3}, 4).has_value());
  CHECK(!check_scalable({{1, 2, 3}, 3}).has_value());
  CHECK(check_scalable({{1, 2}, 2}).has_value());
  auto u = check_scalable({{1, 1, 1, 2}, 2});
  CHECK(u.has_value() && u->find("fold 1") != std::string::npos);
  CHECK((complement_rows({1, 3}, 5) == std::vector<Index>{0, 2, 4}));
  std::mt19937_64 r(5489);
  uint64_t v = 0;
  for (int i = 0; i < 10000; ++i) v = r();
  CHECK(v == 9981545732273789042ULL);
}

// ----------------------------------------------------------- acceptance.cpp
void acceptance_c1() {  // 62-84
  std::mt19937_64 rng(101);
  const auto data = random_dataset(200, 30, 5, rng);
  double worst = 0.0;
  for (int p : {2, 5, 10, 200}) {
    const auto part = random_partitioning(200, p, rng);
    std::vector<PreprocessConfig> cfgs;
    for (int bits = 0; bits < 16; ++bits) cfgs.push_back(from_bits(bits));
    const auto all = run_all_folds_configs(data, part, cfgs);  // one Gram pass, 16 configs
    for (int bits = 0; bits < 16; ++bits) {
      const auto base = oracle_baseline(data, part, cfgs[bits]);
      for (size_t f = 0; f < all[bits].size(); ++f) {
        worst = std::max(worst, max_rel_diff(all[bits][f].xtx_t, base.xtx[f]));
        worst = std::max(worst, max_rel_diff(all[bits][f].xty_t, base.xty[f]));
      }
    }
  }
  std::printf("  acceptance C1 worst max_rel_diff %.3e\n", worst);
  CHECK(worst <= 1e-8);
}

// Lazy per-fold generation (beyond the reference API): same bits as run_all_folds_configs, early stop honoured.
void for_each_fold_streams_the_same_results() {
  std::mt19937_64 rng(77);
  const auto data = random_dataset(300, 12, 3, rng);
  const auto part = random_partitioning(300, 41, rng);
  const std::vector<PreprocessConfig> cfgs{from_bits(15), from_bits(0), from_bits(12)};
  const auto all = run_all_folds_configs(data, part, cfgs);
  int seen = 0;
  bool same = true;
  for_each_fold(
      data, part, cfgs,
      [&](int c, FoldResult&& r) {
        const FoldResult& ref = all[c][r.fold_id - 1];
        same = same && r.xtx_t == ref.xtx_t && r.xty_t == ref.xty_t && r.stats.n_val == ref.stats.n_val &&
               r.stats.std_x_t == ref.stats.std_x_t && r.stats.mean_y_t == ref.stats.mean_y_t;
        ++seen;
      },
      /*batch=*/7);
  CHECK(same);
  CHECK(seen == 3 * 41);
  int calls = 0;
  for_each_fold(data, part, cfgs, [&](int, FoldResult&&) { return ++calls == 5; }, 4);
  CHECK(calls == 5);
}

}  // namespace

int main(int argc, char** argv) {
  const bool host_only = argc > 1 && std::string(argv[1]) == "--host";
  struct T {
    const char* name;
    std::function<void()> fn;
    bool device;
  };
  const std::vector<T> tests = {
      {"dataset_pair_invariants", dataset_pair_invariants, false},
      {"partition_predicates", partition_predicates, false},
      {"precompute_global_worked_values", precompute_global_worked_values, true},
      {"precompute_global_degenerate", precompute_global_degenerate, true},
      {"training_mean_worked_values", training_mean_worked_values, true},
      {"training_std_worked_values", training_std_worked_values, true},
      {"fold_products_micro", fold_products_micro, true},
      {"fold_products_rejects", fold_products_rejects, true},
      {"fast_matches_baseline_all_16", fast_matches_baseline_all_16, true},
      {"leave_one_out_boundary", leave_one_out_boundary, true},
      {"statistic_reconstruction", statistic_reconstruction, true},
      {"thread_count_invariance", thread_count_invariance, true},
      {"hadamard_values", hadamard_values, true},
      {"zero_variance_column", zero_variance_column, true},
      {"device_baseline_micro_and_errors", device_baseline_micro_and_errors, true},
      {"errors_like_the_reference", errors_like_the_reference, true},
      {"acceptance_c1", acceptance_c1, true},
      {"for_each_fold_streams_the_same_results", for_each_fold_streams_the_same_results, true},
  };
  int failed_tests = 0;
  for (const auto& t : tests) {
    if (host_only && t.device) continue;
    const int before = g_fail;
    try {
      t.fn();
    } catch (const std::exception& e) {
      ++g_fail;
      std::printf("  exception: %s\n", e.what());
    }
    const bool ok = g_fail == before;
    failed_tests += !ok;
    std::printf("%s %s\n", ok ? "PASS" : "FAIL", t.name);
  }
  std::printf("%d checks, %d failed, %d failing tests\n", g_checks, g_fail, failed_tests);
  return failed_tests ? 1 : 0;
}
