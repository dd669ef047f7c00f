// Compile-only check of the headers' Eigen branch (include/cvgram/core.hpp: Matrix / Vector / Index are the
// reference's Eigen typedefs when <Eigen/Dense> is on the include path).  Eigen itself is absent from this
// image, so eigen_shape/Eigen/Dense stands in with Eigen's spelling of the members the headers may touch.
#include "cvgram/cvgram.hpp"

#ifndef CVGRAM_WITH_EIGEN
#error "the Eigen branch was not selected"
#endif

int eigen_shape_check() {
  using namespace cvgram;
  static_assert(std::is_same_v<Matrix, Eigen::Matrix<double, Eigen::Dynamic, Eigen::Dynamic, Eigen::RowMajor>>);
  static_assert(std::is_same_v<Vector, Eigen::RowVectorXd>);
  auto data = random_dataset(40, 3, 2, 7);
  auto part = random_partitioning(40, 4, 8);
  auto runs = run_all_folds(data, part, PreprocessConfig{true, true, true, true});
  auto base = baseline_fold_products(data, part, PreprocessConfig{true, false, true, false});
  auto g = precompute_global(data, PreprocessConfig{true, true, false, false});
  auto r = fold_products(g, data, build_validation_partitions(part).sets[0], PreprocessConfig{}, 1);
  auto h = hadamard_outer_divide(r.xtx_t, r.stats.std_x_t, r.stats.std_x_t);
  return static_cast<int>(runs.size() + base.size()) + (max_rel_diff(h, h) == 0.0) +
         (rel_frobenius_dist(r.xtx_t, r.xtx_t) == 0.0);
}
