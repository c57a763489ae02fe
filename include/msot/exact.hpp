// msot/exact.hpp — the exact transport oracle (module
// exact_oracle): DensePlan and exact_ot, a single-threaded network simplex on
// the host (csrc/exact_ot.cpp).  Ground truth for small instances (N*M <=
// 1e6): acceptance criteria 1 and 9 and `msot verify`.
#pragma once

#include <cstddef>
#include <vector>

#include "measure.hpp"

namespace msot {

// N x M nonnegative plan, row sums a and column sums b (within 1e-9), and its
// value sum pi_ij C_ij.
struct DensePlan {
  std::size_t rows = 0, cols = 0;
  std::vector<double> pi;  // row-major
  double value = 0.0;
  double operator()(std::size_t i, std::size_t j) const { return pi[i * cols + j]; }
};

// Throws DataError for unbalanced masses (|sum a - sum b| > 1e-9) or N*M > 1e6.
DensePlan exact_ot(const DiscreteMeasure& a, const DiscreteMeasure& b, const CostSpec& spec = {});

}  // namespace msot
