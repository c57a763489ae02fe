// msot/labels.hpp — the labeling module of SPEC.md:400-467 (§2,
// eq. 7): atlas label transfer through the implicit transport plan, flip
// resolution and outlier classification, on the GPU through the C ABI.
#pragma once

#include <string>
#include <vector>

#include "measure.hpp"
#include "sinkhorn.hpp"

namespace msot {

// L classes, their names, one class index per atlas atom.
struct LabelSet {
  int L = 0;
  std::vector<std::string> names;
  std::vector<int> assignments;
};

// N x L nonnegative scores (row-major) and the row masses.
struct SoftLabels {
  std::size_t n = 0;
  int L = 0;
  std::vector<double> scores;
  std::vector<double> row_mass;
  double score(std::size_t i, int l) const { return scores[i * L + l]; }
};

// transfer_labels:
//   Lab_i = sum_j b_j l_j exp((f_i + g_j - C(x_i, y_j)) / eps) / ...,
// with (f, g) = (b_yx, a_xy) the converged cross potentials of (a, b).  The
// duals are computed on the device by the same call (the GPU keeps them
// resident), so the precondition "duals converged for (a, b)" holds by
// construction; the plan is never materialised.
SoftLabels transfer_labels(const DiscreteMeasure& a, const DiscreteMeasure& b,
                           const LabelSet& labels, const SolverParams& params,
                           Device& dev = default_device());

// resolve_flips: one row per original fibre, the
// orientation with the larger row mass (ties -> the original).
SoftLabels resolve_flips(const SoftLabels& soft, const FlipMap& map);

// classify: OUTLIER (-1) iff row_mass < tau, else the
// argmax class (ties -> lowest index); confidence = max score / row_mass.
constexpr int OUTLIER = -1;
struct Classification {
  std::vector<int> label;
  std::vector<double> confidence;
};
Classification classify(const SoftLabels& soft, double tau = 0.5);

}  // namespace msot
