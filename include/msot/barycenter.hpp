// msot/barycenter.hpp — gradients_barycenter module of SPEC.md:325-398
// (PAPER.md:374-386): the envelope-theorem position gradient of S_eps and the
// Wasserstein barycenter by descent on the atom positions, on the GPU.
#pragma once

#include <vector>

#include "measure.hpp"
#include "sinkhorn.hpp"

namespace msot {

// grad_weights: gradient of S with respect to the weights
// of a, potentials frozen: (rho + eps/2)(e^{-a_xx/rho} - e^{-b_yx/rho}) for a
// finite reach, b_yx - a_xx + eps (sum a - sum b) for reach = inf; host-side.
std::vector<double> grad_weights(const DiscreteMeasure& a, const DiscreteMeasure& b,
                                 const DualPotentials& duals, const SolverParams& params);

// grad_positions, p = 2: N x D (row-major) gradient of
// S(a, b) with respect to the atoms of a.
std::vector<double> grad_positions(const DiscreteMeasure& a, const DiscreteMeasure& b,
                                   const SolverParams& params, double* loss = nullptr,
                                   Device& dev = default_device());

struct BarycenterConfig {
  int iters = 100;
  double step = 1.0;
  double tol = 1e-4;   // relative decrease below which the descent stops
};

struct BarycenterResult {
  DiscreteMeasure measure;        // the barycenter (init's weights, moved atoms)
  std::vector<double> loss;       // mean divergence per accepted step (iters + 1)
};

// barycenter: minimises (1/K) sum_k S(alpha, beta_k) over
// the atom positions of `init` (weights frozen), step halved <= 10 times.
BarycenterResult barycenter(const std::vector<DiscreteMeasure>& targets,
                            const DiscreteMeasure& init, const SolverParams& params,
                            const BarycenterConfig& cfg = {}, Device& dev = default_device());

}  // namespace msot
