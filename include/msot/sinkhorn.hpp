// msot/sinkhorn.hpp — the solver operations of SPEC.md (sinkhorn_core
// :122-242, multiscale :244-323), running on the GPU through the C ABI of
// include/msot_gpu.h.  Failures surface as DataError / NumericError (the
// reference's types, common.hpp) or DeviceError.
#pragma once

#include <cmath>
#include <limits>
#include <memory>
#include <vector>

#include "../msot_gpu.h"
#include "common.hpp"
#include "measure.hpp"

namespace msot {

// SolverParams + the multiscale knobs (msot_params).
struct SolverParams {
  double blur = 0.05;
  double reach = std::numeric_limits<double>::infinity();
  CostSpec cost{};
  double scaling = 0.9;
  int max_full_iters = 10000;
  bool multiscale = false;
  int retruncate = 0;
  double cluster_scale = 0.0;  // <= 0: automatic
  double theta = 20.0;
  double switch_factor = 2.0;
  int mask_rule = 0;
  int transfer_rule = 0;
  int pair_eval = 1;   // evaluate-once fine phase
  int clusters = 0;    // D > 3: K-means clusters per measure (0 = ceil(sqrt(N)))
  int seed = 0;        // K-means seeding
  int super_level = -1;  // voxel multiscale super-voxel level: -1 auto, 0 off, 1 on

  msot_params to_c() const;
};

struct EpsSchedule {
  std::vector<double> sigma, eps, lambda;
  std::size_t size() const { return sigma.size(); }
};

// a_xx (N), b_yy (M), a_xy (M), b_yx (N) and the final eps.
struct DualPotentials {
  std::vector<double> a_xx, b_yy, a_xy, b_yx;
  double eps = 0.0;
};

// One GPU (RAII over msot_ctx).  One host thread per Device.
class Device {
 public:
  explicit Device(int device = 0);
  Device(int device, int rank, int world, const unsigned char nccl_id[128]);
  ~Device();
  Device(const Device&) = delete;
  Device& operator=(const Device&) = delete;
  msot_ctx* get() const { return ctx_; }

 private:
  msot_ctx* ctx_ = nullptr;
};

// The calling thread's default device (cuda:0), created on first use.
Device& default_device();

double diameter_estimate(const DiscreteMeasure& a, const DiscreteMeasure& b, double blur);
EpsSchedule make_schedule(double d, const SolverParams& params);

// Row-wise softmin of SPEC.md:164-172 on the GPU: for every atom x_i of
// `rows`, -lambda eps log sum_j w_j exp((h_j - C(x_i, y_j)) / eps) over the
// atoms of `cols` (p = 2).
std::vector<double> softmin(const DiscreteMeasure& rows, const DiscreteMeasure& cols,
                            const std::vector<double>& h, double eps, double lambda = 1.0,
                            Device& dev = default_device());

DualPotentials symmetric_sinkhorn(const DiscreteMeasure& a, const DiscreteMeasure& b,
                                  const SolverParams& params, Device& dev = default_device());
DualPotentials multiscale_sinkhorn(const DiscreteMeasure& a, const DiscreteMeasure& b,
                                   SolverParams params, Device& dev = default_device());
double divergence(const DiscreteMeasure& a, const DiscreteMeasure& b, const SolverParams& params,
                  Device& dev = default_device());

// plan_entry: a_i b_j exp((f_i + g_j - C(x_i, y_j)) / eps)
// with (f, g) = (b_yx, a_xy); host-side.
double plan_entry(std::size_t i, std::size_t j, const DiscreteMeasure& a,
                  const DiscreteMeasure& b, const DualPotentials& duals,
                  const SolverParams& params);
// plan_apply: (pi v)_i on the GPU without materialising pi
// (D <= 3).
std::vector<double> plan_apply(const DiscreteMeasure& a, const DiscreteMeasure& b,
                               const DualPotentials& duals, const SolverParams& params,
                               const std::vector<double>& v, Device& dev = default_device());
// ot_value: the dual objective of PAPER.md eq. 3 at
// (f, g) = (b_yx, a_xy); the plan mass term comes from plan_apply(1).
double ot_value(const DiscreteMeasure& a, const DiscreteMeasure& b, const DualPotentials& duals,
                const SolverParams& params, Device& dev = default_device());

}  // namespace msot
